"""BASELINE config C5 on one B200 (dev tool): 32768^3 HGEMM / SGEMM row-major
NN through `distributed.gemm_sharded`, timed per shard for world = 1, 2, 4, 8
(the compute each rank would run; the multi-GPU run itself needs >1 GPU), plus
the SURVEY §8d correctness check on 64 sampled rows x 64 sampled columns
(float64 product within gemm_tolerance; S also bitwise vs the C oracle)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200 import distributed as D  # noqa: E402
from oracle import gemm_oracle as orc  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
ctx = tb.context_create(tb.host_device())
L, T = tb.Layout.ROW_MAJOR, tb.Transpose.NO
for prec, code in ((tb.Precision.H, "H"), (tb.Precision.S, "S")):
    g = torch.Generator(device="cuda").manual_seed(12345)
    at = (torch.rand(N * N, device="cuda", generator=g) * 2 - 1).to(prec.torch_dtype)
    bt = (torch.rand(N * N, device="cuda", generator=g) * 2 - 1).to(prec.torch_dtype)
    a = tb.buffer_from_tensor(ctx, prec, at)
    b = tb.buffer_from_tensor(ctx, prec, bt)
    c = tb.buffer_alloc(ctx, prec, N * N)
    for world in (1, 2, 4, 8):
        fn = lambda: D.gemm_sharded(ctx, L, T, T, N, N, N, 1.0, a, b, 0.0, c, rank=0, world=world)
        fn()
        torch.cuda.synchronize()
        reps = 2 if (code == "S" and world <= 2) else 3
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        tf = 2.0 * N * N * N / world / ms / 1e9
        print(f"C5 {code} {N}^3 world={world}: rank-0 shard {ms:9.2f} ms  {tf:7.1f} TFLOP/s per GPU  "
              f"({ctx.last_launch.native['kernel']})", flush=True)
    # full product (world = 1) for the check
    D.gemm_sharded(ctx, L, T, T, N, N, N, 1.0, a, b, 0.0, c, rank=0, world=1)
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(1).choice(N, 64, replace=False))
    cols = np.sort(np.random.default_rng(2).choice(N, 64, replace=False))
    ri, ci = torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()
    A = at.view(N, N)[ri].cpu().numpy()
    B = bt.view(N, N)[:, ci].cpu().numpy()
    got = c.device_tensor().view(N, N)[ri][:, ci].cpu().numpy()
    want = orc.wide_oracle(1.0, A, B, 0.0, None)
    tol = orc.gemm_tolerance(A, B, code)
    if code == "H":
        tol = tol + 2.0 ** -11 * np.abs(want)
    err = np.abs(got.astype(np.float64) - want) / tol
    print(f"C5 {code} sampled 64x64 max err/tol = {err.max():.4f}", flush=True)
    assert err.max() <= 1.0
    if code == "S":
        sub = np.zeros(64 * 64, np.float32)
        orc.seqk_gemm("S", True, False, False, 64, 64, N, 1.0, np.ascontiguousarray(A).reshape(-1), 0, N,
                      np.ascontiguousarray(B).reshape(-1), 0, 64, 0.0, sub, 0, 64)
        assert sub.reshape(64, 64).tobytes() == np.ascontiguousarray(got).tobytes()
        print("C5 S sampled 64x64 bitwise equal to the sequential-k C oracle", flush=True)
    del a, b, c, at, bt
    torch.cuda.empty_cache()
