"""Large HGEMM probe (dev tool): row-major NN N^3 through the public API, CUDA-event timed."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_05249_b200 as tb  # noqa: E402
ctx = tb.context_create(tb.host_device())
for N in map(int, sys.argv[1:] or ["16384", "32768"]):
    H = tb.Precision.H
    a = tb.buffer_from_tensor(ctx, H, (torch.rand(N * N, device="cuda") * 2 - 1).half())
    b = tb.buffer_from_tensor(ctx, H, (torch.rand(N * N, device="cuda") * 2 - 1).half())
    c = tb.buffer_alloc(ctx, H, N * N)
    T = tb.Transpose.NO
    fn = lambda: tb.gemm(ctx, tb.Layout.ROW_MAJOR, T, T, N, N, N, 1.0, a, b, 0.0, c)
    fn(); torch.cuda.synchronize()
    reps = 5
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"H {N}^3: {ms:.2f} ms {2*N**3/ms/1e9:.1f} TFLOP/s {ctx.last_launch.native['kernel']}", flush=True)
    del a, b, c
    torch.cuda.empty_cache()
