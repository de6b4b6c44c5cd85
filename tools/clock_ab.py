"""HGEMM 8192^3: this library's pair kernels vs cuBLAS (torch.matmul) in
long back-to-back runs, with nvidia-smi sampling SM clock and power in the
background — is the gap to cuBLAS clock (power) or per-clock throughput?
Dev tool."""
import subprocess
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.kernels.dispatch import gemm_native  # noqa: E402

S = 8192
ctx = tb.context_create(tb.host_device())
H = tb.Precision.H
at = (torch.rand(S * S, device="cuda") * 2 - 1).half()
bt = (torch.rand(S * S, device="cuda") * 2 - 1).half()
a, b = tb.buffer_from_tensor(ctx, H, at), tb.buffer_from_tensor(ctx, H, bt)
c = tb.buffer_alloc(ctx, H, S * S)
A, B = at.view(S, S), bt.view(S, S)
names = ("MWG", "NWG", "KWG", "STAGES", "CTA_GROUP", "SPLIT_K", "GROUP_M")


def ours(nwg):
    cfg = tb.Configuration.make("gemm_b200", dict(zip(names, (256, nwg, 64, 0, 2, 1, 0))))
    return lambda: gemm_native(ctx, H, tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.NO, S, S, S, 1.0, a, 0, S,
                               b, 0, S, 0.0, c, 0, S, cfg, 0)


def cublas():
    return lambda: torch.matmul(A, B)


def run(name, fn, iters=300):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "20"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    vals = [tuple(float(x) for x in ln.split(",")) for ln in out if ln.count(",") == 1]
    vals = vals[len(vals) // 4: -2] or vals
    mhz = sorted(v[0] for v in vals)[len(vals) // 2] if vals else 0
    pw = sorted(v[1] for v in vals)[len(vals) // 2] if vals else 0
    us = e0.elapsed_time(e1) * 1e3 / iters
    tf = 2 * S ** 3 / us / 1e6
    print(f"{name:12s} {us:8.1f} us  {tf:7.1f} TF  sm {mhz:6.0f} MHz  power {pw:6.1f} W  "
          f"TF per GHz {tf / (mhz / 1000) if mhz else 0:7.1f}", flush=True)


for rep in range(2):
    run("cublas", cublas())
    run("ours 256x256", ours(256))
    run("ours 256x512", ours(512))
