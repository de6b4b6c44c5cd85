"""SGEMM 8192^3 probe (dev tool): our FFMA kernel through the C-ABI vs cuBLAS
FP32 (torch.mm with TF32 disabled), CUDA-event timed, L2 not flushed (large
operands).  `--ours-only --reps 1` is the ncu capture mode."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.kernels import native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--ours-only", action="store_true")
ap.add_argument("--trans", default="NN")
args = ap.parse_args()
N = args.n
torch.backends.cuda.matmul.allow_tf32 = False
so = native.lib()
a = torch.rand(N * N, device="cuda") * 2 - 1
b = torch.rand(N * N, device="cuda") * 2 - 1
c = torch.zeros(N * N, device="cuda")
ta, tbb = (0 if ch == "N" else 1 for ch in args.trans)


def ours():
    rc = so.tb_gemm(1, 1, ta, tbb, N, N, N, 1.0, a.data_ptr(), 0, N, b.data_ptr(), 0, N, 0.0,
                    c.data_ptr(), 0, N, None, 0, torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc


def ev(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t = ev(ours, args.reps)
print(f"ours {args.trans} {N}^3: {t:.3f} ms {2 * N**3 / t / 1e9:.1f} TFLOPS {native.last_launch()['kernel']}")
if not args.ours_only:
    A, B = a.view(N, N), b.view(N, N)
    C = torch.empty(N, N, device="cuda")
    t = ev(lambda: torch.mm(A, B, out=C), args.reps)
    print(f"cublas fp32 {N}^3: {t:.3f} ms {2 * N**3 / t / 1e9:.1f} TFLOPS")
