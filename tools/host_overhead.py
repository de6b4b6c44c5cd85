"""Host-side cost of one public ``gemm`` call (CPU-bound loop of tiny
problems; the GPU is idle-waiting) and of its pieces.  Dev tool."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.kernels.dispatch import gemm_native  # noqa: E402

ctx = tb.context_create(tb.host_device())
H = tb.Precision.H
m = n = k = 64
a = tb.buffer_from_tensor(ctx, H, torch.rand(m * k, device="cuda").half())
b = tb.buffer_from_tensor(ctx, H, torch.rand(k * n, device="cuda").half())
c = tb.buffer_alloc(ctx, H, m * n)
L, T = tb.Layout.ROW_MAJOR, tb.Transpose.NO


def per_call(fn, reps=3000):
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / reps * 1e6


print(f"tb.gemm (public routine):     {per_call(lambda: tb.gemm(ctx, L, T, T, m, n, k, 1.0, a, b, 0.0, c)):6.2f} us")
print(f"gemm_native (dispatch layer): "
      f"{per_call(lambda: gemm_native(ctx, H, L, T, T, m, n, k, 1.0, a, 0, k, b, 0, n, 0.0, c, 0, n, None, 0)):6.2f} us")
x = torch.empty(1, device="cuda")
print(f"torch x.add_(1) for scale:    {per_call(lambda: x.add_(1)):6.2f} us")
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for _ in range(2000):
    tb.gemm(ctx, L, T, T, m, n, k, 1.0, a, b, 0.0, c)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
