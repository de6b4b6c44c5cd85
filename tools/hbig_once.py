"""One large row-major NN HGEMM launch through the C-ABI with optional flags (ncu capture helper)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.kernels.dispatch import gemm_native  # noqa: E402
N = int(sys.argv[1]); flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = tb.context_create(tb.host_device())
H, L, T = tb.Precision.H, tb.Layout.ROW_MAJOR, tb.Transpose.NO
a = tb.buffer_from_tensor(ctx, H, (torch.rand(N * N, device="cuda") * 2 - 1).half())
b = tb.buffer_from_tensor(ctx, H, (torch.rand(N * N, device="cuda") * 2 - 1).half())
c = tb.buffer_alloc(ctx, H, N * N)
cfg = tb.routines.common.get_store(ctx).resolve("gemm", H, ctx.device, (N, N, N))[0]
for _ in range(2):
    rec = gemm_native(ctx, H, L, T, T, N, N, N, 1.0, a, 0, N, b, 0, N, 0.0, c, 0, N, cfg, flags)
torch.cuda.synchronize()
print(rec["kernel"])
