import sys, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.kernels import native
from paper_1705_05249_b200.kernels.dispatch import gemm_native
ctx = tb.context_create(tb.host_device())
T = tb.Transpose
cfg = tb.routines.common.get_store(ctx).resolve('gemm', tb.Precision.H, ctx.device, (1, 1, 1))[0]
N = 8192
a = tb.buffer_from_tensor(ctx, tb.Precision.H, (torch.rand(N*N, device='cuda')*2-1).half())
b = tb.buffer_from_tensor(ctx, tb.Precision.H, (torch.rand(N*N, device='cuda')*2-1).half())
c = tb.buffer_alloc(ctx, tb.Precision.H, N*N)
for flags in (0, native.FLAG_NO_2SM):
    for _ in range(3):
        gemm_native(ctx, tb.Precision.H, tb.Layout.ROW_MAJOR, T.NO, T.NO, N, N, N, 1.0, a, 0, N, b, 0, N, 0.0, c, 0, N, cfg, flags)
    torch.cuda.synchronize()
print("ok")
