"""One launch of each small batched config (for ncu)."""
import sys, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.kernels.dispatch import gemm_strided_batched_native
ctx = tb.context_create(tb.host_device())
T = tb.Transpose
cfg = tb.routines.common.get_store(ctx).resolve("gemm", tb.Precision.H, ctx.device, (1,1,1))[0]
for prec in (tb.Precision.H, tb.Precision.S):
    for s in (32, 64):
        e = s*s; B = 16384
        a = tb.buffer_from_tensor(ctx, prec, (torch.rand(B*e, device='cuda')*2-1).to(prec.torch_dtype))
        b = tb.buffer_from_tensor(ctx, prec, (torch.rand(B*e, device='cuda')*2-1).to(prec.torch_dtype))
        c = tb.buffer_alloc(ctx, prec, B*e)
        gemm_strided_batched_native(ctx, prec, tb.Layout.ROW_MAJOR, T.NO, T.NO, s, s, s, 1.0, a, 0, s, e, b, 0, s, e, 0.0, c, 0, s, e, B, cfg)
        torch.cuda.synchronize()
print("ok")
