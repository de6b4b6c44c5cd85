"""One C3 H launch (4096 x 128 x 9216 row-major NN) for ncu."""
import sys, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
ctx = tb.context_create(tb.host_device())
T = tb.Transpose
m, n, k = 4096, 128, 9216
P = tb.Precision.H
a = tb.buffer_from_tensor(ctx, P, (torch.rand(m * k, device='cuda') * 2 - 1).half())
b = tb.buffer_from_tensor(ctx, P, (torch.rand(k * n, device='cuda') * 2 - 1).half())
c = tb.buffer_alloc(ctx, P, m * n)
for _ in range(3):
    tb.gemm(ctx, tb.Layout.ROW_MAJOR, T.NO, T.NO, m, n, k, 1.0, a, b, 0.0, c)
torch.cuda.synchronize()
print(ctx.last_launch.native)
