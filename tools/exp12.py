"""cProfile of the public gemm call path (host overhead)."""
import sys, cProfile, pstats, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
ctx = tb.context_create(tb.host_device())
T = tb.Transpose
prec = tb.Precision.H
m = n = k = 256
a = tb.buffer_from_tensor(ctx, prec, torch.rand(m*k, device='cuda').half())
b = tb.buffer_from_tensor(ctx, prec, torch.rand(k*n, device='cuda').half())
c = tb.buffer_alloc(ctx, prec, m*n)
f = lambda: tb.gemm(ctx, tb.Layout.ROW_MAJOR, T.NO, T.NO, m, n, k, 1.0, a, b, 0.0, c)
for _ in range(100): f()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(2000): f()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats('tottime').print_stats(25)
