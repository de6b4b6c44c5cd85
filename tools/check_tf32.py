import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
ctx = tb.context_create(tb.host_device())
T = tb.Transpose
for lay in (tb.Layout.COL_MAJOR, tb.Layout.ROW_MAJOR):
    for ta in (T.NO, T.YES):
        for tbt in (T.NO, T.YES):
            m, n, k = 512, 512, 256
            A = torch.rand(m*k, device='cuda')*2-1
            B = torch.rand(k*n, device='cuda')*2-1
            a = tb.buffer_from_tensor(ctx, tb.Precision.S, A)
            b = tb.buffer_from_tensor(ctx, tb.Precision.S, B)
            c = tb.buffer_alloc(ctx, tb.Precision.S, m*n)
            c2 = tb.buffer_alloc(ctx, tb.Precision.S, m*n)
            tb.gemm(ctx, lay, ta, tbt, m, n, k, 1.0, a, b, 0.0, c, tf32=True)
            kern = ctx.last_launch.native['kernel']
            tb.gemm(ctx, lay, ta, tbt, m, n, k, 1.0, a, b, 0.0, c2)
            x, y = c.device_tensor(), c2.device_tensor()
            print(lay.value, ta.value, tbt.value, kern, 'maxabs', x.abs().max().item(), 'maxdiff', (x-y).abs().max().item(), 'ref maxabs', y.abs().max().item(), flush=True)
