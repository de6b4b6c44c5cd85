import sys, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.kernels import native
from paper_1705_05249_b200.kernels.dispatch import gemm_native
ctx = tb.context_create(tb.host_device())
T = tb.Transpose
cfg = tb.routines.common.get_store(ctx).resolve('gemm', tb.Precision.H, ctx.device, (1, 1, 1))[0]
for (M, N, K) in ((8192, 8192, 16384), (8192, 8192, 32768), (16384, 16384, 4096), (16384, 16384, 8192), (16384, 16384, 16384), (4096, 4096, 32768), (32768, 32768, 2048)):
    a = tb.buffer_from_tensor(ctx, tb.Precision.H, (torch.rand(M*K, device='cuda')*2-1).half())
    b = tb.buffer_from_tensor(ctx, tb.Precision.H, (torch.rand(K*N, device='cuda')*2-1).half())
    c = tb.buffer_alloc(ctx, tb.Precision.H, M*N)
    res = []
    for flags in (0, native.FLAG_NO_2SM):
        rec = {}
        fn = lambda: rec.update(gemm_native(ctx, tb.Precision.H, tb.Layout.ROW_MAJOR, T.NO, T.NO, M, N, K, 1.0, a, 0, K, b, 0, N, 0.0, c, 0, N, cfg, flags))
        fn(); torch.cuda.synchronize()
        reps = max(2, int(4e12 / (2*M*N*K)))
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res.append(f"{rec['kernel'][:12]} {2*M*N*K/ms/1e9:7.1f}")
    print(M, N, K, ' | '.join(res), flush=True)
    del a, b, c; torch.cuda.empty_cache()
