"""DL shapes (C3), all transposes at 8192, and the 32768^3 HGEMM (C5 on one GPU)."""
import sys, time, torch
sys.path.insert(0, '.')
import numpy as np
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.kernels.dispatch import gemm_native
ctx = tb.context_create(tb.host_device())
T = tb.Transpose
store = tb.routines.common.get_store(ctx)
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)/reps
def bench(prec, lay, ta, tbt, m, n, k, reps=10):
    a = tb.buffer_from_tensor(ctx, prec, (torch.rand(m*k, device='cuda')*2-1).to(prec.torch_dtype))
    b = tb.buffer_from_tensor(ctx, prec, (torch.rand(k*n, device='cuda')*2-1).to(prec.torch_dtype))
    c = tb.buffer_alloc(ctx, prec, m*n)
    cfg = store.resolve("gemm", prec, ctx.device, (m, n, k))[0]
    rows = (m, k) if ta is T.NO else (k, m)
    lda = rows[0] if lay is tb.Layout.COL_MAJOR else rows[1]
    rows = (k, n) if tbt is T.NO else (n, k)
    ldb = rows[0] if lay is tb.Layout.COL_MAJOR else rows[1]
    ldc = m if lay is tb.Layout.COL_MAJOR else n
    rec = {}
    fn = lambda: rec.update(gemm_native(ctx, prec, lay, ta, tbt, m, n, k, 1.0, a, 0, lda, b, 0, ldb, 0.0, c, 0, ldc, cfg))
    ms = timeit(fn, reps)
    print(f"{prec.value} {lay.value} {ta.value}{tbt.value} {m}x{n}x{k}: {ms*1e3:9.1f} us {2*m*n*k/ms/1e9:8.1f} TFLOPS  {rec['kernel']}", flush=True)
for prec in (tb.Precision.H, tb.Precision.S):
    for (m, n, k) in ((64, 3136, 576), (4096, 128, 9216), (1024, 1024, 1024), (256, 256, 256)):
        bench(prec, tb.Layout.ROW_MAJOR, T.NO, T.NO, m, n, k)
    for ta in (T.NO, T.YES):
        for tbt in (T.NO, T.YES):
            bench(prec, tb.Layout.ROW_MAJOR, ta, tbt, 8192, 8192, 8192, reps=3)
if len(sys.argv) > 1:
    bench(tb.Precision.H, tb.Layout.ROW_MAJOR, T.NO, T.NO, 32768, 32768, 32768, reps=2)
