import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.kernels import native
ctx = tb.context_create(tb.host_device())
L, T = tb.Layout.ROW_MAJOR, tb.Transpose
def gp(nwg, mwg=128, vw=4):
    return tb.GemmParams(MWG=mwg, NWG=nwg, KWG=32, MDIMC=16 if mwg>=64 else 8, NDIMC=16 if nwg >= 64 else 8, MDIMA=16 if mwg>=64 else 8, NDIMB=16 if nwg>=64 else 8, KWI=8, VWM=vw, VWN=vw).to_config()
store = tb.routines.common.get_store(ctx)
# 1. BN invariance of HGEMM bits
for (m,n,k) in ((512,512,512),(256,384,1000),(1024,1024,4096)):
    a = tb.buffer_from_tensor(ctx, tb.Precision.H, (torch.rand(m*k, device='cuda')*2-1).half())
    b = tb.buffer_from_tensor(ctx, tb.Precision.H, (torch.rand(k*n, device='cuda')*2-1).half())
    outs = []
    for nwg in (128, 64, 32):
        store.set_override("gemm", tb.Precision.H, ctx.device, (m,n,k), gp(nwg))
        c = tb.buffer_alloc(ctx, tb.Precision.H, m*n)
        for lay in (tb.Layout.ROW_MAJOR,):
            tb.gemm(ctx, lay, T.NO, T.NO, m, n, k, 1.0, a, b, 0.0, c)
        outs.append((ctx.last_launch.native['kernel'], c.device_tensor().clone()))
    base = outs[0][1]
    print((m,n,k), [(kname, bool(torch.equal(o, base))) for kname, o in outs], flush=True)
store.clear_overrides()
# 2. batched timing per tile choice
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)/reps
for prec in (tb.Precision.H, tb.Precision.S):
    for s in (32, 64):
        e = s*s; B = 16384
        a = tb.buffer_from_tensor(ctx, prec, (torch.rand(B*e, device='cuda')*2-1).to(prec.torch_dtype))
        b = tb.buffer_from_tensor(ctx, prec, (torch.rand(B*e, device='cuda')*2-1).to(prec.torch_dtype))
        c = tb.buffer_alloc(ctx, prec, B*e)
        for nwg in (128, 64, 32):
            store.set_override("gemm", prec, ctx.device, (s,s,s), gp(nwg, mwg=nwg))
            fn = lambda: tb.gemm_strided_batched(ctx, L, T.NO, T.NO, s, s, s, 1.0, a, e, b, e, 0.0, c, e, B)
            ms = timeit(fn)
            bytes_ = 3*e*B*prec.elemsize
            print(prec.value, s, nwg, ctx.last_launch.native['kernel'], f"{ms*1e3:.1f} us {bytes_/ms/1e6:.0f} GB/s", flush=True)
        store.clear_overrides()
# 3. sgemm variants at 4096 / 8192
for N in (4096, 8192):
    a = tb.buffer_from_tensor(ctx, tb.Precision.S, torch.rand(N*N, device='cuda'))
    b = tb.buffer_from_tensor(ctx, tb.Precision.S, torch.rand(N*N, device='cuda'))
    c = tb.buffer_alloc(ctx, tb.Precision.S, N*N)
    for (mwg, nwg) in ((128,128),(128,64),(64,128),(64,64)):
        store.set_override("gemm", tb.Precision.S, ctx.device, (N,N,N), gp(nwg, mwg=mwg))
        fn = lambda: tb.gemm(ctx, L, T.NO, T.NO, N, N, N, 1.0, a, b, 0.0, c)
        ms = timeit(fn, 3)
        print("S", N, ctx.last_launch.native['kernel'], f"{ms:.3f} ms {2*N**3/ms/1e9:.1f} TFLOPS", flush=True)
    store.clear_overrides()
