import sys, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
ctx = tb.context_create(tb.host_device())
L, T = tb.Layout.ROW_MAJOR, tb.Transpose
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)/reps
for prec in (tb.Precision.H, tb.Precision.S):
    for s in (16, 32, 64):
        e = s*s; B = 16384
        a = tb.buffer_from_tensor(ctx, prec, (torch.rand(B*e, device='cuda')*2-1).to(prec.torch_dtype))
        b = tb.buffer_from_tensor(ctx, prec, (torch.rand(B*e, device='cuda')*2-1).to(prec.torch_dtype))
        c = tb.buffer_alloc(ctx, prec, B*e)
        for lay in (tb.Layout.ROW_MAJOR, tb.Layout.COL_MAJOR):
            fn = lambda: tb.gemm_strided_batched(ctx, lay, T.NO, T.NO, s, s, s, 1.0, a, e, b, e, 0.0, c, e, B)
            ms = timeit(fn)
            print(prec.value, s, lay.value, ctx.last_launch.native['kernel'], f"{ms*1e3:.1f} us {3*e*B*prec.elemsize/ms/1e6:.0f} GB/s {2*s**3*B/ms/1e9:.1f} TFLOPS", flush=True)
