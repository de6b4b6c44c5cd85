"""im2col timing: single call after a flush (bench style) vs 20 back-to-back
calls between events vs host time per call."""
import sys, time, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
ctx = tb.context_create(tb.host_device())
c, h, w, kh, kw = 256, 56, 56, 3, 3
rows, cols = c * kh * kw, h * w
for prec in (tb.Precision.H, tb.Precision.S):
    im = tb.buffer_from_tensor(ctx, prec, torch.rand(c * h * w, device='cuda').to(prec.torch_dtype))
    col = tb.buffer_alloc(ctx, prec, rows * cols)
    fn = lambda: tb.im2col(ctx, c, h, w, kh, kw, 1, 1, 1, 1, 1, 1, im, col)
    for _ in range(5): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200): fn()
    host = (time.perf_counter() - t0) / 200 * 1e6
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) / 20 * 1e3
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20): fn()
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    gr = e0.elapsed_time(e1) / 20 * 1e3
    print(f"{prec.value}: host {host:.1f} us/call, back-to-back {b2b:.1f} us, graph {gr:.2f} us", flush=True)
