"""Host overhead vs kernel time for small GEMMs: public API loop, bare C-ABI loop,
CUDA-graph replay of the C-ABI call (kernel-only floor)."""
import sys, time, ctypes, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.kernels import native
ctx = tb.context_create(tb.host_device())
T = tb.Transpose
so = native.lib()

def ev_time(fn, reps):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3

for prec in (tb.Precision.H, tb.Precision.S):
    for (m, n, k) in ((256, 256, 256), (1024, 1024, 1024), (64, 3136, 576), (4096, 128, 9216)):
        dt = prec.torch_dtype
        a = tb.buffer_from_tensor(ctx, prec, (torch.rand(m*k, device='cuda')*2-1).to(dt))
        b = tb.buffer_from_tensor(ctx, prec, (torch.rand(k*n, device='cuda')*2-1).to(dt))
        c = tb.buffer_alloc(ctx, prec, m*n)
        api = lambda: tb.gemm(ctx, tb.Layout.ROW_MAJOR, T.NO, T.NO, m, n, k, 1.0, a, b, 0.0, c)
        t_api = ev_time(api, 50)
        t0 = time.perf_counter()
        for _ in range(200): api()
        t_host = (time.perf_counter() - t0) / 200 * 1e6
        torch.cuda.synchronize()
        pa, pb, pc = a.data_ptr(), b.data_ptr(), c.data_ptr()
        pcode = 0 if prec is tb.Precision.H else 1
        s = torch.cuda.Stream()
        def raw(strm):
            return so.tb_gemm(pcode, 1, 0, 0, m, n, k, 1.0, pa, 0, k, pb, 0, n, 0.0, pc, 0, n, None, 0, strm)
        with torch.cuda.stream(s):
            t_raw = ev_time(lambda: raw(s.cuda_stream), 50)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20): raw(s.cuda_stream)
        t_graph = ev_time(g.replay, 10) / 20
        print(f"{prec.value} {m}x{n}x{k}: api {t_api:7.1f} us (host {t_host:6.1f} us/call)  raw-cabi {t_raw:7.1f} us  graph {t_graph:7.2f} us"
              f" -> {2*m*n*k/t_graph/1e6:7.1f} TFLOPS  {native.last_launch()['kernel']}", flush=True)
