"""Effect of the L2-flush style on HBM-bound timings: write-only flush (L2 left
full of dirty lines) vs write + clean read (dirty lines evicted before the
timed kernel)."""
import sys, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
ctx = tb.context_create(tb.host_device())
T, L = tb.Transpose.NO, tb.Layout.ROW_MAJOR
buf1 = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
buf2 = torch.ones(256 << 20, dtype=torch.uint8, device='cuda')
sink = torch.empty(1, dtype=torch.int64, device='cuda')
flush_w = lambda: buf1.fill_(1)
def flush_wr():
    buf1.fill_(1)
    buf2.view(torch.int64).sum()
def run(name, fn):
    for fl_name, fl in (("write", flush_w), ("write+read", flush_wr), ("none", lambda: None)):
        for _ in range(3): fl(); fn()
        ts = []
        for _ in range(20):
            fl()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"{name:28s} flush={fl_name:10s} {sum(ts)/len(ts):8.1f} us", flush=True)
P = tb.Precision.H
m, n, k = 4096, 128, 9216
a = tb.buffer_from_tensor(ctx, P, torch.rand(m * k, device='cuda').half())
b = tb.buffer_from_tensor(ctx, P, torch.rand(k * n, device='cuda').half())
c = tb.buffer_alloc(ctx, P, m * n)
run("hgemm_c3", lambda: tb.gemm(ctx, L, T, T, m, n, k, 1.0, a, b, 0.0, c))
for prec, s in ((tb.Precision.H, 64), (tb.Precision.H, 32), (tb.Precision.S, 32)):
    e, B = s * s, 16384
    a = tb.buffer_from_tensor(ctx, prec, torch.rand(e * B, device='cuda').to(prec.torch_dtype))
    b = tb.buffer_from_tensor(ctx, prec, torch.rand(e * B, device='cuda').to(prec.torch_dtype))
    c = tb.buffer_alloc(ctx, prec, e * B)
    run(f"batched {prec.value}{s}", lambda: tb.gemm_strided_batched(ctx, L, T, T, s, s, s, 1.0, a, e, b, e, 0.0, c, e, B))
