"""Launch overhead around the C3 split-K HGEMM: event time (L2 flushed, as
bench.py) of a 1-element torch kernel, of small / C3 HGEMMs through the
library, and of cuBLAS on C3.  Run with and without TB_NO_PDL=1.  Dev tool."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402

ctx = tb.context_create(tb.host_device())
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=30, flush=True):
    for _ in range(3):
        fn()
    ev = []
    for _ in range(reps):
        if flush:
            flush_buf.fill_(1)
            clean.view(torch.int64).sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return v[len(v) // 2]


x = torch.zeros(1, device="cuda")
print(f"torch 1-element add: {t(lambda: x.add_(1)):7.2f} us (flushed)  {t(lambda: x.add_(1), flush=False):7.2f} us")
H = tb.Precision.H
for (m, n, k) in ((128, 128, 64), (128, 128, 9216), (4096, 128, 9216), (1024, 1024, 1024)):
    a = tb.buffer_from_tensor(ctx, H, (torch.rand(m * k, device="cuda") * 2 - 1).half())
    b = tb.buffer_from_tensor(ctx, H, (torch.rand(k * n, device="cuda") * 2 - 1).half())
    c = tb.buffer_alloc(ctx, H, m * n)

    def f():
        tb.gemm(ctx, tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.NO, m, n, k, 1.0, a, b, 0.0, c)

    us = t(f)
    print(f"tb H {m}x{n}x{k}: {us:7.2f} us flushed, {t(f, flush=False):7.2f} us warm  "
          f"{ctx.last_launch.native['kernel']}", flush=True)
    at = a.device_tensor().view(m, k)
    bt = b.device_tensor().view(k, n)
    print(f"   cuBLAS: {t(lambda: torch.matmul(at, bt)):7.2f} us flushed, "
          f"{t(lambda: torch.matmul(at, bt), flush=False):7.2f} us warm", flush=True)
