"""im2col probe (dev tool): the bench's ResNet-style layer (256 x 56 x 56,
3x3, pad 1) and the C3 layer (64 channels), H and S, device-timed with the
L2 flushed before every call (bench.py's protocol)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1705_05249_b200 as tb  # noqa: E402

ctx = tb.context_create(tb.host_device())
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=30):
    for _ in range(3):
        fn()
    ev = []
    for _ in range(reps):
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


for c in (256, 64):
    h, w, kh, kw = 56, 56, 3, 3
    for prec in (tb.Precision.H, tb.Precision.S):
        im = tb.buffer_from_tensor(ctx, prec, torch.rand(c * h * w, device="cuda").to(prec.torch_dtype))
        col = tb.buffer_alloc(ctx, prec, c * kh * kw * h * w)
        us = t(lambda: tb.im2col(ctx, c, h, w, kh, kw, 1, 1, 1, 1, 1, 1, im, col))
        nbytes = (c * h * w + c * kh * kw * h * w) * prec.elemsize
        # steady state: 20 calls captured in a CUDA graph, L2-warm, no host overhead
        s_ = torch.cuda.Stream()
        g_ = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s_):
            tb.im2col(ctx, c, h, w, kh, kw, 1, 1, 1, 1, 1, 1, im, col)
            torch.cuda.synchronize()
            with torch.cuda.graph(g_, stream=s_):
                for _ in range(20):
                    tb.im2col(ctx, c, h, w, kh, kw, 1, 1, 1, 1, 1, 1, im, col)
        g_.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g_.replay()
        e1.record()
        torch.cuda.synchronize()
        warm = e0.elapsed_time(e1) * 1e3 / 20
        print(f"{prec.value} im2col {c}x{h}x{w} 3x3: {us:7.2f} us  {nbytes / us / 1e3:7.1f} GB/s  "
              f"(graph, L2-warm: {warm:6.2f} us/call)  {ctx.last_launch.native['kernel']}", flush=True)

# reference points: writing (zero_) and copying a column matrix's bytes
for nbytes in (256 * 9 * 56 * 56 * 2, 256 * 9 * 56 * 56 * 4):
    x = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    y = torch.empty_like(x)
    print(f"torch zero_ {nbytes / 1e6:.1f} MB: {t(lambda: x.zero_()):7.2f} us   "
          f"copy_: {t(lambda: y.copy_(x)):7.2f} us", flush=True)
