"""Time convgemm against im2col + gemm on the BASELINE C3 conv layer
(64 x 56 x 56 image, 3x3, pad 1 -> (64, 3136, 576) GEMM) and a larger one,
L2 flushed before every call.  Dev tool."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402

ctx = tb.context_create(tb.host_device())
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=20):
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


for prec in (tb.Precision.H, tb.Precision.S):
    for (c, h, w, nk, batch) in ((64, 56, 56, 64, 1), (256, 56, 56, 256, 1), (64, 56, 56, 64, 32)):
        rows, cols = c * 9, h * w
        im = tb.buffer_from_tensor(ctx, prec, torch.rand(batch * c * h * w, device="cuda").to(prec.torch_dtype))
        kern = tb.buffer_from_tensor(ctx, prec, torch.rand(nk * rows, device="cuda").to(prec.torch_dtype))
        res = tb.buffer_alloc(ctx, prec, batch * nk * cols)
        col = tb.buffer_alloc(ctx, prec, rows * cols)

        def fused():
            tb.convgemm(ctx, c, h, w, 3, 3, 1, 1, 1, 1, 1, 1, nk, batch, im, kern, res)

        def two_step():
            for b in range(batch):
                tb.im2col(ctx, c, h, w, 3, 3, 1, 1, 1, 1, 1, 1, im, col, im_offset=b * c * h * w)
                tb.gemm(ctx, tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.YES, nk, cols, rows, 1.0,
                        kern, col, 0.0, res, lda=rows, ldb=rows, c_offset=b * nk * cols, ldc=cols)

        tf = t(fused)
        kname = ctx.last_launch.native["kernel"]
        t2 = t(two_step)
        fl = 2.0 * nk * cols * rows * batch
        print(f"{prec.value} conv {c}x{h}x{w} 3x3 -> {nk} filters, batch {batch}: convgemm {tf:8.1f} us "
              f"({fl / tf / 1e6:7.1f} TF, {kname})   im2col+gemm {t2:8.1f} us", flush=True)
