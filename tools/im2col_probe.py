"""im2col probe (dev tool): the bench's ResNet-style layer, H and S, a few calls."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_05249_b200 as tb  # noqa: E402
ctx = tb.context_create(tb.host_device())
c, h, w, kh, kw = 256, 56, 56, 3, 3
for prec in (tb.Precision.H, tb.Precision.S):
    im = tb.buffer_from_tensor(ctx, prec, torch.rand(c * h * w, device="cuda").to(prec.torch_dtype))
    col = tb.buffer_alloc(ctx, prec, c * kh * kw * h * w)
    for _ in range(3):
        tb.im2col(ctx, c, h, w, kh, kw, 1, 1, 1, 1, 1, 1, im, col)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(50):
        tb.im2col(ctx, c, h, w, kh, kw, 1, 1, 1, 1, 1, 1, im, col)
    e1.record(); torch.cuda.synchronize()
    print(prec.value, f"{e0.elapsed_time(e1) / 50 * 1e3:.2f} us/call (L2-warm, back-to-back)", ctx.last_launch.native["kernel"])
