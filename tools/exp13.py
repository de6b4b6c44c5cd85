"""One launch of each C4 batched workload (16384 x 32^3 / 64^3, H and S, row-major NN)."""
import sys, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
ctx = tb.context_create(tb.host_device())
T = tb.Transpose
which = sys.argv[1:] or ["H32", "H64", "S32", "S64"]
for w in which:
    prec = tb.Precision.H if w[0] == "H" else tb.Precision.S
    d = int(w[1:]); B = 16384
    dt = prec.torch_dtype
    a = tb.buffer_from_tensor(ctx, prec, (torch.rand(B*d*d, device='cuda')*2-1).to(dt))
    b = tb.buffer_from_tensor(ctx, prec, (torch.rand(B*d*d, device='cuda')*2-1).to(dt))
    c = tb.buffer_alloc(ctx, prec, B*d*d)
    for _ in range(int(__import__("os").environ.get("REPS", "2"))):
        tb.gemm_strided_batched(ctx, tb.Layout.ROW_MAJOR, T.NO, T.NO, d, d, d, 1.0, a, d*d, b, d*d, 0.0, c, d*d, B)
    torch.cuda.synchronize()
    print(w, ctx.last_launch.native["kernel"], flush=True)
