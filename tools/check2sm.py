import sys, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.kernels import native
from paper_1705_05249_b200.kernels.dispatch import gemm_native
ctx = tb.context_create(tb.host_device())
T = tb.Transpose
cfg = tb.routines.common.get_store(ctx).resolve("gemm", tb.Precision.H, ctx.device, (1, 1, 1))[0]
fails = 0
for (m, n, k) in ((4096, 4096, 512), (4000, 4100, 333), (2560, 8192, 1024), (8192, 8192, 8192)):
    for lay in (tb.Layout.ROW_MAJOR, tb.Layout.COL_MAJOR):
        for ta in (T.NO, T.YES):
            for tbt in (T.NO, T.YES):
                if (m, n, k) == (8192, 8192, 8192) and (ta, tbt) != (T.NO, T.NO):
                    continue
                a = tb.buffer_from_tensor(ctx, tb.Precision.H, (torch.rand(m * k, device='cuda') * 2 - 1).half())
                b = tb.buffer_from_tensor(ctx, tb.Precision.H, (torch.rand(k * n, device='cuda') * 2 - 1).half())
                rows = (m, k) if ta is T.NO else (k, m)
                lda = rows[0] if lay is tb.Layout.COL_MAJOR else rows[1]
                rows = (k, n) if tbt is T.NO else (n, k)
                ldb = rows[0] if lay is tb.Layout.COL_MAJOR else rows[1]
                ldc = m if lay is tb.Layout.COL_MAJOR else n
                outs = []
                for flags in (0, native.FLAG_NO_2SM):
                    c = tb.buffer_alloc(ctx, tb.Precision.H, m * n)
                    rec = gemm_native(ctx, tb.Precision.H, lay, ta, tbt, m, n, k, 1.0, a, 0, lda, b, 0, ldb, 0.0, c, 0, ldc, cfg, flags)
                    torch.cuda.synchronize()
                    outs.append((rec["kernel"], c.device_tensor().clone()))
                # reference via torch fp32
                A = a.device_tensor().float().view(*((m, k) if ta is T.NO else (k, m))) if lay is tb.Layout.ROW_MAJOR else a.device_tensor().float().view(*(((k, m) if ta is T.NO else (m, k))))
                same = torch.equal(outs[0][1], outs[1][1])
                diff = (outs[0][1].float() - outs[1][1].float()).abs().max().item()
                ok = same
                fails += not ok
                print(("OK  " if ok else "BAD ") + f"{m}x{n}x{k} {lay.value} {ta.value}{tbt.value} {outs[0][0]} vs {outs[1][0]} bitwise={same} maxdiff={diff:.3e}", flush=True)
print("FAILS", fails)
