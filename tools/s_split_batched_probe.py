import sys; sys.path.insert(0, ".")
import torch
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.kernels.dispatch import gemm_strided_batched_native
ctx = tb.context_create(tb.host_device())
S = tb.Precision.S
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
names = ("MWG", "NWG", "KWG", "STAGES", "CTA_GROUP", "SPLIT_K", "GROUP_M")
split = tb.Configuration.make("gemm_b200", dict(zip(names, (64, 32, 32, 0, 1, 2, 0))))
for (m, n, k, batch) in ((512, 512, 640, 64), (256, 256, 768, 256), (256, 512, 640, 128), (128, 1024, 768, 64), (512, 512, 512, 32)):
    a = tb.buffer_from_tensor(ctx, S, torch.rand(m * k * batch, device="cuda") * 2 - 1)
    b = tb.buffer_from_tensor(ctx, S, torch.rand(k * n * batch, device="cuda") * 2 - 1)
    c = tb.buffer_alloc(ctx, S, m * n * batch)
    res = {}
    for _ in range(15):
        for name, cfg in (("route", None), ("split2", split)):
            flush.fill_(1); clean.view(torch.int64).sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = gemm_strided_batched_native(ctx, S, tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.NO, m, n, k, 1.0,
                                            a, 0, k, m * k, b, 0, n, k * n, 0.0, c, 0, n, m * n, batch, cfg, 0)
            e1.record(); e1.synchronize()
            res.setdefault(name, []).append(e0.elapsed_time(e1) * 1e3); res[name + "_k"] = r["kernel"]
    out = []
    for name in ("route", "split2"):
        v = sorted(res[name]); out.append(f"{name} {v[len(v)//2]:8.1f} us {res[name + '_k']}")
    print(f"{m}x{n}x{k} x{batch}: " + " | ".join(out), flush=True)
