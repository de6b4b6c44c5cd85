"""HGEMM 8192^3 pair-kernel variants (raster group height, wave barrier),
bench protocol (L2 flushed, events).  Dev tool."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.kernels import native  # noqa: E402
from paper_1705_05249_b200.kernels.dispatch import gemm_native  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ctx = tb.context_create(tb.host_device())
prec = tb.Precision.H
a = tb.buffer_from_tensor(ctx, prec, (torch.rand(S * S, device="cuda") * 2 - 1).half())
b = tb.buffer_from_tensor(ctx, prec, (torch.rand(S * S, device="cuda") * 2 - 1).half())
c = tb.buffer_alloc(ctx, prec, S * S)
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
names = ("MWG", "NWG", "KWG", "STAGES", "CTA_GROUP", "SPLIT_K", "GROUP_M")


def run(cfg, flags):
    return gemm_native(ctx, prec, tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.NO, S, S, S, 1.0, a, 0, S,
                       b, 0, S, 0.0, c, 0, S, cfg, flags)


def t(cfg, flags, reps=15):
    for _ in range(3):
        run(cfg, flags)
    ev = []
    for _ in range(reps):
        flush_buf.fill_(1)
        clean.view(torch.int64).sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rec = run(cfg, flags)
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(x.elapsed_time(y) * 1e3 for x, y in ev)
    return v[len(v) // 2], rec["kernel"]


order = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 4, 8, 16, 32]
wss = (0,) if len(sys.argv) > 3 else (0, native.FLAG_WAVE_SYNC)
for gm in order:
    for ws in wss:
        cfg = None if gm == 0 else tb.Configuration.make("gemm_b200", dict(zip(names, (256, 256, 64, 0, 2, 1, gm))))
        us, k = t(cfg, ws)
        print(f"group_m {gm:2d} wave_sync {bool(ws):d}: {us:8.1f} us  {2 * S ** 3 / us / 1e6:7.1f} TF  {k}", flush=True)
