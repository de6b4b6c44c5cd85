"""Kernel / copy timeline of one netlib_call HGEMM 8192^3 on pinned host
arrays (the bench's e2e step), from the torch profiler.  Dev tool."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.routines.netlib import pinned_empty  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
prec = tb.Precision.H
ctx = tb.context_create(tb.host_device())
a, b, c = (pinned_empty(S * S, prec) for _ in range(3))
a[:] = 0.5
b[:] = 0.25
L, T = tb.Layout.ROW_MAJOR, tb.Transpose.NO
for _ in range(3):
    tb.netlib_call("hgemm", L, T, T, S, S, S, 1.0, a, b, 0.0, c, ctx=ctx)
torch.cuda.synchronize()
ev = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tb.netlib_call("hgemm", L, T, T, S, S, S, 1.0, a, b, 0.0, c, ctx=ctx)
    e1.record()
    torch.cuda.synchronize()
    ev.append(e0.elapsed_time(e1))
print("ms per call:", [round(x, 3) for x in ev])
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tb.netlib_call("hgemm", L, T, T, S, S, S, 1.0, a, b, 0.0, c, ctx=ctx)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in evs)
for e in sorted(evs, key=lambda e: e.time_range.start):
    s, f = e.time_range.start - t0, e.time_range.end - t0
    print(f"{s:9.1f} {f:9.1f} {f - s:8.1f} {e.name[:60]}")
