import sys, cProfile, pstats, io, time
sys.path.insert(0, ".")
import torch
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.routines.netlib import pinned_empty
S = 8192
prec = tb.Precision.H
ctx = tb.context_create(tb.host_device())
a, b, c = (pinned_empty(S * S, prec) for _ in range(3))
L, T = tb.Layout.ROW_MAJOR, tb.Transpose.NO
for _ in range(3):
    tb.netlib_call("hgemm", L, T, T, S, S, S, 1.0, a, b, 0.0, c, ctx=ctx)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    tb.netlib_call("hgemm", L, T, T, S, S, S, 1.0, a, b, 0.0, c, ctx=ctx)
pr.disable()
s = io.StringIO()
st = pstats.Stats(pr, stream=s).sort_stats("tottime")
st.print_stats(25)
print(s.getvalue()[:6000])
