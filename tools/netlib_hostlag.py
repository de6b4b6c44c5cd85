import sys, time
sys.path.insert(0, ".")
import torch
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.routines import netlib
from paper_1705_05249_b200.routines.netlib import pinned_empty
S = 8192
prec = tb.Precision.H
ctx = tb.context_create(tb.host_device())
a, b, c = (pinned_empty(S * S, prec) for _ in range(3))
L, T = tb.Layout.ROW_MAJOR, tb.Transpose.NO
log = []
def wrap(obj, name):
    f = getattr(obj, name)
    def g(*args, **kw):
        t0 = time.perf_counter(); r = f(*args, **kw); log.append((name, t0, time.perf_counter())); return r
    setattr(obj, name, g)
wrap(netlib.level3, "gemm"); wrap(netlib._Transfer, "upload"); wrap(netlib._Transfer, "download")
for _ in range(3):
    tb.netlib_call("hgemm", L, T, T, S, S, S, 1.0, a, b, 0.0, c, ctx=ctx)
torch.cuda.synchronize()
log.clear()
T0 = time.perf_counter()
tb.netlib_call("hgemm", L, T, T, S, S, S, 1.0, a, b, 0.0, c, ctx=ctx)
T1 = time.perf_counter()
for n, s, e in log:
    print(f"{n:9s} {1e6*(s-T0):9.1f} {1e6*(e-T0):9.1f} {1e6*(e-s):8.1f}")
print("total", 1e6*(T1-T0))
