"""Host time of netlib_call's prelude (before the first copy is queued), per
piece.  Dev tool."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.routines import netlib  # noqa: E402

S = 8192
prec = tb.Precision.H
ctx = tb.context_create(tb.host_device())
a, b, c = (netlib.pinned_empty(S * S, prec) for _ in range(3))
L, T = tb.Layout.ROW_MAJOR, tb.Transpose.NO
acc = {}


def wrap(obj, name, label):
    f = getattr(obj, name)

    def g(*args, **kw):
        t0 = time.perf_counter()
        r = f(*args, **kw)
        acc[label] = acc.get(label, 0.0) + time.perf_counter() - t0
        return r
    setattr(obj, name, g)


wrap(netlib, "_is_pinned", "_is_pinned")
wrap(netlib._Transfer, "__init__", "_Transfer.__init__ (incl. _is_pinned)")
wrap(netlib, "_storage", "_storage")
wrap(netlib, "_pipeline", "_pipeline")
wrap(netlib.level3, "gemm", "level3.gemm (validate + 8 launches)")
wrap(netlib, "_gemm_pipelined", "_gemm_pipelined (incl. final sync)")
wrap(netlib.np, "shares_memory", "np.shares_memory")
for _ in range(3):
    tb.netlib_call("hgemm", L, T, T, S, S, S, 1.0, a, b, 0.0, c, ctx=ctx)
torch.cuda.synchronize()
acc.clear()
N = 10
t0 = time.perf_counter()
for _ in range(N):
    tb.netlib_call("hgemm", L, T, T, S, S, S, 1.0, a, b, 0.0, c, ctx=ctx)
tot = time.perf_counter() - t0
print(f"total per call {1e6 * tot / N:.1f} us")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"{1e6 * v / N:10.1f} us  {k}")
