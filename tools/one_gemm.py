"""One HGEMM S^3 row-major NN call on a given CTA-pair tile (for ncu).
usage: python tools/one_gemm.py S NWG [GROUP_M] [calls]   (NWG 0 = built-in route)"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.kernels.dispatch import gemm_native  # noqa: E402

S, nwg = int(sys.argv[1]), int(sys.argv[2])
gm = int(sys.argv[3]) if len(sys.argv) > 3 else 8
calls = int(sys.argv[4]) if len(sys.argv) > 4 else 3
ctx = tb.context_create(tb.host_device())
prec = tb.Precision.H
a = tb.buffer_from_tensor(ctx, prec, (torch.rand(S * S, device="cuda") * 2 - 1).half())
b = tb.buffer_from_tensor(ctx, prec, (torch.rand(S * S, device="cuda") * 2 - 1).half())
c = tb.buffer_alloc(ctx, prec, S * S)
cfg = None if nwg == 0 else tb.Configuration.make(
    "gemm_b200", dict(zip(("MWG", "NWG", "KWG", "STAGES", "CTA_GROUP", "SPLIT_K", "GROUP_M"),
                          (256, nwg, 64, 0, 2, 1, gm))))
for _ in range(calls):
    rec = gemm_native(ctx, prec, tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.NO, S, S, S, 1.0, a, 0, S,
                      b, 0, S, 0.0, c, 0, S, cfg, 0)
torch.cuda.synchronize()
print(rec["kernel"])
