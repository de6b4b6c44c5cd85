"""Device-time chosen shapes under the built-in route and forced gemm_b200
configurations, L2 flushed before every call (the bench's protocol).

    python tools/route_probe.py H 4096 128 9216 [--cfg MWG,NWG,KWG,STAGES,CTA_GROUP,SPLIT_K,GROUP_M ...]
"""
import argparse
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("prec")
ap.add_argument("m", type=int)
ap.add_argument("n", type=int)
ap.add_argument("k", type=int)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--cfg", nargs="*", default=[])
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
prec = tb.Precision.H if args.prec == "H" else tb.Precision.S
ctx = tb.context_create(tb.host_device())
m, n, k, batch = args.m, args.n, args.k, args.batch
dev = ctx.torch_device
a = tb.buffer_from_tensor(ctx, prec, (torch.rand(m * k * batch, device=dev) * 2 - 1).to(prec.torch_dtype))
b = tb.buffer_from_tensor(ctx, prec, (torch.rand(k * n * batch, device=dev) * 2 - 1).to(prec.torch_dtype))
c = tb.buffer_alloc(ctx, prec, m * n * batch)
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
clean = torch.ones(256 << 20, dtype=torch.uint8, device=dev)
store = tb.routines.common.get_store(ctx)
L, T = tb.Layout.ROW_MAJOR, tb.Transpose.NO
names = ("MWG", "NWG", "KWG", "STAGES", "CTA_GROUP", "SPLIT_K", "GROUP_M")


def call():
    if batch == 1:
        tb.gemm(ctx, L, T, T, m, n, k, 1.0, a, b, 0.0, c)
    else:
        tb.gemm_strided_batched(ctx, L, T, T, m, n, k, 1.0, a, m * k, b, k * n, 0.0, c, m * n, batch)


def timeit():
    for _ in range(3):
        call()
    ts = []
    for _ in range(args.reps):
        flush_buf.fill_(1)
        clean.view(torch.int64).sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ts)
    return v[len(v) // 2], v[0]


for spec in ["auto"] + args.cfg:
    store.clear_overrides()
    if spec != "auto":
        vals = [int(x) for x in spec.split(",")]
        store.set_override("gemm_b200", prec, ctx.device, (m, n, k),
                           tb.Configuration.make("gemm_b200", dict(zip(names, vals))))
    med, best = timeit()
    fl = 2.0 * m * n * k * batch
    by = (m * k + k * n + m * n) * batch * (2 if prec is tb.Precision.H else 4)
    print(f"{spec:28s} {ctx.last_launch.native['kernel']:44s} median {med:8.2f} us  min {best:8.2f} us  "
          f"{fl / med / 1e6:8.1f} TF  {by / med / 1e3:7.1f} GB/s", flush=True)
