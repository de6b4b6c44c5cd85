"""HGEMM CTA-pair tile 256x256 against 256x512, interleaved, bench protocol
(L2 flushed, events), plus a bitwise check between the two.  Dev tool.
usage: python tools/pair512_probe.py [S | MxNxK ...]"""
import os
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.kernels import native  # noqa: E402
from paper_1705_05249_b200.kernels.dispatch import gemm_native  # noqa: E402

names = ("MWG", "NWG", "KWG", "STAGES", "CTA_GROUP", "SPLIT_K", "GROUP_M")
ctx = tb.context_create(tb.host_device())
prec = tb.Precision.H
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
sizes = [tuple(int(v) for v in x.split("x")) if "x" in x else (int(x),) * 3 for x in sys.argv[1:]] or [(8192,) * 3]
cfgs = {"route": None, "256x256 g8": (256, 256, 64, 0, 2, 1, 8),
        "256x512 g8": (256, 512, 64, 0, 2, 1, 8)}
if os.environ.get("PAIR_WS"):  # 256x512 g16 with and without the wave barrier
    cfgs = {"256x512 g16": (256, 512, 64, 0, 2, 1, 16), "256x512 g16 ws": (256, 512, 64, 0, 2, 1, 16, "ws")}
if os.environ.get("PAIR_GROUPS"):  # 256x512 raster group heights instead
    cfgs = {f"256x512 g{g}": (256, 512, 64, 0, 2, 1, int(g)) for g in os.environ["PAIR_GROUPS"].split(",")}
for (M, N, K) in sizes:
    S = f"{M}x{N}x{K}"
    a = tb.buffer_from_tensor(ctx, prec, (torch.rand(M * K, device="cuda") * 2 - 1).half())
    b = tb.buffer_from_tensor(ctx, prec, (torch.rand(K * N, device="cuda") * 2 - 1).half())
    c = tb.buffer_alloc(ctx, prec, M * N)

    def run(cfg):
        flags = native.FLAG_WAVE_SYNC if cfg is not None and cfg[-1] == "ws" else 0
        conf = None if cfg is None else tb.Configuration.make("gemm_b200", dict(zip(names, cfg[:7])))
        return gemm_native(ctx, prec, tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.NO, M, N, K, 1.0, a, 0, K,
                           b, 0, N, 0.0, c, 0, N, conf, flags)

    outs = {}
    for name, cfg in cfgs.items():
        run(cfg)
        torch.cuda.synchronize()
        outs[name] = c.device_tensor().clone()
    ref = next(iter(outs.values()))
    for name, o in outs.items():
        print(f"S={S} {name:12s} bitwise-equal-to-256x256: {torch.equal(o, ref)}", flush=True)
    del outs
    reps = 20 if M * N * K <= 8192 ** 3 else 8
    res = {n: [] for n in cfgs}
    blocks = {n: [] for n in cfgs}
    kern = {}
    names_ = list(cfgs)
    for _round in range(int(os.environ.get("ROUNDS", "8"))):  # bench-protocol blocks (3 warm-up + reps timed), ABBA order
        order = names_ if _round % 2 == 0 else names_[::-1]
        for name in order:
            cfg = cfgs[name]
            time.sleep(3)  # each block starts from an idle GPU, as the driver's bench run does
            for _ in range(3):
                run(cfg)
            ev = []
            for _ in range(reps):
                flush_buf.fill_(1)
                clean.view(torch.int64).sum()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rec = run(cfg)
                e1.record()
                ev.append((e0, e1))
            torch.cuda.synchronize()
            v = sorted(x.elapsed_time(y) * 1e3 for x, y in ev)
            res[name] += v
            blocks[name].append(round(v[len(v) // 2], 1))
            kern[name] = rec["kernel"]
    for name in cfgs:
        print(f"S={S} {name:12s} block medians {blocks[name]}", flush=True)
    for name, v in res.items():
        v.sort()
        med = v[len(v) // 2]
        print(f"S={S} {name:12s} median {med:10.1f} us  min {v[0]:10.1f}  {2 * M * N * K / med / 1e6:7.1f} TF  {kern[name]}",
              flush=True)
