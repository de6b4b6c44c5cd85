"""Route audit (dev tool): for a grid of shapes, device-time the built-in
route and every instantiated gemm_b200 variant (bench protocol: L2 flushed,
CUDA events, median of a few runs) and print where the built-in route is
more than 5 % slower than the best variant.

    python tools/route_audit.py [H|S] [--set2] [--trans=nt|tn|tt] [--batched] [--shapes=MxNxK,...]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.kernels.dispatch import gemm_native  # noqa: E402
from paper_1705_05249_b200.kernels.params import b200_variants  # noqa: E402

ctx = tb.context_create(tb.host_device())
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
names = ("MWG", "NWG", "KWG", "STAGES", "CTA_GROUP", "SPLIT_K", "GROUP_M")
precs = [a for a in sys.argv[1:] if a in ("H", "S")] or ["H", "S"]
SET2 = "--set2" in sys.argv
TRANS = next((a[len("--trans="):] for a in sys.argv if a.startswith("--trans=")), "nn")
BATCHED = "--batched" in sys.argv


def timed(fn, reps):
    fn()
    ev = []
    for _ in range(reps):
        flush_buf.fill_(1)
        clean.view(torch.int64).sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rec = fn()
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return v[len(v) // 2], rec["kernel"]


SHAPES = [(256, 256, 256), (512, 512, 512), (768, 768, 768), (1024, 1024, 1024), (1536, 1536, 1536),
          (2048, 2048, 2048), (3072, 3072, 3072), (4096, 4096, 4096),
          (1024, 1024, 8192), (2048, 2048, 8192), (512, 512, 16384), (8192, 256, 1024),
          (256, 8192, 1024), (4096, 512, 4096), (512, 4096, 4096), (16384, 64, 2048),
          (2048, 512, 512), (3000, 2000, 1000)]
if SET2:
    SHAPES = [(1000, 1000, 1000), (4000, 1000, 500), (100, 10000, 1000), (6000, 300, 3000), (128, 128, 65536),
              (8192, 8192, 256), (256, 256, 32768), (12288, 1024, 1024), (1024, 12288, 1024), (2500, 2500, 2500),
              (5000, 5000, 500), (640, 640, 8192), (96, 4096, 4096), (4096, 96, 4096), (1500, 700, 3000)]
CUSTOM = next((a[len("--shapes="):] for a in sys.argv if a.startswith("--shapes=")), None)
if CUSTOM:  # --shapes=MxNxK,MxNxK (no size cap)
    SHAPES = [tuple(int(v) for v in x.split("x")) for x in CUSTOM.split(",")]
if BATCHED:
    from paper_1705_05249_b200.kernels.dispatch import gemm_strided_batched_native  # noqa: E402
    for p in precs:
        prec = tb.Precision.H if p == "H" else tb.Precision.S
        for (s_, batch) in ((16, 65536), (48, 8192), (96, 2048), (128, 1024), (200, 256), (256, 256), (384, 64)):
            e = s_ * s_
            a = tb.buffer_from_tensor(ctx, prec, (torch.rand(e * batch, device="cuda") * 2 - 1).to(prec.torch_dtype))
            b = tb.buffer_from_tensor(ctx, prec, (torch.rand(e * batch, device="cuda") * 2 - 1).to(prec.torch_dtype))
            c = tb.buffer_alloc(ctx, prec, e * batch)

            def run(cfg):
                return lambda: gemm_strided_batched_native(ctx, prec, tb.Layout.ROW_MAJOR, tb.Transpose.NO,
                                                           tb.Transpose.NO, s_, s_, s_, 1.0, a, 0, s_, e, b, 0, s_, e,
                                                           0.0, c, 0, s_, e, batch, cfg, 0)
            auto_us, auto_k = timed(run(None), 7)
            best = (auto_us, auto_k, "auto")
            for v in b200_variants(prec):
                cfg = tb.Configuration.make("gemm_b200", dict(zip(names, v + (0,))))
                try:
                    us, kern = timed(run(cfg), 7)
                except Exception:  # noqa: BLE001
                    continue
                if us < best[0]:
                    best = (us, kern, v)
            flag = "  <== " if best[0] < 0.95 * auto_us else ""
            print(f"{p} {s_}^3 x {batch}: auto {auto_us:9.2f} us {auto_k:40s} best {best[0]:9.2f} us {best[1]:40s}"
                  f" {best[2]}{flag}", flush=True)
    sys.exit(0)
for p in precs:
    prec = tb.Precision.H if p == "H" else tb.Precision.S
    for (m, n, k) in SHAPES:
        if prec is tb.Precision.S and m * n * k > 2 ** 35 and not CUSTOM:
            continue
        a = tb.buffer_from_tensor(ctx, prec, (torch.rand(m * k, device="cuda") * 2 - 1).to(prec.torch_dtype))
        b = tb.buffer_from_tensor(ctx, prec, (torch.rand(k * n, device="cuda") * 2 - 1).to(prec.torch_dtype))
        ta = tb.Transpose.YES if TRANS[0] == "t" else tb.Transpose.NO
        tbt = tb.Transpose.YES if TRANS[1] == "t" else tb.Transpose.NO
        lda = m if TRANS[0] == "t" else k
        ldb = k if TRANS[1] == "t" else n
        c = tb.buffer_alloc(ctx, prec, m * n)
        reps = 5 if m * n * k > 2 ** 33 else 9

        def run(cfg):
            return lambda: gemm_native(ctx, prec, tb.Layout.ROW_MAJOR, ta, tbt, m, n, k,
                                       1.0, a, 0, lda, b, 0, ldb, 0.0, c, 0, n, cfg, 0)
        auto_us, auto_k = timed(run(None), reps)
        best = (auto_us, auto_k, "auto")
        for v in b200_variants(prec):
            cfg = tb.Configuration.make("gemm_b200", dict(zip(names, v + (0,))))
            try:
                us, kern = timed(run(cfg), reps)
            except Exception as e:  # noqa: BLE001
                continue
            if us < best[0]:
                best = (us, kern, v)
        flag = "  <== " if best[0] < 0.95 * auto_us else ""
        print(f"{p} {m}x{n}x{k}: auto {auto_us:9.2f} us {auto_k:40s} best {best[0]:9.2f} us {best[1]:40s}"
              f" {best[2]}{flag}", flush=True)
