#!/usr/bin/env python3
"""Driver benchmark: GEMM GFLOPS of the B200-native hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload hgemm|sgemm|batched_h32|batched_s32|batched_h64|batched_s64|
                                sgemm_c1|hgemm_c3|sgemm_c3|hgemm_c3b|sgemm_c3b|hgemm_c5|sgemm_c5]
                    [--replicate-c] [--chunks C] [--no-extra] [--no-cpu-baseline]
                    [--sweep-out PATH]

A "step" is one call of the hot path on one batch of synthetic input:
* hgemm (default, the headline): C = A·B, 8192^3, FP16 storage / FP32
  accumulate, row-major NN, alpha=1, beta=0 (BASELINE configs[1], largest
  square size of the sweep);
* sgemm: the same shape in FP32 (FFMA);
* batched_*: gemm_strided_batched, 16384 instances of 32^3 / 64^3 (configs[3]);
* sgemm_c1: 1024^3 (configs[0]); *_c3 / *_c3b: (4096,128,9216) / (64,3136,576)
  (configs[2]); *_c5: 32768^3 (configs[4]).

value   = whole-job GFLOPS with inputs resident in HBM, CUDA-event timed per
          step on the launching stream (max over ranks), L2 flushed between
          steps (256 MiB write + 256 MiB read) so no step reads a warm L2.
e2e     = the same metric through the public API with HOST buffers: pinned
          host → device copy of A and B, the routine, device → host copy of C,
          all inside the timed region.
N > 1   = every rank runs the library's sharding (paper_1705_05249_b200/
          distributed.py) one process per GPU over NCCL:
          * gemm workloads: weak scaling — rank r computes its M-block (row-major
            C) of an (m·N) x n x k GEMM through ``gemm_sharded``;
          * *_c5: strong scaling — the fixed 32768^3 GEMM split into N row
            blocks through ``gemm_sharded``;
          * batched: weak scaling — N·16384 instances, rank r its contiguous
            16384 through ``gemm_strided_batched_sharded``;
          * --replicate-c adds the replication of C to every rank inside the
            timed step (--chunks C > 1: overlapped per-sub-block transfers).
--impl reference times the reference's CPU implementation of the path (the
oracle port of tunedblas' tiled algorithm, oracle/gemm_oracle.py) on the
host cores, each step a bounded row-block sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GEMM GFLOPS (SGEMM/HGEMM, batched) and % of B200 peak at 1/2/4/8 GPUs"
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
FFMA_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # derived FP32 FFMA peak at sm_max_mhz


def load_peaks():
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        with open(path) as fh:
            doc = json.load(fh)
        return doc, "measured"
    return dict(FALLBACK), "fallback"


WORKLOADS = {
    "hgemm": dict(kind="gemm", prec="H", m=8192, n=8192, k=8192, batch=1),
    "sgemm": dict(kind="gemm", prec="S", m=8192, n=8192, k=8192, batch=1),
    "batched_h32": dict(kind="batched", prec="H", m=32, n=32, k=32, batch=16384),
    "batched_s32": dict(kind="batched", prec="S", m=32, n=32, k=32, batch=16384),
    "batched_h64": dict(kind="batched", prec="H", m=64, n=64, k=64, batch=16384),
    "batched_s64": dict(kind="batched", prec="S", m=64, n=64, k=64, batch=16384),
    # the other BASELINE shapes: C1 (the reference's canonical 1024^3 SGEMM)
    # and C3 (the im2col'd DL layer (4096, 128, 9216))
    "sgemm_c1": dict(kind="gemm", prec="S", m=1024, n=1024, k=1024, batch=1),
    "hgemm_c3": dict(kind="gemm", prec="H", m=4096, n=128, k=9216, batch=1),
    "sgemm_c3": dict(kind="gemm", prec="S", m=4096, n=128, k=9216, batch=1),
    # C3's other im2col'd layer (64, 3136, 576)
    "hgemm_c3b": dict(kind="gemm", prec="H", m=64, n=3136, k=576, batch=1),
    "sgemm_c3b": dict(kind="gemm", prec="S", m=64, n=3136, k=576, batch=1),
    # C5: the large GEMM (under torchrun: strong scaling, the fixed problem
    # split into N row blocks)
    "hgemm_c5": dict(kind="gemm", prec="H", m=32768, n=32768, k=32768, batch=1),
    "sgemm_c5": dict(kind="gemm", prec="S", m=32768, n=32768, k=32768, batch=1),
}


def describe(w: dict) -> str:
    p = "HGEMM FP16 (FP32 accumulate)" if w["prec"] == "H" else "SGEMM FP32 (FFMA)"
    if w["kind"] == "gemm":
        return f"{p} {w['m']}x{w['n']}x{w['k']} row-major NN alpha=1 beta=0"
    return f"{p} strided batched {w['batch']} x {w['m']}^3 row-major NN alpha=1 beta=0"


def flops(w: dict) -> float:
    return 2.0 * w["m"] * w["n"] * w["k"] * w["batch"]


def alg_bytes(w: dict) -> float:
    es = 2 if w["prec"] == "H" else 4
    return (w["m"] * w["k"] + w["k"] * w["n"] + w["m"] * w["n"]) * es * w["batch"]


# ---------------------------------------------------------------------------
# clocks during the timed region (pynvml poller)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.002):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self.ok = False
        self.period = period_s
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.ok = False
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": float(s[len(s) // 2]), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def is_strong(name: str) -> bool:
    """C5 is strong-scaled (the fixed 32768^3 problem split over the ranks);
    every other workload is weak-scaled (per-rank work fixed)."""
    return name.endswith("_c5")


def shard_of(w: dict, name: str, world: int, rank: int) -> dict:
    """The whole job's problem and this rank's share of it: row blocks of a
    row-major C for gemm (distributed.plan_gemm_shards), contiguous instance
    blocks for batched (distributed.gemm_strided_batched_sharded)."""
    from paper_1705_05249_b200.distributed import shard_range

    if w["kind"] == "gemm":
        M = w["m"] if is_strong(name) else w["m"] * world
        s0, cnt = shard_range(M, world, rank)
        return dict(M=M, batch=1, s0=s0, cnt=cnt)
    total = w["batch"] * world
    s0, cnt = shard_range(total, world, rank)
    return dict(M=w["m"], batch=total, s0=s0, cnt=cnt)


def job_flops(w: dict, sh: dict) -> float:
    if w["kind"] == "gemm":
        return 2.0 * sh["M"] * w["n"] * w["k"]
    return 2.0 * w["m"] * w["n"] * w["k"] * sh["batch"]


def rank_flops(w: dict, sh: dict) -> float:
    if w["kind"] == "gemm":
        return 2.0 * sh["cnt"] * w["n"] * w["k"]
    return 2.0 * w["m"] * w["n"] * w["k"] * sh["cnt"]


def rank_bytes(w: dict, sh: dict) -> float:
    es = 2 if w["prec"] == "H" else 4
    if w["kind"] == "gemm":
        return (sh["cnt"] * w["k"] + w["k"] * w["n"] + sh["cnt"] * w["n"]) * es
    return (w["m"] * w["k"] + w["k"] * w["n"] + w["m"] * w["n"]) * es * sh["cnt"]


def make_operands(tb, ctx, w, sh, torch):
    """Whole-job buffers; only this rank's rows / instances (and, for gemm,
    the replicated B) are filled: U(-1, 1), seeded per rank."""
    prec = tb.Precision.H if w["prec"] == "H" else tb.Precision.S
    dt = prec.torch_dtype
    dev = ctx.torch_device
    g = torch.Generator(device=dev).manual_seed(12345 + sh["s0"])
    if w["kind"] == "gemm":
        m_all, n, k = sh["M"], w["n"], w["k"]
        na, nb, nc = m_all * k, k * n, m_all * n
        a_lo, a_hi = sh["s0"] * k, (sh["s0"] + sh["cnt"]) * k
        b_lo, b_hi = 0, nb
    else:
        e = w["m"] * w["k"]
        na = nb = nc = e * sh["batch"]
        a_lo, a_hi = sh["s0"] * e, (sh["s0"] + sh["cnt"]) * e
        b_lo, b_hi = a_lo, a_hi
    at = torch.zeros(na, device=dev, dtype=dt)
    bt = torch.zeros(nb, device=dev, dtype=dt)
    at[a_lo:a_hi] = (torch.rand(a_hi - a_lo, device=dev, generator=g) * 2 - 1).to(dt)
    bt[b_lo:b_hi] = (torch.rand(b_hi - b_lo, device=dev, generator=g) * 2 - 1).to(dt)
    ct = torch.zeros(nc, device=dev, dtype=dt)
    return prec, tb.buffer_from_tensor(ctx, prec, at), tb.buffer_from_tensor(ctx, prec, bt), \
        tb.buffer_from_tensor(ctx, prec, ct)


def step_fn(tb, ctx, w, sh, a, b, c, rank, world, replicate_c=False, chunks=1):
    """One step = this rank's share through the library's sharding (a plain
    gemm / gemm_strided_batched call at N = 1)."""
    from paper_1705_05249_b200 import distributed as D

    L, T = tb.Layout.ROW_MAJOR, tb.Transpose.NO
    if w["kind"] == "gemm":
        M, n, k = sh["M"], w["n"], w["k"]
        return lambda: D.gemm_sharded(ctx, L, T, T, M, n, k, 1.0, a, b, 0.0, c, rank=rank, world=world,
                                      replicate_c=replicate_c, chunks=chunks)
    s, e, total = w["m"], w["m"] * w["m"], sh["batch"]
    return lambda: D.gemm_strided_batched_sharded(ctx, L, T, T, s, s, s, 1.0, a, e, b, e, 0.0, c, e, total,
                                                  rank=rank, world=world, replicate_c=replicate_c,
                                                  chunks=chunks)


def device_time(fn, steps, warmup, stream, torch, flush):
    """Per-step CUDA-event times (s) on `stream`, L2 flushed before each step."""
    for _ in range(warmup):
        flush()
        fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    torch.cuda.synchronize()
    for e0, e1 in evs:
        flush()
        e0.record(stream)
        fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return [e0.elapsed_time(e1) / 1e3 for e0, e1 in evs]


def roofline_of(w, per_launch, peaks, peak_src, sh):
    """Bound, peak and achieved for the dominant kernel of one rank's step."""
    fl, by = rank_flops(w, sh), rank_bytes(w, sh)
    ai = fl / by
    ridge = (peaks["bf16_tflops"] if w["prec"] == "H" else FFMA_TFLOPS) * 1e12 / (peaks["hbm_gbs"] * 1e9)
    if w["kind"] == "gemm" and ai < ridge:
        bound, peak, unit, achieved = "hbm", peaks["hbm_gbs"], "GB/s", by / per_launch / 1e9
        note = (f"HBM copy bandwidth ({peak_src}: MEASURED_PEAKS.json hbm_gbs); "
                f"arithmetic intensity {ai:.0f} flop/B < ridge {ridge:.0f}")
    elif w["prec"] == "H" and w["kind"] == "gemm":
        bound, peak, unit, achieved = "tensor", peaks["bf16_tflops"], "TFLOP/s", fl / per_launch / 1e12
        note = f"dense FP16/BF16 tensor, burst ({peak_src}: MEASURED_PEAKS.json bf16_tflops)"
    elif w["kind"] == "gemm":
        bound, peak, unit, achieved = "ffma", FFMA_TFLOPS, "TFLOP/s", fl / per_launch / 1e12
        note = "FP32 FFMA 148 SM x 128 lanes x 2 x 1.965 GHz (derived, no measured FFMA peak)"
    else:
        bound, peak, unit, achieved = "hbm", peaks["hbm_gbs"], "GB/s", by / per_launch / 1e9
        note = f"HBM copy bandwidth ({peak_src}: MEASURED_PEAKS.json hbm_gbs)"
    return {"bound": bound, "achieved": round(achieved, 2), "peak": peak, "unit": unit,
            "frac": round(achieved / peak, 4), "traffic": None, "peak_source": note,
            "per_launch_ms": round(per_launch * 1e3, 4),
            "algorithmic": f"{fl:.4g} FLOP, {by:.4g} B per launch"}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1705_05249_b200 as tb

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = tb.context_create(tb.host_device())
    ctx.device_index = local_rank
    stream = torch.cuda.current_stream(dev)
    # L2 flush before every step: a 256 MiB write evicts the inputs (126 MB
    # L2), then a 256 MiB read of a second buffer evicts the flush's dirty
    # lines, so the timed kernel starts from a cold, clean L2 and does not pay
    # for unrelated write-backs (measured: C3 34.9 -> 30.5 us).
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    clean_buf = torch.ones(256 << 20, dtype=torch.uint8, device=dev)

    def flush():
        flush_buf.fill_(1)
        clean_buf.view(torch.int64).sum()
    peaks, peak_src = load_peaks()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def measure(name, steps, warmup, replicate_c=False, chunks=1):
        w = WORKLOADS[name]
        sh = shard_of(w, name, world, rank)
        prec, a, b, c = make_operands(tb, ctx, w, sh, torch)
        fn = step_fn(tb, ctx, w, sh, a, b, c, rank, world, replicate_c, chunks)
        fn()
        torch.cuda.synchronize()
        kernel = ctx.last_launch.native["kernel"]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler = ClockSampler(local_rank)
        with sampler:
            times = device_time(fn, steps, warmup, stream, torch, flush)
        total = max_over_ranks(sum(times))
        per_launch = sum(times) / steps
        gflops = job_flops(w, sh) * steps / total / 1e9
        roof = roofline_of(w, per_launch, peaks, peak_src, sh)
        roof["kernel"] = kernel
        return dict(name=name, w=w, sh=sh, times=times, total=total, gflops=gflops, kernel=kernel,
                    clocks=sampler.summary(), a=a, b=b, c=c, prec=prec, fn=fn, roofline=roof)

    main = measure(args.workload, args.steps, args.warmup, args.replicate_c, args.chunks)
    w, sh = main["w"], main["sh"]

    # ---- e2e: the library's host-array API (netlib_call) on this rank's share ----
    e2e = e2e_netlib(tb, ctx, w, sh, main, args, stream, torch, max_over_ranks, world)
    del main["a"], main["b"], main["c"], main["fn"]
    torch.cuda.empty_cache()

    # ---- extras: the other headline configs (device-timed, this rank) ----
    extra = {}
    if not args.no_extra:
        for name in WORKLOADS:
            if name == args.workload:
                continue
            try:
                big = WORKLOADS[name]["m"] >= 32768
                r = measure(name, 3 if big else max(5, min(args.steps, 20)),
                            min(args.warmup, 3) if big else args.warmup)
                extra[name] = {"workload": describe(r["w"]), "value": round(r["gflops"], 1),
                               "unit": "GFLOPS", "ms_per_step": round(r["total"] / max(1, len(r["times"])) * 1e3, 4),
                               "roofline": r["roofline"], "clocks": r["clocks"]}
                del r
            except Exception as exc:  # noqa: BLE001
                extra[name] = {"error": repr(exc)}
            torch.cuda.empty_cache()
        try:
            extra["c2_sweep"] = c2_sweep(tb, ctx, stream, torch, flush, peaks, peak_src, args.sweep_out)
        except Exception as exc:  # noqa: BLE001
            extra["c2_sweep"] = {"error": repr(exc)}
        torch.cuda.empty_cache()
        try:
            extra["im2col"] = im2col_extra(tb, ctx, stream, torch, flush, peaks, peak_src)
        except Exception as exc:  # noqa: BLE001
            extra["im2col"] = {"error": repr(exc)}
        torch.cuda.empty_cache()
        # North star: batched small-matrix GEMM >= 10x the naive per-matrix
        # launch loop.  Loop = one public `gemm` call per instance (first 1024
        # instances of the 16384 x 32^3 batch, device-timed), per instance.
        try:
            extra["batched_vs_loop"] = batched_vs_loop(tb, ctx, stream, torch)
        except Exception as exc:  # noqa: BLE001
            extra["batched_vs_loop"] = {"error": repr(exc)}

    if rank != 0:
        return None
    traffic = load_traffic(args.workload, main["kernel"])
    if traffic is not None:
        main["roofline"]["traffic"] = traffic
    summary = {}
    for name, ex in extra.items():
        if isinstance(ex, dict) and isinstance(ex.get("roofline"), dict):
            t = load_traffic(name, ex["roofline"].get("kernel", ""))
            if t is not None:
                ex["roofline"]["traffic"] = t
            summary[name] = [ex["value"], ex["roofline"]["frac"], ex["roofline"]["kernel"]]
    if isinstance(extra.get("c2_sweep"), dict) and "min_frac" in extra["c2_sweep"]:
        summary["c2_sweep"] = {"min_frac": extra["c2_sweep"]["min_frac"],
                               "at_8192": extra["c2_sweep"].get("at_8192")}
    strong = is_strong(args.workload)
    par = ("row-block sharded" if w["kind"] == "gemm" else "batch-sharded") + f" x{world}" + \
        (" via distributed.gemm_sharded" if w["kind"] == "gemm" else " via distributed.gemm_strided_batched_sharded")
    launches = args.steps * (min(args.chunks, max(1, sh["cnt"])) if args.replicate_c and world > 1 else 1)
    line = {
        "metric": METRIC,
        "value": round(main["gflops"], 2),
        "unit": "GFLOPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(main["total"] / args.steps * 1e3, 4),
        "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None,
        "dtype": "f16" if w["prec"] == "H" else "f32",
        "data": "synthetic U(-1,1) operands, seeded, resident in HBM",
        "config": {"workload": describe(w), "m": sh["M"], "n": w["n"], "k": w["k"],
                   "batch": sh["batch"], "per_rank": {"rows" if w["kind"] == "gemm" else "instances": sh["cnt"]},
                   "layout": "row-major", "trans": "NN", "alpha": 1.0, "beta": 0.0,
                   "parallelism": par, "replicate_c": bool(args.replicate_c and world > 1),
                   "chunks": args.chunks,
                   "l2": "flushed before every step (256 MiB write + 256 MiB read of a second buffer: "
                         "inputs evicted, no dirty lines left)"},
        "extra_summary": summary,
        "e2e": e2e,
        "gpu_launches": launches,
        "kernel": main["kernel"],
        "clocks": main["clocks"],
        "roofline": main["roofline"],
        "frac_of_peak": main["roofline"]["frac"],
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(w, seconds_budget=args.cpu_seconds)
    if extra:
        line["extra"] = extra
    return line


def e2e_netlib(tb, ctx, w, sh, main, args, stream, torch, max_over_ranks, world) -> dict:
    """The metric end to end through the library's own host-array API:
    every step is one ``netlib_call`` on this rank's share with host arrays
    in pinned memory (``routines.netlib.pinned_empty``) — H2D of A and B,
    the GEMM, D2H of C, pipelined in sub-blocks inside the call — timed with
    CUDA events on the compute stream around all steps (each call returns
    with its result in host memory)."""
    from paper_1705_05249_b200.routines.netlib import pinned_empty

    prec = main["prec"]
    es = prec.elemsize
    L, T = tb.Layout.ROW_MAJOR, tb.Transpose.NO
    if w["kind"] == "gemm":
        k, n, cnt = w["k"], w["n"], sh["cnt"]
        a0 = sh["s0"] * k
        host_a = pinned_empty(cnt * k, prec)
        host_b = pinned_empty(k * n, prec)
        host_c = pinned_empty(cnt * n, prec)
        host_a[:] = main["a"].device_tensor()[a0:a0 + cnt * k].cpu().numpy()
        host_b[:] = main["b"].device_tensor().cpu().numpy()
        rid = "hgemm" if w["prec"] == "H" else "sgemm"

        def step():
            tb.netlib_call(rid, L, T, T, cnt, n, k, 1.0, host_a, host_b, 0.0, host_c, ctx=ctx)
        fl = 2.0 * cnt * n * k
    else:
        s, e, cnt = w["m"], w["m"] * w["m"], sh["cnt"]
        a0 = sh["s0"] * e
        host_a, host_b, host_c = (pinned_empty(cnt * e, prec) for _ in range(3))
        host_a[:] = main["a"].device_tensor()[a0:a0 + cnt * e].cpu().numpy()
        host_b[:] = main["b"].device_tensor()[a0:a0 + cnt * e].cpu().numpy()
        rid = "hgemm_strided_batched" if w["prec"] == "H" else "sgemm_strided_batched"

        def step():
            tb.netlib_call(rid, L, T, T, s, s, s, 1.0, host_a, e, host_b, e, 0.0, host_c, e, cnt, ctx=ctx)
        fl = 2.0 * s * s * s * cnt
    steps = max(4, min(args.steps, 20))
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    total = max_over_ranks(t0.elapsed_time(t1) / 1e3)
    return {"value": round(fl * world * steps / total / 1e9, 2), "unit": "GFLOPS",
            "h2d_bytes_per_step": (host_a.size + host_b.size) * es, "d2h_bytes_per_step": host_c.size * es,
            "ms_per_step": round(total / steps * 1e3, 4), "steps": steps,
            "path": "netlib_call (the library's host-array API) on pinned host arrays: H2D of A and B, "
                    "GEMM, D2H of C, pipelined in sub-blocks over copy and compute streams inside each call"}


C2_SIZES = (256, 512, 1024, 2048, 4096, 8192)
C2_LAYOUTS = ("NN", "NT", "TN", "TT")


def c2_sweep(tb, ctx, stream, torch, flush, peaks, peak_src, out_path=None, steps=5) -> dict:
    """BASELINE configs[1]: square sizes 256..8192 x {N,T}^2 x S/H, row-major,
    device-timed with an L2 flush per step (the reference's sweep client,
    tb/bench.py:124-129,235-267).  Returns {prec: {layout: {size: [GFLOPS,
    frac, kernel]}}} plus the minimum fraction over the tensor-/FFMA-bound
    points (N >= 1024) and the 8192 values."""
    out = {"sizes": list(C2_SIZES), "layout": "row-major", "steps": steps}
    fracs, at_8192 = [], {}
    T = {"N": tb.Transpose.NO, "T": tb.Transpose.YES}
    for p in ("H", "S"):
        prec = tb.Precision.H if p == "H" else tb.Precision.S
        res = {}
        for lay in C2_LAYOUTS:
            res[lay] = {}
            for N in C2_SIZES:
                dev = ctx.torch_device
                a = tb.buffer_from_tensor(ctx, prec, (torch.rand(N * N, device=dev) * 2 - 1).to(prec.torch_dtype))
                b = tb.buffer_from_tensor(ctx, prec, (torch.rand(N * N, device=dev) * 2 - 1).to(prec.torch_dtype))
                c = tb.buffer_alloc(ctx, prec, N * N)
                fn = lambda: tb.gemm(ctx, tb.Layout.ROW_MAJOR, T[lay[0]], T[lay[1]], N, N, N, 1.0, a, b, 0.0, c)  # noqa: E731
                times = device_time(fn, steps, 2, stream, torch, flush)
                t = sum(times) / len(times)
                w = dict(kind="gemm", prec=p, m=N, n=N, k=N, batch=1)
                roof = roofline_of(w, t, peaks, peak_src, dict(M=N, batch=1, s0=0, cnt=N))
                res[lay][N] = [round(2.0 * N ** 3 / t / 1e9, 1), roof["frac"], ctx.last_launch.native["kernel"]]
                if N >= 1024:
                    fracs.append(roof["frac"])
                if N == 8192:
                    at_8192[f"{p}{lay}"] = res[lay][N][:2]
                del a, b, c
        out[p] = res
    out["min_frac"] = round(min(fracs), 4) if fracs else None
    out["at_8192"] = at_8192
    if out_path:
        with open(out_path, "w") as fh:
            json.dump(out, fh, indent=1)
    return out


def im2col_extra(tb, ctx, stream, torch, flush, peaks, peak_src) -> dict:
    """im2col on a ResNet-style layer: 256 x 56 x 56 image,
    3x3 kernel, pad 1, stride 1 -> 2304 x 3136 column matrix.  HBM-bound:
    algorithmic bytes = image read + column matrix write."""
    c, h, w_, kh, kw = 256, 56, 56, 3, 3
    rows, cols = c * kh * kw, h * w_
    out = {"workload": f"im2col {c}x{h}x{w_} image, {kh}x{kw} kernel, pad 1, stride 1 -> {rows}x{cols}"}
    for prec in (tb.Precision.H, tb.Precision.S):
        dev = ctx.torch_device
        im = tb.buffer_from_tensor(ctx, prec, torch.rand(c * h * w_, device=dev).to(prec.torch_dtype))
        col = tb.buffer_alloc(ctx, prec, rows * cols)
        fn = lambda: tb.im2col(ctx, c, h, w_, kh, kw, 1, 1, 1, 1, 1, 1, im, col)  # noqa: E731
        times = device_time(fn, 20, 3, stream, torch, flush)
        t = sum(times) / len(times)
        nbytes = (c * h * w_ + rows * cols) * prec.elemsize
        gbs = nbytes / t / 1e9
        out[prec.value] = {"us_per_call": round(t * 1e6, 2), "GB/s": round(gbs, 1),
                           "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"],
                                        "unit": "GB/s", "frac": round(gbs / peaks["hbm_gbs"], 4),
                                        "peak_source": f"{peak_src}: MEASURED_PEAKS.json hbm_gbs",
                                        "kernel": ctx.last_launch.native["kernel"]}}
    return out


def batched_vs_loop(tb, ctx, stream, torch, loop_instances: int = 1024) -> dict:
    out = {}
    for prec in (tb.Precision.H, tb.Precision.S):
        w = WORKLOADS["batched_h32" if prec is tb.Precision.H else "batched_s32"]
        _, a, b, c = make_operands(tb, ctx, w, shard_of(w, "", 1, 0), torch)
        s, e, batch = w["m"], w["m"] * w["m"], w["batch"]
        L, T = tb.Layout.ROW_MAJOR, tb.Transpose.NO

        def batched():
            tb.gemm_strided_batched(ctx, L, T, T, s, s, s, 1.0, a, e, b, e, 0.0, c, e, batch)

        def loop():
            for i in range(loop_instances):
                tb.gemm(ctx, L, T, T, s, s, s, 1.0, a, b, 0.0, c, a_offset=i * e, b_offset=i * e,
                        c_offset=i * e)

        t_b = sum(device_time(batched, 10, 3, stream, torch, lambda: None)) / 10
        t_l = sum(device_time(loop, 2, 1, stream, torch, lambda: None)) / 2
        per_inst_loop = t_l / loop_instances
        out[prec.value] = {"batched_ms": round(t_b * 1e3, 4), "loop_ms_per_instance": round(per_inst_loop * 1e3, 5),
                           "speedup": round(per_inst_loop * batch / t_b, 1),
                           "workload": f"{batch} x {s}^3 strided batched vs {loop_instances} single gemm calls"}
    return out


def load_traffic(workload: str, kernel: str):
    """dram bytes per launch from the committed ncu capture of this workload
    (profiles/traffic.json: {workload: {"kernel": name, "bytes": B}}), used
    only when the capture was of the same kernel."""
    path = ROOT / "profiles" / "traffic.json"
    if not path.exists():
        return None
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except (OSError, ValueError):
        return None
    ent = doc.get(workload)
    if isinstance(ent, dict) and ent.get("kernel") == kernel:
        return ent.get("bytes")
    return None


# ---------------------------------------------------------------------------
# CPU: the reference's algorithm (oracle port) on the host cores
# ---------------------------------------------------------------------------
def cpu_sample(w: dict, rows: int | None = None):
    """A bounded sample of the workload: a row block of the same GEMM (same
    K and N), or a prefix of the batch.  Returns (callable, flops)."""
    import numpy as np

    from oracle import gemm_oracle as orc

    dt = np.float16 if w["prec"] == "H" else np.float32
    rng = np.random.default_rng(12345)
    pool = orc.make_pool()
    if w["kind"] == "gemm":
        m = rows or 512
        k, n = w["k"], w["n"]
        a = rng.uniform(-1, 1, m * k).astype(dt)
        b = rng.uniform(-1, 1, k * n).astype(dt)
        c = np.zeros(m * n, dt)

        def run():
            orc.port_gemm(w["prec"], True, False, False, m, n, k, 1.0, a, b, 0.0, c, pool=pool)

        return run, 2.0 * m * n * k, f"row block {m} x {n} x {k} of the {describe(w)}"
    batch = rows or 256
    e = w["m"] * w["k"]
    a = rng.uniform(-1, 1, batch * e).astype(dt)
    b = rng.uniform(-1, 1, batch * e).astype(dt)
    c = np.zeros(batch * e, dt)

    def run():
        orc.port_gemm_strided_batched(w["prec"], True, False, False, w["m"], w["n"], w["k"], 1.0,
                                      a, e, b, e, 0.0, c, e, batch)

    return run, 2.0 * w["m"] * w["n"] * w["k"] * batch, \
        f"first {batch} instances of the {describe(w)} (sequential backend, as the reference's fastest batched mode)"


def prewarm(seconds=3.0):
    import numpy as np

    x = np.ones((512, 512), np.float32)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        x @ x


def cpu_baseline(w: dict, seconds_budget: float = 12.0) -> dict:
    import numpy as np

    prewarm(3.0)
    run, fl, sample = cpu_sample(w)
    run()
    t0 = time.perf_counter()
    run()
    one = time.perf_counter() - t0
    reps = max(1, int(seconds_budget / max(one, 1e-6)))
    reps = min(reps, 50)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    value = fl / float(np.mean(times)) / 1e9
    return {"value": round(value, 3), "unit": "GFLOPS", "cores": os.cpu_count(), "kind": "port",
            "sample": sample + f"; {reps} timed runs after 1 warm-up and a 3 s pre-warm",
            "impl": "oracle/gemm_oracle.py port_gemm (tunedblas tiled algorithm, built-in "
                    "config MWG=NWG=64 KWG=16 KWI=8, ThreadPool of os.cpu_count() workers + OpenBLAS)"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm on the host cores."""
    if rank != 0:
        return None
    import numpy as np

    w = WORKLOADS[args.workload]
    prewarm(3.0)
    run, fl, sample = cpu_sample(w)
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    value = fl / float(np.mean(times)) / 1e9
    return {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(float(np.mean(times)) * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if is_strong(args.workload) else "weak", "vs_baseline": None,
        "dtype": "f16" if w["prec"] == "H" else "f32",
        "data": "synthetic U(-1,1)", "impl": "reference",
        "config": {"workload": describe(w), "sample": sample},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOPS", "cores": os.cpu_count(),
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GFLOPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="hgemm")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--replicate-c", action="store_true",
                    help="N > 1: replicate C on every rank inside the timed step")
    ap.add_argument("--chunks", type=int, default=4,
                    help="with --replicate-c: sub-blocks whose transfers overlap the GEMM (1 = one all-gather)")
    ap.add_argument("--sweep-out", default=None, help="also write the C2 sweep JSON here")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist

            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        line = run_ours(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
