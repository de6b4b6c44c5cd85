#!/usr/bin/env python3
"""Driver benchmark: GEMM GFLOPS of the B200-native hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload hgemm|sgemm|batched_h32|batched_s32|batched_h64|batched_s64|
                                sgemm_c1|hgemm_c3|sgemm_c3|hgemm_c5|sgemm_c5]
                    [--no-extra] [--no-cpu-baseline]

A "step" is one call of the hot path on one batch of synthetic input:
* hgemm (default, the headline): C = A·B, 8192^3, FP16 storage / FP32
  accumulate, row-major NN, alpha=1, beta=0 (BASELINE configs[1], largest
  square size of the sweep);
* sgemm: the same shape in FP32 (FFMA);
* batched_*: gemm_strided_batched, 16384 instances of 32^3 / 64^3 (configs[3]).

value   = whole-job GFLOPS with inputs resident in HBM, CUDA-event timed per
          step on the launching stream (max over ranks), L2 flushed between
          steps (256 MiB write + 256 MiB read) so no step reads a warm L2.
e2e     = the same metric through the public API with HOST buffers: pinned
          host → device copy of A and B, the routine, device → host copy of C,
          all inside the timed region.
N > 1   = weak scaling: rank r computes its own 8192-column block of an
          8192 x (8192·N) x 8192 GEMM (column-sharded C, no collective) or its
          own 16384-instance block of the batch.
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
    # C5: the large GEMM (per rank under torchrun: weak scaling, each rank its
    # own 32768-column block)
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
def make_operands(tb, ctx, w, rank, world, torch):
    prec = tb.Precision.H if w["prec"] == "H" else tb.Precision.S
    dt = prec.torch_dtype
    dev = ctx.torch_device
    g = torch.Generator(device=dev).manual_seed(12345 + rank)
    if w["kind"] == "gemm":
        m, n, k = w["m"], w["n"], w["k"]
        # rank's column block of an m x (n*world) x k GEMM: A (m x k) replicated,
        # B block (k x n) and C block (m x n) local — row-major packed.
        na, nb, nc = m * k, k * n, m * n
    else:
        e = w["m"] * w["k"]
        na = nb = nc = e * w["batch"]
    at = (torch.rand(na, device=dev, generator=g) * 2 - 1).to(dt)
    bt = (torch.rand(nb, device=dev, generator=g) * 2 - 1).to(dt)
    ct = torch.zeros(nc, device=dev, dtype=dt)
    return prec, tb.buffer_from_tensor(ctx, prec, at), tb.buffer_from_tensor(ctx, prec, bt), \
        tb.buffer_from_tensor(ctx, prec, ct)


def step_fn(tb, ctx, w, prec, a, b, c):
    L, T = tb.Layout.ROW_MAJOR, tb.Transpose.NO
    if w["kind"] == "gemm":
        m, n, k = w["m"], w["n"], w["k"]
        return lambda: tb.gemm(ctx, L, T, T, m, n, k, 1.0, a, b, 0.0, c)
    m, e, bt = w["m"], w["m"] * w["m"], w["batch"]
    return lambda: tb.gemm_strided_batched(ctx, L, T, T, m, m, m, 1.0, a, e, b, e, 0.0, c, e, bt)


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


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1705_05249_b200 as tb
    from paper_1705_05249_b200.kernels import native

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

    def measure(name, steps, warmup):
        w = WORKLOADS[name]
        prec, a, b, c = make_operands(tb, ctx, w, rank, world, torch)
        fn = step_fn(tb, ctx, w, prec, a, b, c)
        fn()
        torch.cuda.synchronize()
        kernel = ctx.last_launch.native["kernel"]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler = ClockSampler(local_rank)
        with sampler:
            times = device_time(fn, steps, warmup, stream, torch, flush)
        total = sum(times)
        if world > 1:
            t = torch.tensor([total], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total = float(t.item())
        per_launch = total / steps
        gflops = flops(w) * world * steps / total / 1e9
        ai = flops(w) / alg_bytes(w)
        ridge = (peaks["bf16_tflops"] if w["prec"] == "H" else FFMA_TFLOPS) * 1e12 / (peaks["hbm_gbs"] * 1e9)
        if w["kind"] == "gemm" and ai < ridge:
            bound = "hbm"
            peak, unit, achieved = peaks["hbm_gbs"], "GB/s", alg_bytes(w) / per_launch / 1e9
            peak_note = (f"HBM copy bandwidth ({peak_src}: MEASURED_PEAKS.json hbm_gbs); "
                         f"arithmetic intensity {ai:.0f} flop/B < ridge {ridge:.0f}")
        elif w["prec"] == "H" and w["kind"] == "gemm":
            bound = "tensor"
            peak, unit, achieved = peaks["bf16_tflops"], "TFLOP/s", flops(w) / per_launch / 1e12
            peak_note = f"dense FP16/BF16 tensor, burst ({peak_src}: MEASURED_PEAKS.json bf16_tflops)"
        elif w["kind"] == "gemm":
            bound = "ffma"
            peak, unit, achieved = FFMA_TFLOPS, "TFLOP/s", flops(w) / per_launch / 1e12
            peak_note = "FP32 FFMA 148 SM x 128 lanes x 2 x 1.965 GHz (derived, no measured FFMA peak)"
        else:
            bound = "hbm"
            peak, unit, achieved = peaks["hbm_gbs"], "GB/s", alg_bytes(w) / per_launch / 1e9
            peak_note = f"HBM copy bandwidth ({peak_src}: MEASURED_PEAKS.json hbm_gbs)"
        return dict(name=name, w=w, times=times, total=total, gflops=gflops, kernel=kernel,
                    clocks=sampler.summary(), a=a, b=b, c=c, prec=prec, fn=fn,
                    roofline={"bound": bound, "achieved": round(achieved, 2), "peak": peak,
                              "unit": unit, "frac": round(achieved / peak, 4),
                              "traffic": None, "peak_source": peak_note,
                              "kernel": kernel, "per_launch_ms": round(per_launch * 1e3, 4),
                              "algorithmic": f"{flops(w):.4g} FLOP, {alg_bytes(w):.4g} B per launch"})

    main = measure(args.workload, args.steps, args.warmup)
    w = main["w"]

    # ---- e2e: public API with host buffers, copies inside the timed region ----
    # Every step copies its A and B from pinned host memory, runs the routine
    # and copies C back.  Steps are software-pipelined over three streams
    # (H2D copy engine, compute, D2H copy engine) with double-buffered device
    # operands, so step i's D2H and step i+1's H2D overlap (PCIe is full
    # duplex) — the copies of every step stay inside the timed region.
    prec, a, b, c = main["prec"], main["a"], main["b"], main["c"]
    dt = prec.torch_dtype
    host_a = torch.empty(a.length, dtype=dt, pin_memory=True)
    host_b = torch.empty(b.length, dtype=dt, pin_memory=True)
    host_c = [torch.empty(c.length, dtype=dt, pin_memory=True) for _ in range(2)]
    host_a.copy_(a.device_tensor())
    host_b.copy_(b.device_tensor())
    sets = [(a, b, c)]
    sets.append(tuple(tb.buffer_from_tensor(ctx, prec, torch.empty(x.length, dtype=dt, device=dev))
                      for x in (a, b, c)))
    s_h2d, s_cmp, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    fns = [step_fn(tb, ctx, w, prec, *st) for st in sets]

    def run_e2e(n_steps):
        done_cmp = [None, None]   # compute finished with set i (its inputs are free)
        done_d2h = [None, None]   # D2H finished with set i (its C is free)
        for i in range(n_steps):
            j = i & 1
            da, db, dc = (x.device_tensor() for x in sets[j])
            with torch.cuda.stream(s_h2d):
                if done_cmp[j] is not None:
                    s_h2d.wait_event(done_cmp[j])
                da.copy_(host_a, non_blocking=True)
                db.copy_(host_b, non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_h2d)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in)
                if done_d2h[j] is not None:
                    s_cmp.wait_event(done_d2h[j])
                fns[j]()
                done_cmp[j] = torch.cuda.Event()
                done_cmp[j].record(s_cmp)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(done_cmp[j])
                host_c[j].copy_(dc, non_blocking=True)
                done_d2h[j] = torch.cuda.Event()
                done_d2h[j].record(s_d2h)

    e2e_steps = max(4, min(args.steps, 20))
    run_e2e(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0_ev, t1_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0_ev.record(s_h2d)
    for st_ in (s_cmp, s_d2h):
        st_.wait_event(t0_ev)
    run_e2e(e2e_steps)
    for st_ in (s_cmp, s_h2d):
        s_d2h.wait_stream(st_)
    t1_ev.record(s_d2h)
    torch.cuda.synchronize()
    e2e_total = t0_ev.elapsed_time(t1_ev) / 1e3
    if world > 1:
        t = torch.tensor([e2e_total], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    es = prec.elemsize
    e2e = {"value": round(flops(w) * world * e2e_steps / e2e_total / 1e9, 2), "unit": "GFLOPS",
           "h2d_bytes_per_step": (a.length + b.length) * es, "d2h_bytes_per_step": c.length * es,
           "ms_per_step": round(e2e_total / e2e_steps * 1e3, 4), "steps": e2e_steps,
           "path": "pinned host A,B -> device (copy stream); public gemm API (compute stream); "
                   "device C -> pinned host (copy stream); steps pipelined, double-buffered"}

    # ---- extras: the other headline configs (device-timed, this rank) ----
    extra = {}
    if not args.no_extra:
        for name in WORKLOADS:
            if name == args.workload:
                continue
            try:
                big = WORKLOADS[name]["m"] >= 32768
                r = measure(name, 3 if big else max(5, min(args.steps, 20)), min(args.warmup, 3) if big else args.warmup)
                extra[name] = {"workload": describe(r["w"]), "value": round(r["gflops"], 1),
                               "unit": "GFLOPS", "ms_per_step": round(r["total"] / max(1, len(r["times"])) * 1e3, 4),
                               "roofline": r["roofline"], "clocks": r["clocks"]}
                del r
            except Exception as exc:  # noqa: BLE001
                extra[name] = {"error": repr(exc)}
            torch.cuda.empty_cache()

    if not args.no_extra:
        try:
            extra["im2col"] = im2col_extra(tb, ctx, stream, torch, flush, peaks, peak_src)
        except Exception as exc:  # noqa: BLE001
            extra["im2col"] = {"error": repr(exc)}
        torch.cuda.empty_cache()

    # North star: batched small-matrix GEMM >= 10x the naive per-matrix launch
    # loop.  Loop = one public `gemm` call per instance (first 1024 instances
    # of the 16384 x 32^3 batch, device-timed), extrapolated per instance.
    if not args.no_extra:
        try:
            extra["batched_vs_loop"] = batched_vs_loop(tb, ctx, stream, torch)
        except Exception as exc:  # noqa: BLE001
            extra["batched_vs_loop"] = {"error": repr(exc)}

    if rank != 0:
        return None
    traffic = load_traffic(args.workload, main["kernel"])
    if traffic is not None:
        main["roofline"]["traffic"] = traffic
    for name, ex in extra.items():
        if isinstance(ex, dict) and isinstance(ex.get("roofline"), dict):
            t = load_traffic(name, ex["roofline"].get("kernel", ""))
            if t is not None:
                ex["roofline"]["traffic"] = t
    line = {
        "metric": METRIC,
        "value": round(main["gflops"], 2),
        "unit": "GFLOPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(main["total"] / args.steps * 1e3, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f16" if w["prec"] == "H" else "f32",
        "data": "synthetic U(-1,1) operands, seeded, resident in HBM",
        "config": {"workload": describe(w), "m": w["m"], "n": w["n"] * (world if w["kind"] == "gemm" else 1),
                   "k": w["k"], "batch": w["batch"] * (world if w["kind"] == "batched" else 1),
                   "layout": "row-major", "trans": "NN", "alpha": 1.0, "beta": 0.0,
                   "parallelism": f"column-sharded x{world}" if w["kind"] == "gemm" else f"batch-sharded x{world}",
                   "l2": "flushed before every step (256 MiB write + 256 MiB read of a second buffer: "
                         "inputs evicted, no dirty lines left)"},
        "e2e": e2e,
        "gpu_launches": args.steps,
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
        _, a, b, c = make_operands(tb, ctx, w, 0, 1, torch)
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
        "scaling": "weak", "vs_baseline": None, "dtype": "f16" if w["prec"] == "H" else "f32",
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
