"""Benchmark clients: GFLOPS, size sweeps, CSV/JSON reports and the
problem-specific-tuning heat map (pkg/src/tunedblas/bench.py:45-356 of the
reference), measured on the GPU.

Timing: CUDA events on the context's stream around each run (the reference
timed host ``perf_counter``, bench.py:132-146); 1 warm-up + 10 runs by
default.  The comparison arm is the vendor library on the same device
(``torch.matmul`` → cuBLAS), where the reference compared against its naive
NumPy ``ref_gemm``; correctness is checked against a float64 device product
with the reference tolerance.
"""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass, field

import numpy as np

from .core import Context, Layout, Precision, Transpose, buffer_alloc, buffer_write
from .errors import ExperimentError, UsageError
from .reference import device_expected, device_within_tol, gemm_tolerance_device
from .routines import gemm
from .routines.common import get_store
from .tuner import TuningTask, tune
from .tuningdb import Database

__all__ = ["BenchRow", "HeatmapResult", "METRIC_TABLE", "metrics", "sweep_sizes", "run_client",
           "heatmap_experiment", "write_report", "time_on_stream"]

#: metric kind and formula (bench.py:45-51); gemm counts 2mnk (8mnk complex).
METRIC_TABLE = {
    "gemm": ("GFLOPS", lambda m, n, k, es, cplx: (8 if cplx else 2) * m * n * k),
    "gemm_batched": ("GFLOPS", lambda m, n, k, es, cplx: (8 if cplx else 2) * m * n * k),
}


def metrics(routine: str, size, precision: Precision, seconds: float):
    """(value, kind) for one timed execution (bench.py:54-67)."""
    if seconds <= 0:
        raise UsageError("time must be > 0")
    if routine not in METRIC_TABLE:
        raise UsageError(f"no metric formula for routine {routine!r}")
    kind, formula = METRIC_TABLE[routine]
    m, n, k = (tuple(size) + (0, 0, 0))[:3]
    amount = formula(m, n, k, precision.elemsize, precision.is_complex)
    return amount / seconds / 1e9, kind


@dataclass
class BenchRow:
    routine: str
    precision: str
    size: tuple
    mean_time: float
    per_run_times: list
    metric_value: float
    metric_kind: str
    reference_mean_time: float
    reference_per_run_times: list
    correct: bool
    kernel: str = ""

    def to_json(self) -> dict:
        return {
            "routine": self.routine,
            "precision": self.precision,
            "size": {"m": self.size[0], "n": self.size[1], "k": self.size[2]},
            "mean_time_s": self.mean_time,
            "per_run_times_s": list(self.per_run_times),
            "metric_value": self.metric_value,
            "metric_kind": self.metric_kind,
            "reference_mean_time_s": self.reference_mean_time,
            "reference_per_run_times_s": list(self.reference_per_run_times),
            "correct": self.correct,
            "kernel": self.kernel,
        }


CSV_HEADER = ["routine", "precision", "m", "n", "k", "mean_time_s", "metric_value",
              "metric_kind", "reference_mean_time_s", "correct"]


@dataclass
class HeatmapResult:
    tuned_sizes: list
    bench_sizes: list
    relative_perf: np.ndarray
    times: np.ndarray = field(default=None)

    def to_json(self) -> dict:
        return {
            "tuned_sizes": [list(s) for s in self.tuned_sizes],
            "bench_sizes": [list(s) for s in self.bench_sizes],
            "relative_perf_percent": self.relative_perf.tolist(),
            "times_s": self.times.tolist() if self.times is not None else None,
        }


def sweep_sizes(start: int, step: int, count: int) -> list[int]:
    if count < 1 or start < 1 or step < 0:
        raise UsageError("sweep requires start >= 1, step >= 0, count >= 1")
    return [start + i * step for i in range(count)]


def time_on_stream(fn, warmup: int, runs: int, stream) -> list[float]:
    """Per-run seconds from CUDA events recorded on ``stream``."""
    import torch

    for _ in range(warmup):
        fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(runs)]
    for e0, e1 in evs:
        e0.record(stream)
        fn()
        e1.record(stream)
    stream.synchronize()
    return [e0.elapsed_time(e1) / 1e3 for e0, e1 in evs]


class _ClientCase:
    """Buffers, tuned closure, library closure and oracle for one size
    (bench.py:149-232; seed 98765, U(-1, 1), column-major NN, alpha=1, beta=0)."""

    def __init__(self, routine: str, size, precision: Precision, ctx: Context):
        import torch

        if routine != "gemm":
            raise UsageError(f"client does not support routine {routine!r}")
        rng = np.random.default_rng(98765)
        m, n, k = (tuple(size) + (0, 0, 0))[:3]
        self.size = (m, n, k)
        a = rng.uniform(-1, 1, (m, k)).astype(precision.dtype)
        b = rng.uniform(-1, 1, (k, n)).astype(precision.dtype)
        ab = buffer_alloc(ctx, precision, m * k)
        bb = buffer_alloc(ctx, precision, k * n)
        cb = buffer_alloc(ctx, precision, m * n)
        buffer_write(ab, 0, a.reshape(-1, order="F"))
        buffer_write(bb, 0, b.reshape(-1, order="F"))
        dev = ctx.torch_device
        at, bt = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
        self.expected = device_expected(at, bt)
        self.tol = gemm_tolerance_device(at, bt, precision)
        self.kernel = ""

        def tuned():
            gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, ab, bb, 0.0, cb)
            if ctx.last_launch is not None and ctx.last_launch.native:
                self.kernel = ctx.last_launch.native["kernel"]

        lib_out = torch.empty((m, n), dtype=precision.torch_dtype, device=dev)

        def library():
            torch.matmul(at, bt, out=lib_out)

        self.tuned, self.library = tuned, library
        self.result_of = lambda: cb.device_tensor().view(n, m).t()

    def verify(self) -> bool:
        self.tuned()
        return device_within_tol(self.result_of(), self.expected, self.tol)


def run_client(routine: str, sizes, precision: Precision, ctx: Context,
               db: Database | None = None, warmup: int = 1, runs: int = 10):
    """Benchmark ``routine`` over ``sizes`` (bench.py:235-267)."""
    if not sizes:
        raise UsageError("size sweep must be non-empty")
    if db is not None:
        get_store(ctx).database = db
    rows = []
    for size in sizes:
        case = _ClientCase(routine, size, precision, ctx)
        correct = case.verify()
        tuned_times = time_on_stream(case.tuned, warmup, runs, ctx.stream)
        lib_times = time_on_stream(case.library, warmup, runs, ctx.stream)
        mean = float(np.mean(tuned_times))
        value, kind = metrics(routine, case.size, precision, mean)
        rows.append(BenchRow(routine=routine, precision=precision.value, size=case.size,
                             mean_time=mean, per_run_times=tuned_times, metric_value=value,
                             metric_kind=kind, reference_mean_time=float(np.mean(lib_times)),
                             reference_per_run_times=lib_times, correct=bool(correct),
                             kernel=case.kernel))
    return rows


def write_report(rows, csv_path=None, json_path=None) -> None:
    if csv_path:
        with open(csv_path, "w", newline="", encoding="utf-8") as fh:
            writer = csv.writer(fh)
            writer.writerow(CSV_HEADER)
            for r in rows:
                writer.writerow([r.routine, r.precision, r.size[0], r.size[1], r.size[2],
                                 f"{r.mean_time:.9g}", f"{r.metric_value:.6g}", r.metric_kind,
                                 f"{r.reference_mean_time:.9g}", int(r.correct)])
    if json_path:
        with open(json_path, "w", encoding="utf-8") as fh:
            json.dump({"rows": [r.to_json() for r in rows]}, fh, indent=1)


def heatmap_experiment(sizes, precision: Precision, ctx: Context, budget: int = 32,
                       seed: int = 7, warmup: int = 1, runs: int = 10,
                       family: str | None = None) -> HeatmapResult:
    """Problem-specific-tuning heat map (bench.py:287-356): tune once per
    size, then time every (benched size, tuned-for size) pair through a
    runtime override; relative_perf[i][j] = 100 * t(i, p_i) / t(i, p_j).
    ``family`` defaults to gemm_b200 (the family that selects sm_100a
    kernels) on a B200 and to the reference's gemm elsewhere."""
    if family is None:
        family = "gemm_b200" if ctx.device.is_b200 else "gemm"
    sizes = [tuple(int(v) for v in s) for s in sizes]
    if len(set(sizes)) != len(sizes):
        raise UsageError("heat-map sizes must be distinct")
    store = get_store(ctx)
    best = {}
    for size in sizes:
        m, n, k = size
        task = TuningTask(family, precision, {"m": m, "n": n, "k": k}, ctx.device,
                          budget=budget, seed=seed, warmup_runs=warmup, timed_runs=runs)
        try:
            best[size] = tune(task, ctx).best
        except Exception as exc:  # noqa: BLE001
            raise ExperimentError(f"tuning failed for size {size}: {exc}") from exc
    count = len(sizes)
    times = np.zeros((count, count))
    for i, bench_size in enumerate(sizes):
        case = _ClientCase("gemm", bench_size, precision, ctx)
        for j in range(count):
            store.set_override(family, precision, ctx.device, bench_size, best[sizes[j]])
            if not case.verify():
                store.clear_overrides()
                raise ExperimentError(f"correctness failure at size {bench_size} with "
                                      f"parameters tuned for {sizes[j]}")
        per_run = np.zeros((count, runs))
        for r in range(runs):
            for j in range(count):
                store.set_override(family, precision, ctx.device, bench_size, best[sizes[j]])
                per_run[j, r] = time_on_stream(case.tuned, warmup if r == 0 else 0, 1, ctx.stream)[0]
        times[i, :] = per_run.mean(axis=1)
        store.clear_overrides()
    rel = np.empty((count, count))
    for i in range(count):
        for j in range(count):
            rel[i, j] = 100.0 if i == j else 100.0 * times[i, i] / times[i, j]
    return HeatmapResult(tuned_sizes=sizes, bench_sizes=sizes, relative_perf=rel, times=times)
