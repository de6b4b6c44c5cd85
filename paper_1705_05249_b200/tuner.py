"""Measurement-driven auto-tuning of the GEMM kernel family on the GPU.

Same protocol and data model as the reference tuner (pkg/src/tunedblas/
tuner.py:44-358): explore the valid curated set (params.py:221-243) plus
``budget`` seeded random draws from the full grid (deduplicated, filtered,
<= 10*budget rejections), verify each candidate once against the oracle
(status "failed" on mismatch or exception), then 1 warm-up + 10 timed runs;
best = lowest mean, then fewest threads, then lexicographic parameters.

What changes on the B200: the family that selects kernels is
``gemm_b200`` (kernels/params.py; include/tbgemm.h tb_gemm_config) — CTA
tile MWG x NWG, K depth per stage KWG, ring depth STAGES, tcgen05
CTA_GROUP, cluster SPLIT_K and raster GROUP_M — whose curated set is the
built-in shape route followed by every instantiated kernel of the precision
under each curated GROUP_M, so the tuned best is never slower than the
untuned default.  Every run is timed with CUDA events on the launching
stream, inputs stay resident in HBM, and the oracle is a float64 product
computed on the device with the exact tolerance bound.  The reference's
14-parameter ``gemm`` family can still be tuned (same protocol; its
configurations are validated and recorded but select no kernel on sm_100a).
"""

from __future__ import annotations

import random
from dataclasses import dataclass, field

import numpy as np

from .core import Context, DeviceSpec, Layout, Precision, Transpose, buffer_alloc, buffer_write
from .errors import TuningError, UsageError
from .kernels.dispatch import gemm_native
from .kernels.params import (
    Configuration,
    curated_b200,
    curated_configurations,
    is_b200_auto,
    random_configuration,
    validate_config,
    work_group_threads,
)
from .reference import device_expected, device_within_tol, gemm_tolerance_device
from .tuningdb import DbEntry, DbKey

__all__ = ["TuningTask", "Measurement", "TuningRun", "measure", "tune", "best_config"]


@dataclass
class TuningTask:
    """What to tune: one kernel family at one precision and problem size."""

    kernel_family: str
    precision: Precision
    args: dict
    device: DeviceSpec
    budget: int = 0
    seed: int = 0
    warmup_runs: int = 1
    timed_runs: int = 10

    def __post_init__(self):
        if self.timed_runs < 1:
            raise UsageError("timed_runs must be >= 1")
        if self.budget < 0:
            raise UsageError("budget must be >= 0")

    def sizes(self) -> tuple:
        return (int(self.args.get("m", 0)), int(self.args.get("n", 0)), int(self.args.get("k", 0)))


@dataclass
class Measurement:
    configuration: Configuration
    status: str  # ok | invalid | failed
    per_run_times: list = field(default_factory=list)
    mean_time: float = float("inf")
    violations: list = field(default_factory=list)
    kernel: str = ""

    def to_json(self) -> dict:
        doc = {
            "params": self.configuration.as_dict(),
            "per_run_times_s": list(self.per_run_times),
            "mean_time_s": self.mean_time if self.status == "ok" else None,
            "status": self.status,
        }
        if self.violations:
            doc["violations"] = list(self.violations)
        if self.kernel:
            doc["kernel"] = self.kernel
        return doc


@dataclass
class TuningRun:
    task: TuningTask
    measurements: list
    best: Configuration

    def to_db_entry(self) -> DbEntry:
        key = DbKey.for_task(self.task.kernel_family, self.task.precision, self.task.device,
                             self.task.sizes())
        return DbEntry(key=key, measurements=[m.to_json() for m in self.measurements], best=self.best)

    def to_json(self) -> dict:
        return {
            "task": {
                "family": self.task.kernel_family,
                "precision": self.task.precision.value,
                "args": {k: int(v) for k, v in self.task.args.items()},
                "device": self.task.device.to_dict(),
                "budget": self.task.budget,
                "seed": self.task.seed,
                "warmup_runs": self.task.warmup_runs,
                "timed_runs": self.task.timed_runs,
            },
            "measurements": [m.to_json() for m in self.measurements],
            "best": self.best.as_dict(),
        }


class _KernelHarness:
    """Fixed device-resident inputs, a run closure and the oracle check.

    Inputs follow the reference harness (tuner.py:152-156, 223-250):
    U(-1, 1) from ``np.random.default_rng(12345)``, A (m x k), B (k x n),
    C = A @ B with alpha = 1, beta = 0, column-major NN.
    """

    def __init__(self, task: TuningTask, ctx: Context):
        import torch

        if task.kernel_family not in ("gemm", "gemm_b200"):
            raise UsageError(f"unknown kernel family {task.kernel_family!r}")
        m, n, k = task.sizes()
        if m < 1 or n < 1 or k < 1:
            raise UsageError("gemm tuning requires m, n, k >= 1")
        self.task, self.ctx = task, ctx
        precision = task.precision
        rng = np.random.default_rng(12345)
        a = rng.uniform(-1.0, 1.0, size=(m, k)).astype(precision.dtype)
        b = rng.uniform(-1.0, 1.0, size=(k, n)).astype(precision.dtype)
        self.m, self.n, self.k = m, n, k
        self.abuf = buffer_alloc(ctx, precision, m * k)
        self.bbuf = buffer_alloc(ctx, precision, k * n)
        self.cbuf = buffer_alloc(ctx, precision, m * n)
        buffer_write(self.abuf, 0, a.reshape(-1, order="F"))
        buffer_write(self.bbuf, 0, b.reshape(-1, order="F"))
        dev = ctx.torch_device
        at = torch.from_numpy(a).to(dev)
        bt = torch.from_numpy(b).to(dev)
        self.expected = device_expected(at, bt)
        self.tol = gemm_tolerance_device(at, bt, precision)
        self.last_kernel = ""

    def run(self, cfg: Configuration):
        t = self.task
        # only gemm_b200 configurations select a kernel (the all-zero one is
        # the built-in shape route); reference configurations are recorded only
        kcfg = cfg if cfg.family == "gemm_b200" and not is_b200_auto(cfg) else None
        launched = gemm_native(self.ctx, t.precision, Layout.COL_MAJOR, Transpose.NO, Transpose.NO,
                               self.m, self.n, self.k, 1.0, self.abuf, 0, self.m,
                               self.bbuf, 0, self.k, 0.0, self.cbuf, 0, self.m, kcfg)
        self.last_kernel = launched["kernel"]
        return self.cbuf

    def result(self):
        return self.cbuf.device_tensor().view(self.n, self.m).t()

    def prewarm(self, cfg: Configuration, seconds: float = 0.05) -> None:
        """Run ``cfg`` back to back for ~``seconds`` of device time before the
        first measurement, so the first candidate (the built-in route) is not
        timed on a GPU still ramping its clocks up from idle."""
        import torch

        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(self.ctx.stream)
        self.run(cfg)
        t1.record(self.ctx.stream)
        t1.synchronize()
        reps = int(min(10000, max(1, seconds * 1e3 / max(t0.elapsed_time(t1), 1e-3))))
        for _ in range(reps):
            self.run(cfg)
        self.ctx.stream.synchronize()

    def verify(self, cfg: Configuration) -> bool:
        self.run(cfg)
        return device_within_tol(self.result(), self.expected, self.tol)


def measure(config: Configuration, task: TuningTask, ctx: Context,
            harness: _KernelHarness | None = None) -> Measurement:
    """Filter, oracle check, warm-up, then CUDA-event-timed runs."""
    import torch

    verdict = validate_config(config, task.device, task.precision)
    if not verdict:
        return Measurement(config, "invalid", violations=verdict.violations)
    harness = harness or _KernelHarness(task, ctx)
    try:
        if not harness.verify(config):
            return Measurement(config, "failed")
    except Exception:  # noqa: BLE001 - any failure marks the candidate failed
        return Measurement(config, "failed")
    stream = ctx.stream
    for _ in range(task.warmup_runs):
        harness.run(config)
    events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(task.timed_runs)]
    # Hold the stream in a ~1 ms device-side spin while the timed runs are
    # enqueued, so each event pair brackets device time only — a kernel
    # shorter than the host's per-call launch cost would otherwise be timed
    # at the launch rate.
    torch.cuda._sleep(2_000_000)
    for e0, e1 in events:
        e0.record(stream)
        harness.run(config)
        e1.record(stream)
    stream.synchronize()
    times = [e0.elapsed_time(e1) / 1e3 for e0, e1 in events]
    return Measurement(config, "ok", per_run_times=times, mean_time=float(np.mean(times)),
                       kernel=harness.last_kernel)


def tune(task: TuningTask, ctx: Context) -> TuningRun:
    """Explore curated + random configurations; return every measurement."""
    if ctx.device != task.device:
        raise UsageError("tuning task device does not match the context device")
    harness = _KernelHarness(task, ctx)
    explored: list[Configuration] = []
    seen = set()
    curated = (curated_b200(task.precision) if task.kernel_family == "gemm_b200"
               else curated_configurations(task.kernel_family))
    for cfg in curated:
        if validate_config(cfg, task.device, task.precision) and cfg not in seen:
            explored.append(cfg)
            seen.add(cfg)
    rng = random.Random(task.seed)
    accepted = rejections = 0
    limit = 10 * task.budget
    while accepted < task.budget and rejections <= limit:
        cand = random_configuration(task.kernel_family, rng)
        if cand in seen or not validate_config(cand, task.device, task.precision):
            rejections += 1
            continue
        explored.append(cand)
        seen.add(cand)
        accepted += 1
    if explored:
        harness.prewarm(explored[0])
    measurements = [measure(cfg, task, ctx, harness) for cfg in explored]
    # The gemm_b200 built-in route is timed first, right after the pre-warm,
    # while the clocks are still settling under the power cap (8192^3 HGEMM:
    # 986 us first against ~720 us later in one run): time it again last and
    # keep the faster of the two, so "tuned vs built-in" compares like with like.
    if (task.kernel_family == "gemm_b200" and explored and is_b200_auto(explored[0])
            and measurements[0].status == "ok"):
        again = measure(explored[0], task, ctx, harness)
        if again.status == "ok" and again.mean_time < measurements[0].mean_time:
            measurements[0] = again
    ok = [m for m in measurements if m.status == "ok"]
    if not ok:
        raise TuningError(f"no valid configuration for device {task.device.name!r} "
                          f"(family {task.kernel_family}, explored {len(explored)})")
    return TuningRun(task=task, measurements=measurements, best=_select_best(ok))


def _tie_break(cfg: Configuration) -> int:
    """Second key after the mean time: fewest threads (reference,
    tuner.py:344-349); for gemm_b200 the built-in route wins ties."""
    if cfg.family == "gemm_b200":
        return 0 if is_b200_auto(cfg) else 1
    return work_group_threads(cfg)


def _select_best(ok_measurements) -> Configuration:
    return min(ok_measurements, key=lambda m: (m.mean_time, _tie_break(m.configuration),
                                               m.configuration.values)).configuration


def best_config(run: TuningRun) -> Configuration:
    ok = [m for m in run.measurements if m.status == "ok"]
    if not ok:
        raise TuningError("tuning run has no ok measurements")
    return _select_best(ok)
