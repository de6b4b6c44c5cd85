"""On-device auto-tuner: protocol, fault injection, persistence
(reference tests/test_tuner.py, test_acceptance.py:120-155)."""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import GemmParams, Precision
from paper_1705_05249_b200.kernels import curated_configurations, validate_config
from paper_1705_05249_b200.tuner import Measurement, TuningRun, TuningTask, _KernelHarness, \
    best_config, measure, tune

pytestmark = pytest.mark.gpu


def small_task(device, prec=Precision.S, budget=0, runs=10, size=64):
    return TuningTask("gemm", prec, {"m": size, "n": size, "k": size}, device, budget=budget,
                      timed_runs=runs)


def test_measure_protocol_counts(ctx):
    task = small_task(ctx.device)
    harness = _KernelHarness(task, ctx)
    calls = {"n": 0}
    inner = harness.run

    def counting(cfg):
        calls["n"] += 1
        return inner(cfg)

    harness.run = counting
    m = measure(GemmParams(MWG=64, NWG=64).to_config(), task, ctx, harness)
    assert m.status == "ok" and len(m.per_run_times) == 10
    assert calls["n"] == 1 + 1 + 10
    assert m.mean_time == pytest.approx(float(np.mean(m.per_run_times)))
    # reference-family configurations select no kernel on sm_100a: the
    # built-in shape route runs (gemm_b200 selects kernels, test_tuner_b200_gpu)
    assert m.kernel.startswith("sgemm_")


def test_measure_invalid_and_failed(ctx):
    task = small_task(ctx.device)
    bad = GemmParams(MDIMC=32, NDIMC=64, MWG=16, NWG=16).to_config()
    m = measure(bad, task, ctx)
    assert m.status == "invalid" and m.violations and m.per_run_times == []
    harness = _KernelHarness(task, ctx)
    inner = harness.result
    harness.result = lambda: inner() + 1.0          # injected fault
    m = measure(GemmParams().to_config(), task, ctx, harness)
    assert m.status == "failed" and m.per_run_times == []


@pytest.mark.parametrize("prec", [Precision.S, Precision.H])
def test_tune_budget_and_db_roundtrip(ctx, tmp_path, prec):
    task = small_task(ctx.device, prec=prec, budget=8, runs=2, size=256)
    run = tune(task, ctx)
    valid = [c for c in curated_configurations("gemm") if validate_config(c, ctx.device, prec)]
    explored = [m.configuration for m in run.measurements]
    assert explored[:len(valid)] == valid
    assert 0 < len(explored) - len(valid) <= 8
    assert len(set(explored)) == len(explored)
    assert all(m.status == "ok" for m in run.measurements)
    assert best_config(run) == run.best
    db = tb.Database()
    tb.db_insert(db, run)
    path = tmp_path / "db.json"
    db.save(path)
    loaded = tb.Database.load(path)
    cfg, level = tb.db_lookup(loaded, ctx.device, "gemm", prec, (256, 256, 256))
    assert cfg == run.best and level == "device"
    # the tuned configuration is selected at call time
    tb.routines.common.get_store(ctx).database = loaded
    n = 256
    a = tb.buffer_alloc(ctx, prec, n * n)
    tb.gemm(ctx, tb.Layout.COL_MAJOR, tb.Transpose.NO, tb.Transpose.NO, n, n, n, 1.0, a, a, 0.0,
            tb.buffer_alloc(ctx, prec, n * n))
    assert ctx.last_launch.params == run.best.as_dict()


def test_tuner_cli_smoke(tmp_path, capsys):
    from paper_1705_05249_b200.cli import tuner_main

    db_path, json_path = tmp_path / "db.json", tmp_path / "run.json"
    rc = tuner_main("gemm", ["-m", "128", "-n", "128", "-k", "128", "--runs", "2", "--budget", "2",
                             "--db", str(db_path), "--json", str(json_path), "--precision", "16"])
    assert rc == 0
    assert "best:" in capsys.readouterr().out
    assert db_path.exists() and json_path.exists()


def test_client_and_heatmap(ctx):
    rows = tb.run_client("gemm", [(256, 256, 256), (129, 129, 129)], Precision.S, ctx, runs=3)
    assert all(r.correct for r in rows) and all(r.metric_kind == "GFLOPS" for r in rows)
    res = tb.heatmap_experiment([(64, 64, 64), (512, 512, 512)], Precision.H, ctx, budget=0,
                                runs=2)
    assert np.all(np.diag(res.relative_perf) == 100.0)
