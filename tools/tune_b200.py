"""On-device tuning of the BASELINE C3 shapes + the problem-specific-tuning
heat map (paper Fig. 4) on the B200.  Writes gpurun_out/r1_tuning_db.json and
profiles/r1_heatmap_*.json.  Dev tool; uses only the public API."""
import json, sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.tuner import TuningTask, tune

ctx = tb.context_create(tb.host_device())
db = tb.Database()
summary = []
shapes = [(64, 3136, 576), (4096, 128, 9216), (1024, 1024, 1024), (8192, 8192, 8192)]
for prec in (tb.Precision.H, tb.Precision.S):
    for (m, n, k) in shapes:
        if prec is tb.Precision.S and m * n * k > 2e11:
            continue
        t0 = time.perf_counter()
        task = TuningTask("gemm", prec, {"m": m, "n": n, "k": k}, ctx.device, budget=16, seed=1,
                          warmup_runs=1, timed_runs=5 if m * n * k > 1e11 else 10)
        run = tune(task, ctx)
        tb.db_insert(db, run)
        ok = [x for x in run.measurements if x.status == "ok"]
        best = min(ok, key=lambda x: x.mean_time)
        default = [x for x in ok if x.configuration == tb.kernels.default_config("gemm", ctx.device, prec)]
        kernels = sorted({x.kernel for x in ok})
        row = dict(precision=prec.value, m=m, n=n, k=k, explored=len(run.measurements), ok=len(ok),
                   best_us=best.mean_time * 1e6, best_kernel=best.kernel, best=run.best.as_dict(),
                   default_us=default[0].mean_time * 1e6 if default else None,
                   median_us=float(np.median([x.mean_time for x in ok])) * 1e6,
                   gflops_best=2 * m * n * k / best.mean_time / 1e9, distinct_kernels=kernels,
                   seconds=time.perf_counter() - t0)
        summary.append(row)
        print(json.dumps({k_: v for k_, v in row.items() if k_ != "best"}), flush=True)
db.save("gpurun_out/r1_tuning_db.json")
json.dump(summary, open("gpurun_out/r1_tuning_summary.json", "w"), indent=1)
for prec in (tb.Precision.S, tb.Precision.H):
    res = tb.heatmap_experiment([(64, 3136, 576), (4096, 128, 9216), (1024, 1024, 1024)], prec, ctx,
                                budget=8, seed=5, runs=5)
    json.dump(res.to_json(), open(f"gpurun_out/r1_heatmap_{prec.value}.json", "w"), indent=1)
    print(prec.value, "heatmap %", np.round(res.relative_perf, 1).tolist(), flush=True)
