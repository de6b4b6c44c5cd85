"""On-device tuning of the BASELINE shapes over the gemm_b200 family + the
problem-specific-tuning heat map (paper Fig. 4) on the B200.  Writes
gpurun_out/r2_tuning_db.json, gpurun_out/r2_tuning_summary.json and
gpurun_out/r2_heatmap_*.json.  Dev tool; uses only the public API."""
import json
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.kernels.params import is_b200_auto  # noqa: E402
from paper_1705_05249_b200.tuner import TuningTask, tune  # noqa: E402

ctx = tb.context_create(tb.host_device())
db = tb.Database()
summary = []
shapes = [(64, 3136, 576), (4096, 128, 9216), (1024, 1024, 1024), (8192, 8192, 8192)]
for prec in (tb.Precision.H, tb.Precision.S):
    for (m, n, k) in shapes:
        t0 = time.perf_counter()
        big = m * n * k > 1e11
        task = TuningTask("gemm_b200", prec, {"m": m, "n": n, "k": k}, ctx.device, budget=0,
                          warmup_runs=1, timed_runs=3 if (big and prec is tb.Precision.S) else (5 if big else 10))
        run = tune(task, ctx)
        tb.db_insert(db, run)
        ok = [x for x in run.measurements if x.status == "ok"]
        best = min(ok, key=lambda x: x.mean_time)
        auto = [x for x in ok if is_b200_auto(x.configuration)]
        kernels = sorted({x.kernel for x in ok})
        per_kernel = {}
        for x in ok:
            per_kernel[x.kernel] = min(per_kernel.get(x.kernel, 1e9), x.mean_time * 1e6)
        row = dict(precision=prec.value, m=m, n=n, k=k, explored=len(run.measurements), ok=len(ok),
                   best_us=best.mean_time * 1e6, best_kernel=best.kernel, best=run.best.as_dict(),
                   auto_us=auto[0].mean_time * 1e6 if auto else None,
                   auto_kernel=auto[0].kernel if auto else None,
                   gflops_best=2 * m * n * k / best.mean_time / 1e9,
                   distinct_kernels=len(kernels), best_us_per_kernel=per_kernel,
                   failed=[x.configuration.as_dict() for x in run.measurements if x.status != "ok"],
                   seconds=time.perf_counter() - t0)
        summary.append(row)
        print(json.dumps({k_: v for k_, v in row.items() if k_ not in ("best", "best_us_per_kernel")}),
              flush=True)
db.save("gpurun_out/r2_tuning_db.json")
json.dump(summary, open("gpurun_out/r2_tuning_summary.json", "w"), indent=1)
for prec in (tb.Precision.S, tb.Precision.H):
    res = tb.heatmap_experiment([(64, 3136, 576), (4096, 128, 9216), (1024, 1024, 1024)], prec, ctx,
                                budget=0, seed=5, runs=5)
    json.dump(res.to_json(), open(f"gpurun_out/r2_heatmap_{prec.value}.json", "w"), indent=1)
    print(prec.value, "heatmap %", np.round(res.relative_perf, 1).tolist(), flush=True)
