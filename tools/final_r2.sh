#!/bin/bash
# Round-2 measurement pass (GPU box): full GPU tests, the driver's bench
# command, the ncu launch list of the same command, and the sweep JSON.
# Usage: tools/final_r2.sh [prefix]   (output files gpurun_out/<prefix>_*)
P=${1:-r2f}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?"
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${P}_gputest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${P}_gputest.log
python bench.py --steps 20 --warmup 5 --sweep-out gpurun_out/${P}_c2_sweep.json > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches_hgemm8192.csv \
  python bench.py --steps 3 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/${P}_ncu_launch.log 2>&1; echo "ncu rc=$?"
