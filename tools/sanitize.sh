#!/bin/bash
# compute-sanitizer passes over the hand-rolled mbarrier / TMEM / TMA
# pipelines (run on the GPU box; SURVEY §5 "build equivalent").
S=/usr/local/cuda/bin/compute-sanitizer
OUT=gpurun_out
$S --tool memcheck --leak-check no --error-exitcode 17 --print-limit 20 \
  python -m pytest tests/test_gemm_gpu.py tests/test_batched_gpu.py tests/test_splitk_gpu.py \
  tests/test_convgemm_gpu.py tests/test_netlib_gpu.py tests/test_tf32_gpu.py -q -p no:cacheprovider -x \
  -k "not large_sampled and not 4096" > $OUT/r2_memcheck.log 2>&1
echo "memcheck rc=$?"
tail -5 $OUT/r2_memcheck.log
$S --tool racecheck --racecheck-report hazard --error-exitcode 18 --print-limit 20 \
  python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r2_racecheck.log 2>&1
echo "racecheck rc=$?"
tail -8 $OUT/r2_racecheck.log
$S --tool synccheck --error-exitcode 19 --print-limit 20 \
  python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r2_synccheck.log 2>&1
echo "synccheck rc=$?"
tail -5 $OUT/r2_synccheck.log
