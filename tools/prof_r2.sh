#!/bin/bash
# ncu captures of the kernels furthest below roofline (run on the GPU box).
set -x
NCU="ncu --set full --import-source on --clock-control none"
B="python bench.py --steps 1 --warmup 3 --no-extra --no-cpu-baseline"
$NCU -k regex:hgemm_tc_small -c 1 -o gpurun_out/r2_h32 $B --workload batched_h32 > gpurun_out/r2_h32.log 2>&1
$NCU -k regex:splitk -c 1 -o gpurun_out/r2_hc3 $B --workload hgemm_c3 > gpurun_out/r2_hc3.log 2>&1
$NCU -k regex:sgemm_tma -c 1 -o gpurun_out/r2_sc1 $B --workload sgemm_c1 > gpurun_out/r2_sc1.log 2>&1
$NCU -k regex:hgemm_tc -c 1 -o gpurun_out/r2_hc3b $B --workload hgemm_c3b > gpurun_out/r2_hc3b.log 2>&1
for f in r2_h32 r2_hc3 r2_sc1 r2_hc3b; do
  ncu -i gpurun_out/$f.ncu-rep --page details --csv > gpurun_out/${f}_details.csv 2>/dev/null
  ncu -i gpurun_out/$f.ncu-rep --page source --csv --print-source sass > gpurun_out/${f}_sass.csv 2>/dev/null
done
ls -la gpurun_out/
