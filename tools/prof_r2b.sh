#!/bin/bash
# ncu captures of the round-2 kernels (GPU box); summaries go to profiles/.
NCU="ncu --set full --import-source on --clock-control none"
B="python bench.py --steps 1 --warmup 3 --no-extra --no-cpu-baseline"
$NCU -k regex:small32 -c 1 -o gpurun_out/r2b_h32 $B --workload batched_h32 > /dev/null 2>&1
$NCU -k regex:splitk -c 1 -o gpurun_out/r2b_hc3 $B --workload hgemm_c3 > /dev/null 2>&1
$NCU -k regex:sgemm_tma -c 1 -o gpurun_out/r2b_sc3 $B --workload sgemm_c3 > /dev/null 2>&1
$NCU -k regex:2sm -c 1 -o gpurun_out/r2b_hc5 $B --workload hgemm_c5 > /dev/null 2>&1
$NCU -k regex:hgemm_tc_kernel -c 1 -o gpurun_out/r2b_conv python tools/conv_probe.py > /dev/null 2>&1
for f in r2b_h32 r2b_hc3 r2b_sc3 r2b_hc5 r2b_conv; do
  ncu -i gpurun_out/$f.ncu-rep --page details --csv > gpurun_out/${f}_details.csv 2>/dev/null
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$f.ncu-rep --page source --csv --print-source sass > gpurun_out/${f}_sass.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out/r2b_*
