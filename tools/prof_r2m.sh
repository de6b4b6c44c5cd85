#!/bin/bash
# ncu --set full of the 256x512 pair kernel on the headline and on C5 (GPU box).
NCU="ncu --set full --import-source on --clock-control none"
B="python bench.py --steps 1 --warmup 3 --no-extra --no-cpu-baseline"
$NCU -k regex:2sm -c 1 -o gpurun_out/r2m_h8192 $B --workload hgemm > /dev/null 2>&1; echo "h8192 rc=$?"
$NCU -k regex:2sm -c 1 -o gpurun_out/r2m_hc5 $B --workload hgemm_c5 > /dev/null 2>&1; echo "hc5 rc=$?"
for f in r2m_h8192 r2m_hc5; do
  ncu -i gpurun_out/$f.ncu-rep --page details --csv > gpurun_out/${f}_details.csv 2>/dev/null
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out/r2m_h*
