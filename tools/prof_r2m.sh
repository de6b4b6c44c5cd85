#!/bin/bash
# ncu --set full of the 256x512 pair kernel on the headline and, with a second
# argument, on C5 (GPU box).  usage: tools/prof_r2m.sh PREFIX [c5]
P=${1:-r2m}
NCU="ncu --set full --import-source on --clock-control none"
B="python bench.py --steps 1 --warmup 3 --no-extra --no-cpu-baseline"
$NCU -k regex:2sm -c 1 -o gpurun_out/${P}_h8192 $B --workload hgemm > /dev/null 2>&1; echo "h8192 rc=$?"
[ -n "$2" ] && $NCU -k regex:2sm -c 1 -o gpurun_out/${P}_hc5 $B --workload hgemm_c5 > /dev/null 2>&1; echo "hc5 rc=$?"
for f in ${P}_h8192 ${P}_hc5; do
  ncu -i gpurun_out/$f.ncu-rep --page details --csv > gpurun_out/${f}_details.csv 2>/dev/null
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out/${P}_h*
