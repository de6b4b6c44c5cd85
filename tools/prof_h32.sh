ncu --set full --import-source on --clock-control none -k regex:small32 -c 1 -o gpurun_out/r2n_h32 python bench.py --steps 1 --warmup 3 --no-extra --no-cpu-baseline --workload batched_h32 > /dev/null 2>&1; echo rc=$?
ncu -i gpurun_out/r2n_h32.ncu-rep --page details --csv > gpurun_out/r2n_h32_details.csv 2>/dev/null
ncu -i gpurun_out/r2n_h32.ncu-rep --page raw --csv > gpurun_out/r2n_h32_raw.csv 2>/dev/null
ncu -i gpurun_out/r2n_h32.ncu-rep --page source --csv --print-source sass > gpurun_out/r2n_h32_sass.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
