set -x
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
for rep in 1 2; do for lib in main st4; do
  if [ $lib = main ]; then L=""; else L="TBGEMM_LIB=ab/st4.so"; fi
  env $L python bench.py --workload hgemm_c3 --steps 50 --warmup 5 --no-extra --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['kernel'], d['ms_per_step'])"
done; done > gpurun_out/ab_c3.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_hgemm.csv python bench.py --workload hgemm --steps 2 --warmup 3 --no-extra --no-cpu-baseline > /tmp/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:hgemm_tc_small -s 3 -c 1 -o /tmp/h32 python bench.py --workload batched_h32 --steps 2 --warmup 3 --no-extra --no-cpu-baseline > /tmp/ncu2.log 2>&1
ncu -i /tmp/h32.ncu-rep --page details --csv > gpurun_out/final_h32_details.csv 2>&1
ncu -i /tmp/h32.ncu-rep --page raw --csv > gpurun_out/final_h32_raw.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:sgemm_tma -s 3 -c 1 -o /tmp/s1 python bench.py --workload sgemm_c1 --steps 2 --warmup 3 --no-extra --no-cpu-baseline > /tmp/ncu3.log 2>&1
ncu -i /tmp/s1.ncu-rep --page details --csv > gpurun_out/final_sc1_details.csv 2>&1
ncu -i /tmp/s1.ncu-rep --page raw --csv > gpurun_out/final_sc1_raw.csv 2>&1
ncu --set full --clock-control none -k regex:hgemm_tc_splitk -s 3 -c 1 -o /tmp/c3 python bench.py --workload hgemm_c3 --steps 2 --warmup 3 --no-extra --no-cpu-baseline > /tmp/ncu4.log 2>&1
ncu -i /tmp/c3.ncu-rep --page details --csv > gpurun_out/final_hc3_details.csv 2>&1
ls -la gpurun_out; cat gpurun_out/ab_c3.txt
