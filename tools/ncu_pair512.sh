M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed
for v in 256 512; do
ncu --metrics $M --clock-control none -k regex:2sm -c 3 --csv python tools/one_gemm.py 8192 $v 8 3 2>/dev/null | grep -v "^==" > gpurun_out/ncu512_$v.csv
done
python - <<'P'
import csv
for v in (256, 512):
    rows = list(csv.DictReader(open(f"gpurun_out/ncu512_{v}.csv")))
    for r in rows:
        print(v, r["ID"], r["Metric Name"], r["Metric Value"], r["Metric Unit"])
P
