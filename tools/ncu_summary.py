"""Summarise an ncu report (raw page) into per-kernel JSON (dev tool).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/x.json
"""
import csv, io, json, subprocess, sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "%": 1, "": 1,
         "byte/second": 1, "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/second": 1e9, "Tbyte/second": 1e12}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active"]

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = []
for r in rows[2:]:
    d = {"kernel": r[hdr.index("Kernel Name")]}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            try:
                d[k] = float(r[i]) * UNITS.get(units[i], 1)
            except ValueError:
                d[k] = r[i]
    if "dram__bytes_read.sum" in d:
        d["dram_bytes_per_launch"] = d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0)
    out.append(d)
json.dump(out, sys.stdout, indent=1)
print()
