"""Summarise per-case `ncu --set full` captures of tqr_persistent (one report per
bench.py case, the measured launch only) into one JSON (development aid).

    python tools/ncu_cases.py out.json "command text" case1=rep1.ncu-rep case2=rep2.ncu-rep ...
Keeps time, DRAM bytes, L1/L2 hit rates, registers, and every fp64 / dmma pipe
metric the raw page carries.
"""
import csv
import io
import json
import subprocess
import sys

out, cmd = sys.argv[1], sys.argv[2]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1,
         "second": 1e3}
FIXED = {"gpu__time_duration.sum": "gpu_time_ms", "dram__bytes_read.sum": "dram_read_bytes",
         "dram__bytes_write.sum": "dram_write_bytes", "lts__t_sector_hit_rate.pct": "l2_hit_pct",
         "l1tex__t_sector_hit_rate.pct": "l1_hit_pct", "launch__registers_per_thread": "registers_per_thread",
         "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
         "smsp__cycles_elapsed.avg.per_second": "sm_clock"}
res = {"command": cmd, "kernel": "tqr_persistent", "cases": {}}
for arg in sys.argv[3:]:
    name, rep = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    d = dict(zip(h, rows[-1]))
    c = {}
    for k, v in d.items():
        if k in FIXED or ("fp64" in k or "dmma" in k) and ("pct" in k or k.endswith(".sum")):
            try:
                x = float(v.replace(",", "")) * SCALE.get(units[h.index(k)], 1)
            except ValueError:
                continue
            c[FIXED.get(k, k)] = x
    if "dram_read_bytes" in c and "dram_write_bytes" in c:
        c["dram_bytes"] = c["dram_read_bytes"] + c["dram_write_bytes"]
    res["cases"][name] = c
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
