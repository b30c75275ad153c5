"""profiles/ncu_full_summary_square.json (the file bench.py reads roofline.traffic from) and a
launch-list summary from one closing run's scratch output (development aid).

    python tools/ncu_square_summary.py gpurun_out/<prefix>_ncu_cases.json gpurun_out/<prefix>_launches.csv "<build note>"
"""
import collections
import csv
import json
import sys

cases, launches, note = sys.argv[1], sys.argv[2], sys.argv[3]
raw = json.load(open(cases))
out = {"command": raw["command"], "kernel": raw["kernel"], "cases": {}}
tot = tms = 0.0
for k, c in raw["cases"].items():
    dm = c.get("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active")
    ops = [v for kk, v in c.items() if kk.startswith("sm__ops_path_tensor_src_fp64") and "pct" in kk]
    out["cases"][k] = {"gpu_time_ms": round(c["gpu_time_ms"], 3), "dram_read_GB": round(c["dram_read_bytes"] / 1e9, 3),
                       "dram_write_GB": round(c["dram_write_bytes"] / 1e9, 3), "l2_hit_pct": round(c["l2_hit_pct"], 2),
                       "l1_hit_pct": round(c["l1_hit_pct"], 2), "dmma_pipe_active_pct": round(dm, 2),
                       "fp64_tensor_ops_pct_of_peak": round(ops[0], 2) if ops else None,
                       "registers_per_thread": int(c["registers_per_thread"])}
    tot += c["dram_read_bytes"] + c["dram_write_bytes"]
    tms += c["gpu_time_ms"]
n = len(raw["cases"])
out["dram_bytes_per_launch"] = tot / n
out["algorithmic_bytes"] = 1187840000   # A read and written once (2 x 512 MB) + T written (164 MB)
out["gpu_time_ms_mean"] = tms / n
out["note"] = ("one full capture per bench.py case (the measured launch after a warm-up), " + note +
               ". dram_bytes_per_launch = mean over the cases; the DRAM excess over the algorithmic bytes is every "
               "update strip writing its C strip back and re-reading its V tile, which the 126 MB L2 cannot keep "
               "for a 512 MB matrix. Raw per-case metrics: " + cases + " (scratch).")
json.dump(out, open("profiles/ncu_full_summary_square.json", "w"), indent=1)

lines = [l for l in open(launches) if not l.startswith("==")]
agg = collections.OrderedDict()
for row in csv.DictReader(lines):
    if row.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v, u = float(row["Metric Value"].replace(",", "")), row["Metric Unit"]
    ms = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
    a = agg.setdefault(row["Kernel Name"], [0, 0.0])
    a[0] += 1
    a[1] += ms
t = sum(a[1] for a in agg.values())
o = ["ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 (" + note +
     "; cold-cache, serialised; raw: r02_launches_session5.csv)"]
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    o.append(f"{a[0]:6d} launches {a[1]:11.2f} ms {100 * a[1] / t:5.1f}%  {k[:100]}")
open("profiles/r02_launches_session5_summary.txt", "w").write("\n".join(o) + "\n")
print(o[1])
for k, c in out["cases"].items():
    print(k, c)
