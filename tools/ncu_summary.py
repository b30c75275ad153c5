"""Summarise one `ncu --set full` capture of tqr_persistent into the JSON that
bench.py reads for roofline.traffic (development aid).

    python tools/ncu_summary.py report.ncu-rep out.json "command text" [every]
With several captured launches, the per-launch figures are means over launches
every-1, 2*every-1, ... (tools/ncu_one.py: warm-up + measured launch per case, every = 2).
"""
import csv
import io
import json
import subprocess
import sys

rep, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
every = int(sys.argv[4]) if len(sys.argv) > 4 else 1
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
launches = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
keep = launches[every - 1::every]


def val(name):
    u = units[h.index(name)]
    v = sum(float(d[name].replace(",", "")) for d in keep) / len(keep)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1,
             "second": 1e3, "cycle/nsecond": 1, "cycle/usecond": 1e-3, "Ghz": 1, "Mhz": 1e-3}
    return v * scale.get(u, 1)


s = {
    "command": cmd,
    "kernel": "tqr_persistent",
    "gpu_time_ms": val("gpu__time_duration.sum"),
    "dram_bytes_read": val("dram__bytes_read.sum"),
    "dram_bytes_write": val("dram__bytes_write.sum"),
    "sm_clock_ghz": val("smsp__cycles_elapsed.avg.per_second"),
    "sm_throughput_pct": val("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "registers_per_thread": val("launch__registers_per_thread"),
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active":
        val("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active")
        if "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active" in h else None,
}
s["dram_bytes_per_launch"] = s["dram_bytes_read"] + s["dram_bytes_write"]
s["launches_averaged"] = len(keep)
json.dump(s, open(out, "w"), indent=1)
print(json.dumps(s, indent=1))
