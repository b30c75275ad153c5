"""Warp-stall samples of an ncu --set full --import-source capture, summed per
CUDA source line (development aid; needs the same build's -lineinfo).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = next(r for r in rows if len(r) > 3 and r[0] == "Line No")
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
col = {k: h.index(k) for k in stalls}


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


per, src, reasons = {}, {}, {}
cur_file, cur = None, None
total = 0.0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) != len(h) or r[0] == "Line No":
        continue
    if r[0]:
        cur = (cur_file, int(r[0]))
        src[cur] = r[1].strip()
    v = {k: num(r[c]) for k, c in col.items()}
    s = sum(v.values())
    total += s
    if cur:
        per[cur] = per.get(cur, 0.0) + s
        d = reasons.setdefault(cur, {})
        for k, x in v.items():
            d[k] = d.get(k, 0.0) + x
print(f"{rep}: {total:.0f} warp-state samples")
for key, s in sorted(per.items(), key=lambda x: -x[1])[:top]:
    rs = sorted(reasons[key].items(), key=lambda x: -x[1])[:2]
    print(f"{s / total * 100:5.2f}%  {key[0]}:{key[1]:<5d} {src.get(key, '')[:70]:70s} "
          + " ".join(f"{k[6:]}={x / total * 100:.1f}" for k, x in rs))
