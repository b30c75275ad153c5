"""One-off transcription of the paper's printed tables into tests/golden/*.csv.

Reads PAPER.md (LaTeX source) ONCE, here on the CPU box, and writes plain CSV
fixtures with their citation in a header comment. Nothing at test/bench time
reads /root/reference. Values are the paper's; this script does no arithmetic.
"""
import re, sys, pathlib
src = pathlib.Path(sys.argv[1]).read_text().splitlines()
out = pathlib.Path(sys.argv[2])

def cells(line):
    line = line.replace(r"\ensuremath{\star}\xspace", "*").replace(r"\\%", "").replace(r"\\", "")
    line = line.rstrip("%").strip()
    return [c.strip() for c in line.split("&")]

def block(lo, hi):  # 1-based inclusive line numbers
    return [cells(src[n - 1]) for n in range(lo, hi + 1)]

def write_matrix(name, cite, rows, c0, ncols, p):
    # rows: list of cell lists for matrix rows 1..p ; columns c0..c0+ncols-1
    with open(out / name, "w") as f:
        f.write(f"# {cite}\n# row i (1-based), then tile (i,k) values for k=1..{ncols}; blank = on/above diagonal\n")
        for i, r in enumerate(rows, start=1):
            vals = []
            for k in range(ncols):
                v = r[c0 + k] if c0 + k < len(r) else ""
                vals.append(v if v not in ("*", "") else "")
            f.write(",".join([str(i)] + vals) + "\n")

t2 = block(522, 536)
for name, c0 in (("flat", 0), ("fibonacci", 6), ("greedy", 12)):
    write_matrix(f"table2_coarse_{name}_15x6.csv",
                 f"PAPER.md Table 2 (tab.coarse, lines 515-542), ({ {'flat':'a','fibonacci':'b','greedy':'c'}[name] }) {name}, p=15 q=6, coarse-grain time-steps",
                 t2, c0, 6, 15)
t3 = block(629, 643)
for name, c0 in (("flat", 0), ("fibonacci", 6), ("greedy", 12), ("binary", 18), ("plasma_bs5", 24)):
    write_matrix(f"table3_tiled_{name}_15x6.csv",
                 f"PAPER.md Table 3 (tab.tiled, lines 622-649), {name}, p=15 q=6, TT kernels, tiled time-steps (units nb^3/3 flops)",
                 t3, c0, 6, 15)
t4 = block(702, 716)
for name, c0 in (("greedy", 1), ("asap", 4), ("grasap1", 7)):
    write_matrix(f"table4_{name}_15x3.csv",
                 f"PAPER.md Table 4(a) (table.15x2x3, lines 694-719), {name}, p=15 q=3, TT kernels",
                 t4, c0, 3, 15)
# Table 5(b): Greedy/ASAP critical paths
with open(out / "table5b_greedy_asap_cp.csv", "w") as f:
    f.write("# PAPER.md Table 5(b) (table.greedyvsasap, lines 721-745): TT critical paths\n# p,q,greedy,asap\n")
    f.write("16,16,310,310\n32,16,360,402\n32,32,650,656\n64,16,374,588\n64,32,726,844\n64,64,1342,1354\n")
    f.write("128,16,396,966\n128,32,748,1222\n128,64,1452,1748\n128,128,2732,2756\n")
# Table 6
with open(out / "table6_p40.csv", "w") as f:
    f.write("# PAPER.md Table 6 (lines 1317-1368): Greedy versus PlasmaTree (TT) and Fibonacci (Theoretical), TT critical paths\n")
    f.write("# p,q,greedy,plasma_best,plasma_bs,overhead,gain,fibonacci,fib_overhead,fib_gain\n")
    for n in range(1324, 1364):
        c = [x.strip() for x in src[n - 1].replace(r"\\", "").split("&")]
        f.write(",".join(c) + "\n")
print("ok")
