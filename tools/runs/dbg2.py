import os, sys, subprocess
code = r'''
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_1104_4475_b200 as tq
p, q, nb, tree, fam = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
m, n = p*nb, q*nb
A = torch.randn(m*n, dtype=torch.float64, device="cuda")
T = tq.tiled_qr(A, m, n, nb, 32, tree, 1, fam)
torch.cuda.synchronize()
print("ok", sys.argv[1:])
'''
open("/tmp/dbg.py", "w").write(code)
for tma in ("0", "1"):
    for args in [("2", "1", "64", "greedy", "TT"), ("2", "2", "64", "greedy", "TT"), ("2", "2", "64", "greedy", "TS"),
                 ("3", "3", "96", "greedy", "TT"), ("4", "2", "200", "greedy", "TT")]:
        env = dict(os.environ, TQR_TMA=tma)
        try:
            r = subprocess.run([sys.executable, "/tmp/dbg.py", *args], env=env, capture_output=True, text=True, timeout=40)
            print("TMA", tma, args, "->", r.stdout.strip()[-80:], r.stderr.strip()[-200:], flush=True)
        except subprocess.TimeoutExpired:
            print("TMA", tma, args, "-> HANG", flush=True)
