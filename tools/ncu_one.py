"""Warm-up + measured tiled_qr launches of one workload (for ncu captures).

    python tools/ncu_one.py [p q nb] [tree:bs:family,...]
Defaults: configs[2] (40 40 200) with the six bench.py cases. Each case runs a
warm-up launch and a measured launch (ncu: capture them all, keep the odd ones).
"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1104_4475_b200 as tq  # noqa: E402

a = sys.argv[1:]
p, q, nb = (int(x) for x in (a[:3] if len(a) >= 3 else (40, 40, 200)))
cases = (a[3] if len(a) > 3 else "greedy:1:TT,fibonacci:1:TT,flat:1:TT,greedy:1:TS,fibonacci:1:TS,flat:1:TS").split(",")
ib = 32
m, n = p * nb, q * nb
g = torch.Generator(device="cuda").manual_seed(0)
A0 = torch.randn(m * n, dtype=torch.float64, device="cuda", generator=g)
A = torch.empty_like(A0)
T = torch.zeros(tq.t_size(m, n, nb, ib), dtype=torch.float64, device="cuda")
for c in cases:
    tree, bs, fam = (c.split(":") + ["1", "TT"])[:3]
    for _ in range(2):
        A.copy_(A0)
        tq.tiled_qr(A, m, n, nb, ib, tree, int(bs), fam, T=T)
torch.cuda.synchronize()
print("ok", p, q, nb, cases)
