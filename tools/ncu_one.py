"""One warm-up + one timed tiled_qr launch of configs[1] (for ncu captures).

    python tools/ncu_one.py [tree] [bs]
"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1104_4475_b200 as tq  # noqa: E402

tree = sys.argv[1] if len(sys.argv) > 1 else "greedy"
bs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p, q, nb, ib = 40, 10, 200, 32
m, n = p * nb, q * nb
g = torch.Generator(device="cuda").manual_seed(0)
A0 = torch.randn(m * n, dtype=torch.float64, device="cuda", generator=g)
A = torch.empty_like(A0)
T = torch.zeros(tq.t_size(m, n, nb, ib), dtype=torch.float64, device="cuda")
for _ in range(2):
    A.copy_(A0)
    tq.tiled_qr(A, m, n, nb, ib, tree, bs, "TT", T=T)
torch.cuda.synchronize()
print("ok", tree, bs)
