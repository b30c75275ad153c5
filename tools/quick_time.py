"""Quick device timing of tiled_qr for one shape and tree (development aid)."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1104_4475_b200 as tq  # noqa: E402

p, q, nb, ib = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (40, 10, 200, 32)))
trees = sys.argv[5].split(",") if len(sys.argv) > 5 else ["greedy", "fibonacci", "flat", "plasma:5"]
m, n = p * nb, q * nb
g = torch.Generator(device="cuda").manual_seed(0)
A0 = torch.randn(m * n, dtype=torch.float64, device="cuda", generator=g)
A = torch.empty_like(A0)
T = torch.empty(tq.t_size(m, n, nb, ib), dtype=torch.float64, device="cuda")
flops = 2.0 * n * n * (m - n / 3.0)
for spec in trees:
    parts = spec.split(":")
    tree, bs, fam = parts[0], parts[1] if len(parts) > 1 else "1", parts[2] if len(parts) > 2 else "TT"
    bs = int(bs)
    ts = []
    for it in range(5):
        A.copy_(A0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tq.tiled_qr(A, m, n, nb, ib, tree, bs, fam, T=T)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    best = min(ts[1:])
    print(f"{tree}:{bs}:{fam} p={p} q={q} nb={nb}: {best:.3f} ms  {flops / best / 1e9:.1f} TFLOP/s  (all {['%.2f' % t for t in ts]})",
          flush=True)
