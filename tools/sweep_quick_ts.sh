for fam in TT TS; do
for spec in greedy:1 flat:1 plasma:5 plasma:10; do
  python - "$spec" "$fam" <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1104_4475_b200 as tq
tree, bs = sys.argv[1].split(':'); bs = int(bs); fam = sys.argv[2]
p, q, nb, ib = 40, 10, 200, 32
m, n = p * nb, q * nb
g = torch.Generator(device='cuda').manual_seed(0)
A0 = torch.randn(m * n, dtype=torch.float64, device='cuda', generator=g)
A = torch.empty_like(A0); T = torch.zeros(tq.t_size(m, n, nb, ib), dtype=torch.float64, device='cuda')
ts = []
for it in range(5):
    A.copy_(A0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); tq.tiled_qr(A, m, n, nb, ib, tree, bs, fam, T=T); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
best = min(ts[1:])
print(f"{tree}:{bs} {fam}: {best:.3f} ms {2.0*n*n*(m-n/3.0)/best/1e9:.2f} TFLOP/s")
PY
done; done
