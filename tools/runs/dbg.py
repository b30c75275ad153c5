
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_1104_4475_b200 as tq
p, q, nb, tree, fam = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
m, n = p*nb, q*nb
A = torch.randn(m*n, dtype=torch.float64, device="cuda")
T = tq.tiled_qr(A, m, n, nb, 32, tree, 1, fam)
torch.cuda.synchronize()
print("ok", sys.argv[1:])
