"""Per-task trace of one tiled_qr launch: durations per kernel kind, waiting,
SM utilisation (development aid; uses the library's diagnostic tracer).

    python tools/trace_report.py [p q nb ib tree[:bs] [out.npy]]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1104_4475_b200 as tq  # noqa: E402

a = sys.argv[1:]
p, q, nb, ib = (int(x) for x in (a[:4] if len(a) >= 4 else (40, 10, 200, 32)))
spec = (a[4] if len(a) > 4 else "greedy").split(":")
tree, bs = spec[0], int(spec[1]) if len(spec) > 1 else 1
family = spec[2] if len(spec) > 2 else "TT"
m, n = p * nb, q * nb
g = torch.Generator(device="cuda").manual_seed(0)
A0 = torch.randn(m * n, dtype=torch.float64, device="cuda", generator=g)
A = torch.empty_like(A0)
T = torch.zeros(tq.t_size(m, n, nb, ib), dtype=torch.float64, device="cuda")
for it in range(3):
    A.copy_(A0)
    if it == 2:
        tq.trace_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tq.tiled_qr(A, m, n, nb, ib, tree, bs, family, T=T)
    e1.record()
    torch.cuda.synchronize()
tq.trace_enable(False)
ms = e0.elapsed_time(e1)
tr = tq.trace_fetch()
if len(a) > 5:
    np.save(a[5], tr)
t0 = tr["taken"].min()
span = (tr["done"].max() - t0) / 1e3
run = (tr["done"] - tr["ready"]) / 1e3
wait = (tr["ready"] - tr["taken"]) / 1e3
nsm = len(np.unique(tr["sm"]))
print(f"{tree}:{bs}:{family} p={p} q={q} nb={nb} ib={ib}: event {ms:.3f} ms, traced span {span / 1e3:.3f} ms, "
      f"{len(tr)} tasks on {nsm} SMs")
print(f"  busy (sum run) / (SMs x span) = {run.sum() / (nsm * span):.3f};  waiting share = {wait.sum() / (nsm * span):.3f}")
unit = nb ** 3 / 3.0
W = {0: 4, 1: 6, 2: 2, 3: 6, 4: 6, 5: 12}
S = -(-nb // 32) if nb > 32 else 1
for kd in np.unique(tr["kind"]):
    sel = tr["kind"] == kd
    r = run[sel]
    fl = W.get(int(kd), 0) * unit / (S if kd in (1, 3, 5) else 1)
    print(f"  {tq.KIND_NAMES[kd]:8s} n={sel.sum():6d} run mean {r.mean():8.2f} us  p50 {np.median(r):8.2f}  "
          f"max {r.max():8.2f}  sum {r.sum() / 1e3:8.2f} ms  ~{fl / (r.mean() * 1e3):6.1f} GFLOP/s/SM   "
          f"wait mean {wait[sel].mean():7.2f} us")
    cyc = {p: tr[f"c_{p}"][sel].mean() for p in tq.PHASES}
    tot = sum(cyc.values())
    print("           phases (kcycles/task): " + "  ".join(f"{p}={cyc[p] / 1e3:.1f}" for p in tq.PHASES if cyc[p] > 0)
          + f"  total={tot / 1e3:.1f}")
# critical chain: walk back from the last-finishing task through the latest-finishing... (approx: by time)
order = np.argsort(tr["ready"])
first = (tr["ready"] - t0) / 1e3
print(f"  tasks started in first 10% of span: {(first < 0.1 * span).sum()}, last 10%: {(first > 0.9 * span).sum()}")

# critical path of the executed graph with the measured task durations (unbounded SMs)
ptr, idx = tq.trace_graph(len(tr))
dur = (tr["done"] - tr["ready"]) / 1e3
fin = np.zeros(len(tr))
start = np.zeros(len(tr))
for t in range(len(tr)):          # tasks are in a topological order
    fin[t] = start[t] + dur[t]
    for x in range(ptr[t], ptr[t + 1]):
        sc = idx[x]
        if fin[t] > start[sc]:
            start[sc] = fin[t]
cp = fin.max()
print(f"  critical path with measured durations: {cp / 1e3:.3f} ms (span {span / 1e3:.3f} ms, "
      f"work/SMs {run.sum() / nsm / 1e3:.3f} ms)")
# kinds on the critical path
t = int(np.argmax(fin))
path = []
pred = {}
for u in range(len(tr)):
    for x in range(ptr[u], ptr[u + 1]):
        sc = idx[x]
        if abs(fin[u] - start[sc]) < 1e-9:
            pred.setdefault(sc, u)
while True:
    path.append(t)
    if t not in pred:
        break
    t = pred[t]
kinds = {}
for u in path:
    k = tq.KIND_NAMES[tr["kind"][u]]
    kinds[k] = kinds.get(k, 0) + dur[u]
print("  critical path composition (ms): " + ", ".join(f"{k} {v / 1e3:.2f}" for k, v in sorted(kinds.items(), key=lambda x: -x[1])))
# utilisation over time (busy SMs per 5% of the span) and what runs
nb_ = 20
edges = np.linspace(0, span, nb_ + 1)
rs, rd = (tr["ready"] - t0) / 1e3, (tr["done"] - t0) / 1e3
util = []
for b in range(nb_):
    lo, hi = edges[b], edges[b + 1]
    ov = np.clip(np.minimum(rd, hi) - np.maximum(rs, lo), 0, None)
    util.append(ov.sum() / ((hi - lo) * nsm))
print("  busy fraction per 5% of span: " + " ".join(f"{u:.2f}" for u in util))
panel = np.isin(tr["kind"], [9, 11, 13])
cpb = []
for b in range(nb_):
    lo, hi = edges[b], edges[b + 1]
    ov = np.clip(np.minimum(rd, hi) - np.maximum(rs, lo), 0, None)
    cpb.append((ov * panel).sum() / (hi - lo))
print("  concurrent panel tasks per 5%:   " + " ".join(f"{u:4.1f}" for u in cpb))
# executed critical chain: from the last task back through the predecessor that finished last;
# split into execution time and queueing delay (inputs ready -> task started)
preds = [[] for _ in range(len(tr))]
for u in range(len(tr)):
    for x in range(ptr[u], ptr[u + 1]):
        preds[idx[x]].append(u)
t = int(np.argmax(tr["done"]))
exe = que = 0.0
nchain = 0
kinds_e, kinds_q = {}, {}
while True:
    nchain += 1
    k = tq.KIND_NAMES[tr["kind"][t]]
    d = (tr["done"][t] - tr["ready"][t]) / 1e3
    exe += d
    kinds_e[k] = kinds_e.get(k, 0) + d
    if not preds[t]:
        que += (tr["ready"][t] - t0) / 1e3
        break
    u = max(preds[t], key=lambda z: tr["done"][z])
    q_ = max(0.0, (tr["ready"][t] - tr["done"][u]) / 1e3)
    que += q_
    kinds_q[k] = kinds_q.get(k, 0) + q_
    t = u
print(f"  executed chain: {nchain} tasks, execution {exe / 1e3:.3f} ms + queueing {que / 1e3:.3f} ms")
print("   exec by kind (ms): " + ", ".join(f"{k} {v / 1e3:.2f}" for k, v in sorted(kinds_e.items(), key=lambda x: -x[1])))
print("   queue by kind (ms): " + ", ".join(f"{k} {v / 1e3:.2f}" for k, v in sorted(kinds_q.items(), key=lambda x: -x[1])))
if len(a) > 6 and a[6] == "chain":
    t = int(np.argmax(tr["done"]))
    rows = []
    while True:
        rows.append(t)
        if not preds[t]:
            break
        t = max(preds[t], key=lambda z: tr["done"][z])
    for t in reversed(rows):
        u = max(preds[t], key=lambda z: tr["done"][z]) if preds[t] else None
        rdy = (tr["done"][u] - t0) / 1e3 if u is not None else 0.0
        pushed = (tr["c_store"][t] - t0) / 1e3 if tr["c_store"][t] > 0 else float("nan")
        print(f"   {tq.KIND_NAMES[tr['kind'][t]]:8s} i={tr['i'][t]:2d} piv={tr['piv'][t]:2d} k={tr['k'][t]} j={tr['j'][t]} s={tr['s'][t]} "
              f"inputs {rdy:8.1f} pushed {pushed:8.1f} start {(tr['ready'][t] - t0) / 1e3:8.1f} done {(tr['done'][t] - t0) / 1e3:8.1f} us")
