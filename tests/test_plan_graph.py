"""Host checks (no GPU) of the device task graph the persistent kernel runs
(csrc/dag.cpp build_factor_graph + finalize_dataflow), read through the
diagnostic C entry point tqr_plan_graph:

* the priority order is topological and the indegrees match the successor lists;
* panel chains P(b) -> U(b, b+1) -> P(b+1) are successor edges with the chain
  bit set on the target;
* every pair of tasks that write the same (tile, column strip) is ordered by the
  graph (so the dataflow execution is race-free), and every reader of a panel
  block's reflectors runs after the panel task that produced them;
* the task counts follow from the tile-level DAG of Algorithms 2-3 (oracle/dag).
"""
import numpy as np
import pytest

import paper_1104_4475_b200 as tq
from oracle import dag, schemes


def reach(ptr, succ):
    """Transitive closure as Python int bitsets (tasks are in topological order)."""
    n = len(ptr) - 1
    r = [0] * n
    for t in range(n - 1, -1, -1):
        b = 0
        for x in range(ptr[t], ptr[t + 1]):
            s = int(succ[x])
            b |= (1 << s) | r[s]
        r[t] = b
    return r


def writes(t, nb, ib, ws):
    """(tile, strip) slots a task writes; strips are ws columns wide."""
    kind, i, piv, k, j, s = (int(x) for x in t[:6])
    s, ns = s & 0xffff, max(s >> 16, 1)        # multi-strip update tasks: strips s .. s + ns - 1
    name = tq.KIND_NAMES[kind]
    strips_of_block = lambda b: {(b * ib) // ws}
    if name in ("GEQRT_B",):
        return {((i, k), x) for x in strips_of_block(s)}
    if name in ("TTQRT_B", "TSQRT_B"):
        return {((i, k), x) for x in strips_of_block(s)} | {((piv, k), x) for x in strips_of_block(s)}
    if name == "GEQRT_U":
        return {((i, k), s)}
    if name in ("TTQRT_U", "TSQRT_U"):
        return {((i, k), s), ((piv, k), s)}
    if name == "UNMQR":
        return {((i, j), s + u) for u in range(ns)}
    if name in ("TTMQR", "TSMQR", "UNTTMQR"):
        return {((i, j), s + u) for u in range(ns)} | {((piv, j), s + u) for u in range(ns)}
    if name == "GEQRT":
        return {((i, k), x) for x in range(-(-nb // ws))}
    if name in ("TTQRT", "TSQRT"):
        return {((i, k), x) for x in range(-(-nb // ws))} | {((piv, k), x) for x in range(-(-nb // ws))}
    raise AssertionError(name)


CASES = [("greedy", 1, "TT"), ("flat", 1, "TS"), ("fibonacci", 1, "TT"), ("binary", 1, "TT"), ("plasma", 2, "TT"),
         ("plasma", 3, "TS")]


def fused_pairs(tiles):
    """UNMQR(i,k,j) whose next task on tile (i,j), in emission order, is the
    TTMQR(i,piv,k,j) eliminating the same row: these run as one UNTTMQR task."""
    last, pairs = {}, 0
    for t in tiles:
        if t.kind == "GEQRT":
            touched = [(t.i, t.k)]
        elif t.kind == "UNMQR":
            touched = [(t.i, t.j)]
        elif t.kind in ("TTQRT", "TSQRT"):
            touched = [(t.i, t.k), (t.piv, t.k)]
        else:
            touched = [(t.i, t.j), (t.piv, t.j)]
        for tile in touched:
            u = last.get(tile)
            if (u is not None and tile == (t.i, t.j) and u.kind == "UNMQR" and t.kind == "TTMQR"
                    and (u.i, u.k, u.j) == (t.i, t.k, t.j)):
                pairs += 1
            last[tile] = t
    return pairs


@pytest.mark.parametrize("tree,bs,family", CASES)
@pytest.mark.parametrize("p,q,nb,split,mstrip,fuse", [(6, 3, 72, True, 1, False), (6, 3, 72, True, 1, True),
                                                       (6, 3, 72, True, 2, True), (5, 2, 64, True, 2, True),
                                                       (4, 4, 64, False, 1, True), (4, 3, 200, True, 3, True),
                                                       (4, 3, 200, True, 3, False)])
def test_plan_graph_invariants(tree, bs, family, p, q, nb, split, mstrip, fuse):
    ib = ws = 32
    tasks, ptr, succ = tq.plan_graph(p * nb, q * nb, nb, ib, tree, bs, family, ws, split, mstrip, fuse)
    n = len(tasks)
    # topological priority order and indegrees
    indeg = np.zeros(n, np.int64)
    for t in range(n):
        for x in range(ptr[t], ptr[t + 1]):
            assert succ[x] > t
            indeg[succ[x]] += 1
    assert np.array_equal(indeg, tasks[:, 7] & 0xFFFF)
    # chains
    for t in range(n):
        c = int(tasks[t, 6])
        if c >= 0:
            assert c in set(succ[ptr[t]:ptr[t + 1]].tolist())
            assert (tasks[c, 7] >> 20) & 1
    r = reach(ptr, succ)
    # writers of a (tile, strip) are totally ordered
    slots = {}
    for t in range(n):
        for key in writes(tasks[t], nb, ib, ws):
            slots.setdefault(key, []).append(t)
    for key, ws_ in slots.items():
        for a, b in zip(ws_, ws_[1:]):
            assert (r[a] >> b) & 1, (key, tq.KIND_NAMES[tasks[a, 0]], tq.KIND_NAMES[tasks[b, 0]])
    # readers of reflectors follow their panel tasks
    panel_of = {}
    for t in range(n):
        name = tq.KIND_NAMES[tasks[t, 0]]
        i, piv, k, s = (int(x) for x in (tasks[t, 1], tasks[t, 2], tasks[t, 3], tasks[t, 5]))
        if name in ("GEQRT_B", "GEQRT"):
            panel_of.setdefault(("ge", i, k), []).append(t)
        if name in ("TTQRT_B", "TSQRT_B", "TTQRT", "TSQRT"):
            panel_of.setdefault(("tp", i, k), []).append(t)
    for t in range(n):
        name = tq.KIND_NAMES[tasks[t, 0]]
        i, k = int(tasks[t, 1]), int(tasks[t, 3])
        src = ("ge", i, k) if name in ("UNMQR", "GEQRT_U") else (("tp", i, k) if name in (
            "TTMQR", "TSMQR", "TTQRT_U", "TSQRT_U") else None)
        if name == "UNTTMQR":   # reads GEQRT(i,k)'s and TTQRT(i,piv,k)'s reflectors
            need = panel_of[("ge", i, k)] + panel_of[("tp", i, k)]
        elif src is None:
            continue
        else:
            need = panel_of[src] if name in ("UNMQR", "TTMQR", "TSMQR") else [
                u for u in panel_of[src] if int(tasks[u, 5]) & 0xFFFF == int(tasks[t, 4])]
        for u in need:
            assert (r[u] >> t) & 1, (name, src)
    # task counts from the tile-level DAG
    tiles = dag.expand(schemes.elim_list(tree, p, q, bs), p, q, family)
    S = -(-nb // ws)
    nblk = -(-nb // ib)
    expect = 0
    for tt in tiles:
        if tt.kind in ("UNMQR", "TTMQR", "TSMQR"):
            expect += -(-S // mstrip)
        elif split and nb > ib:
            expect += nblk + nblk * (nblk - 1) // 2
        else:
            expect += 1
    if fuse:
        npair = fused_pairs(tiles)
        expect -= npair * -(-S // mstrip)
        assert (tasks[:, 0] == tq.KIND_NAMES.index("UNTTMQR")).sum() == npair * -(-S // mstrip)
        if family == "TT" and q > 1:
            assert npair > 0
    else:
        assert not (tasks[:, 0] == tq.KIND_NAMES.index("UNTTMQR")).any()
    assert n == expect


def test_plan_graph_merge_scheme():
    """The cross-GPU merge graph (tree "merge", 2q x q tiles) is valid as well."""
    q, nb, ib = 3, 64, 32
    tasks, ptr, succ = tq.plan_graph(2 * q * nb, q * nb, nb, ib, "merge")
    assert all(succ[x] > t for t in range(len(tasks)) for x in range(ptr[t], ptr[t + 1]))
    kinds = {tq.KIND_NAMES[k] for k in tasks[:, 0]}
    # the bottom diagonal tiles are triangles already: TTQRT without a GEQRT of them
    assert "TTQRT_B" in kinds and "TTMQR" in kinds
