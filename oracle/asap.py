"""ORACLE (test infrastructure only) — the tiled ASAP and Grasap(k) algorithms.

PAPER.md §3.2 (lines 666-692): "In each column and at each step, the ASAP
algorithm starts the elimination of a tile as soon as there are at least two
rows ready for the transformation. When s >= 2 eliminations can start
simultaneously, ASAP pairs the 2s rows just as Fibonacci and Greedy, the first
row (closest to the diagonal) with row s+1, the second row with row s+2, and so
on." Grasap(k) follows Greedy in columns 1..q-k and ASAP in the last k columns
(Grasap(0) = Greedy, Grasap(q) = ASAP).

Unlike the other trees, ASAP decides its eliminations during the tiled
execution, so this module runs the discrete-event simulation of dag.py
(unbounded processors, Table 1 weights, TT kernels, the same dependency rules)
incrementally, taking decisions as time advances. Readings (R11):
a row is "ready" in column k when its tile (i,k) is a triangle (its GEQRT
finished) and it is not inside a running TTQRT of that column; with r ready rows,
s = floor(r/2) eliminations start, the bottom s ready rows eliminated by the s
ready rows right above them (the pairing rule of Fibonacci/Greedy); a pivot is
ready again when its TTQRT finishes. All rows of a column are decided at the
same instant before time advances; columns are independent.
"""
from __future__ import annotations

from . import dag, schemes


class _Sim:
    """Incremental version of dag.expand + dag.simulate (TT family)."""

    def __init__(self, p, q):
        self.p, self.q = p, q
        self.tasks = []
        self.finish = []
        self.last = {}          # tile -> index of its last writer
        self.tri = set()
        self.lst = []

    def _emit(self, kind, i, piv, k, j, writes, reads=None):
        t = dag.Task(kind, i, piv, k, j, len(self.tasks))
        deps = set()
        if reads is not None:
            deps.add(reads)
        for w in writes:
            if w in self.last:
                deps.add(self.last[w])
        t.deps = sorted(deps)
        for w in writes:
            self.last[w] = t.idx
        s = max((self.finish[d] for d in t.deps), default=0)
        self.tasks.append(t)
        self.finish.append(s + t.weight)
        return t.idx

    def factor(self, r, k):
        """GEQRT(r,k) + UNMQR(r,k,j); returns the GEQRT finish time."""
        g = self._emit("GEQRT", r, None, k, None, [(r, k)])
        for j in range(k + 1, self.q + 1):
            self._emit("UNMQR", r, None, k, j, [(r, j)], reads=g)
        self.tri.add((r, k))
        return self.finish[g]

    def eliminate(self, i, piv, k):
        """TT elimination (Algorithm 3) of tile (i,k) by row piv (both already triangles
        when called by ASAP; factored on demand otherwise, as dag.expand does).
        Returns the TTQRT finish time."""
        if (piv, k) not in self.tri:
            self.factor(piv, k)
        if (i, k) not in self.tri:
            self.factor(i, k)
        x = self._emit("TTQRT", i, piv, k, None, [(piv, k), (i, k)])
        for j in range(k + 1, self.q + 1):
            self._emit("TTMQR", i, piv, k, j, [(piv, j), (i, j)], reads=x)
        self.lst.append((i, piv, k))
        return self.finish[x]


def grasap_list(p: int, q: int, k_asap: int):
    """Elimination list of Grasap(k_asap): Greedy in columns 1..q-k_asap, ASAP after."""
    assert p >= q >= 1 and 0 <= k_asap <= q
    kmax = min(p, q)
    first_asap = q - k_asap + 1          # first ASAP column
    sim = _Sim(p, q)
    # Greedy part: the Greedy list restricted to the first columns, in list order
    for (i, piv, k) in schemes.greedy_list(p, q):
        if k < first_asap:
            sim.eliminate(i, piv, k)
    if first_asap > kmax:
        for k in range(1, kmax + 1):
            if (k, k) not in sim.tri:
                sim.factor(k, k)
        return sim.lst, sim
    # ASAP part. ready[k][r] = time at which row r's tile (r,k) is a triangle and free
    ready = {k: {} for k in range(first_asap, kmax + 1)}
    zeroed = {k: set() for k in range(first_asap, kmax + 1)}
    k0 = first_asap
    for r in range(k0, p + 1):
        # rows entering the first ASAP column: zeroed in column k0-1 (or all rows if k0 = 1)
        if k0 == 1 or any(e[0] == r and e[2] == k0 - 1 for e in sim.lst):
            ready[k0][r] = sim.factor(r, k0)
    t = 0
    while True:
        pending = [tm for k in ready for tm in ready[k].values()]
        if not pending:
            break
        t_next = min(tm for tm in pending if tm >= t) if any(tm >= t for tm in pending) else None
        if t_next is None:
            break
        t = t_next
        progressed = False
        for k in range(first_asap, kmax + 1):
            rows = sorted(r for r, tm in ready[k].items() if tm <= t)
            s = len(rows) // 2
            if s == 0:
                continue
            elim = rows[len(rows) - s:]
            pivs = rows[len(rows) - 2 * s:len(rows) - s]
            for i, pv in zip(elim, pivs):
                done = sim.eliminate(i, pv, k)
                del ready[k][i]
                zeroed[k].add(i)
                ready[k][pv] = done                   # the pivot is free again after its TTQRT
                if k + 1 <= kmax:
                    ready[k + 1][i] = sim.factor(i, k + 1)
            progressed = True
        # a column whose only remaining row is the diagonal is finished
        for k in range(first_asap, kmax + 1):
            if len(ready[k]) == 1 and len(zeroed[k]) == p - k:
                ready[k].clear()
        if not progressed:
            # advance past the current instant
            later = [tm for k in ready for tm in ready[k].values() if tm > t]
            if not later:
                break
            t = min(later)
    # the last diagonal tile of a square matrix is factored at the end (dag.expand)
    for k in range(1, kmax + 1):
        if (k, k) not in sim.tri:
            sim.factor(k, k)
    return sim.lst, sim


def asap_list(p: int, q: int):
    return grasap_list(p, q, q)[0]


def critical_path(p: int, q: int, k_asap: int) -> int:
    lst, sim = grasap_list(p, q, k_asap)
    return max(sim.finish)


def zero_times(p: int, q: int, k_asap: int):
    lst, sim = grasap_list(p, q, k_asap)
    return {(t.i, t.k): sim.finish[t.idx] for t in sim.tasks if t.kind == "TTQRT"}
