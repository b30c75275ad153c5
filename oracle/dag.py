"""ORACLE (test infrastructure only) — kernel tasks, dependencies, critical paths.

Kernel weights: Table 1, unit n_b^3/3 flops:
  GEQRT 4, UNMQR 6, TSQRT 6, TSMQR 12, TTQRT 2, TTMQR 6.

Expansion of an elimination list (in list order):
  TT family, Algorithm 3 (lines 289-307): GEQRT + UNMQR of both rows unless
    the tile is already a triangle (lines 333-335), then TTQRT + TTMQR.
  TS family, Algorithm 2 (lines 254-268): GEQRT + UNMQR of the pivot row
    unless already a triangle, then TSQRT + TSMQR — or TTQRT + TTMQR when the
    eliminated tile is already a triangle (it served as a pivot earlier in the
    column; R6). This keeps the total weight 6pq^2 - 2q^3 for every
    list (line 377).
  Finally every diagonal tile (k,k) not yet a triangle is factored by
  GEQRT(k,k) + UNMQR(k,k,j) (the square case of Theorem 1(1)).

Dependencies (execution semantics §2.3; dependency lists of
§2.1, lines 276-283 and 316-326; NODEP relaxation of §4):
  * every kernel writes tiles: GEQRT(r,k) -> (r,k); UNMQR(r,k,j) -> (r,j);
    TxQRT(i,piv,k) -> (piv,k),(i,k); TxMQR(i,piv,k,j) -> (piv,j),(i,j);
    successive writers of a tile are chained in emission order;
  * an update reads the reflectors of its panel kernel: UNMQR(r,k,j) after
    GEQRT(r,k); TxMQR(i,piv,k,j) after TxQRT(i,piv,k);
  * reading reflectors does NOT block a later writer of that tile (NODEP).
Time is integral; with unbounded processors every task starts when its last
predecessor finishes (lines 388-392).
"""
from __future__ import annotations

WEIGHT = {"GEQRT": 4, "UNMQR": 6, "TSQRT": 6, "TSMQR": 12, "TTQRT": 2, "TTMQR": 6}


class Task:
    __slots__ = ("kind", "i", "piv", "k", "j", "deps", "idx")

    def __init__(self, kind, i, piv, k, j, idx):
        self.kind, self.i, self.piv, self.k, self.j, self.idx = kind, i, piv, k, j, idx
        self.deps = []

    @property
    def weight(self):
        return WEIGHT[self.kind]

    def key(self):
        return (self.kind, self.i, self.piv, self.k, self.j)

    def __repr__(self):
        return f"{self.kind}(i={self.i},piv={self.piv},k={self.k},j={self.j})"


def expand(lst, p: int, q: int, family: str = "TT"):
    """Return the list of Task in emission order, with .deps (indices)."""
    assert family in ("TT", "TS")
    tasks = []
    last_writer = {}
    geqrt_of = {}
    tri = set()

    def emit(kind, i, piv, k, j, writes, reads_v=None):
        t = Task(kind, i, piv, k, j, len(tasks))
        deps = set()
        if reads_v is not None:
            deps.add(reads_v)
        for tile in writes:
            if tile in last_writer:
                deps.add(last_writer[tile])
        t.deps = sorted(deps)
        for tile in writes:
            last_writer[tile] = t.idx
        tasks.append(t)
        return t.idx

    def factor(r, k):
        g = emit("GEQRT", r, None, k, None, [(r, k)])
        geqrt_of[(r, k)] = g
        for j in range(k + 1, q + 1):
            emit("UNMQR", r, None, k, j, [(r, j)], reads_v=g)
        tri.add((r, k))

    for (i, piv, k) in lst:
        if (piv, k) not in tri:
            factor(piv, k)
        if family == "TT" or (i, k) in tri:
            if (i, k) not in tri:
                factor(i, k)
            qrt, mqr = "TTQRT", "TTMQR"
        else:
            qrt, mqr = "TSQRT", "TSMQR"
        e = emit(qrt, i, piv, k, None, [(piv, k), (i, k)])
        for j in range(k + 1, q + 1):
            emit(mqr, i, piv, k, j, [(piv, j), (i, j)], reads_v=e)
    for k in range(1, min(p, q) + 1):
        if (k, k) not in tri:
            factor(k, k)
    return tasks


def simulate(tasks):
    """Unbounded processors: (start, finish) per task; emission order is topological."""
    start = [0] * len(tasks)
    finish = [0] * len(tasks)
    for t in tasks:
        s = max((finish[d] for d in t.deps), default=0)
        start[t.idx] = s
        finish[t.idx] = s + t.weight
    return start, finish


def simulate_bounded(tasks, procs: int):
    """List scheduling on `procs` processors; ready task with smallest index first."""
    import heapq
    n = len(tasks)
    succ = [[] for _ in range(n)]
    indeg = [0] * n
    for t in tasks:
        for d in t.deps:
            succ[d].append(t.idx)
        indeg[t.idx] = len(t.deps)
    ready_time = [0] * n
    ready = [t.idx for t in tasks if indeg[t.idx] == 0]
    heapq.heapify(ready)
    running = []  # (finish, idx)
    now = 0
    start = [None] * n
    finish = [None] * n
    free = procs
    done = 0
    while done < n:
        while free > 0 and ready:
            ti = heapq.heappop(ready)
            start[ti] = max(now, ready_time[ti])
            finish[ti] = start[ti] + tasks[ti].weight
            heapq.heappush(running, (finish[ti], ti))
            free -= 1
        f, ti = heapq.heappop(running)
        now = f
        free += 1
        done += 1
        for s in succ[ti]:
            indeg[s] -= 1
            ready_time[s] = max(ready_time[s], f)
            if indeg[s] == 0:
                heapq.heappush(ready, s)
        # release every task finishing at the same instant before scheduling
        while running and running[0][0] == now:
            f, ti = heapq.heappop(running)
            free += 1
            done += 1
            for s in succ[ti]:
                indeg[s] -= 1
                ready_time[s] = max(ready_time[s], f)
                if indeg[s] == 0:
                    heapq.heappush(ready, s)
    return start, finish


def zero_times(tasks, finish):
    """Time at which tile (i,k) is zeroed: finish of its TxQRT (Table 3 caption)."""
    return {(t.i, t.k): finish[t.idx] for t in tasks if t.kind in ("TTQRT", "TSQRT")}


def critical_path(lst, p: int, q: int, family: str = "TT") -> int:
    tasks = expand(lst, p, q, family)
    _, fin = simulate(tasks)
    return max(fin)


def total_weight(tasks) -> int:
    return sum(t.weight for t in tasks)


# ----------------------------------------------------------------------------
# Closed forms stated by the paper
# ----------------------------------------------------------------------------
def total_weight_formula(p: int, q: int) -> int:
    """6pq^2 - 2q^3 (line 377)."""
    return 6 * p * q * q - 2 * q ** 3


def flat_tt_cp_formula(p: int, q: int) -> int:
    """Theorem 1(1), lines 762-767."""
    if q == 1:
        return 2 * p + 2
    if p > q:
        return 6 * p + 16 * q - 22
    return 22 * p - 24


def flat_ts_cp_formula(p: int, q: int) -> int:
    """Proposition 2, lines 965-972."""
    if q == 1:
        return 6 * p - 2
    if p > q:
        return 12 * p + 18 * q - 32
    return 30 * p - 34


def binary_tt_cp_formula(p: int, q: int) -> int:
    """Proposition 1 proof, line 928: (10 + 6 log2 p) q - 4 log2 p - 6, p, q powers of two, q < p."""
    lp = p.bit_length() - 1
    assert 1 << lp == p and q & (q - 1) == 0 and q < p
    return (10 + 6 * lp) * q - 4 * lp - 6


def fib_cp_upper(p: int, q: int) -> int:
    """Theorem 1(2): 22q + 6 ceil(sqrt(2p))."""
    import math
    r = math.isqrt(2 * p)
    if r * r < 2 * p:
        r += 1
    return 22 * q + 6 * r


def greedy_cp_upper(p: int, q: int) -> int:
    """Theorem 1(2): 22q + 6 ceil(log2 p)."""
    return 22 * q + 6 * (p - 1).bit_length() if p > 1 else 22 * q


def predict_gflops(gamma_seq: float, T: float, cp: float, P: int) -> float:
    """§4 (line 1071): gamma_pred = gamma_seq * T / max(T/P, cp)."""
    return gamma_seq * T / max(T / P, cp)
