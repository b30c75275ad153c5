"""ORACLE (test infrastructure only) — elimination lists of every tree.

Indices are 1-based, as in the paper. An elimination elim(i, piv, k) zeroes
tile (i,k) using row piv (§2, Algorithm 1). A list is
a Python list of (i, piv, k) tuples in list order.

Trees (§3.1 "Coarse-grain algorithms", lines 478-512, and §3.2
"Tiled algorithms", lines 652-956):
  flat       Sameh-Kuck / FlatTree: elim(i,k,k), i = k+1..p   (line 488)
  fibonacci  Fibonacci scheme of order 1                        (lines 490-505)
  greedy     Greedy                                             (lines 507-512)
  binary     BinaryTree                                         (lines 914-918)
  plasma     PlasmaTree(BS): flat inside domains of BS rows, binary merge
             of the domain heads; the bottom domain shrinks     (lines 936-953)

List order (DESIGN.md "Readings" R2): flat by (k, i); fibonacci and greedy by
(coarse step, k, i); binary by (k, round, i); plasma by (k, phase, round, i)
with phase 0 = the flat eliminations inside the domains, phase 1 = the merge.
"""
from __future__ import annotations

TREES = ("flat", "fibonacci", "greedy", "binary", "plasma")


# ----------------------------------------------------------------------------
# Sameh-Kuck / FlatTree (line 488)
# ----------------------------------------------------------------------------
def flat_list(p: int, q: int):
    return [(i, k, k) for k in range(1, min(p, q) + 1) for i in range(k + 1, p + 1)]


def flat_coarse(p: int, q: int):
    """Coarse time-steps of Sameh-Kuck: coarse(i,k) = i + k - 2 (Table 2(a))."""
    return {(i, k): i + k - 2 for k in range(1, min(p, q) + 1) for i in range(k + 1, p + 1)}


# ----------------------------------------------------------------------------
# Fibonacci (lines 490-505)
# ----------------------------------------------------------------------------
def fib_x(p: int) -> int:
    """Least integer x such that x(x+1)/2 >= p-1 (line 495)."""
    x = 0
    while x * (x + 1) // 2 < p - 1:
        x += 1
    return x


def _fib_y(i: int) -> int:
    """Least integer y such that i <= y(y+1)/2 + 1 (line 496)."""
    y = 0
    while i > y * (y + 1) // 2 + 1:
        y += 1
    return y


def fib_coarse(p: int, q: int):
    """coarse(i,1) = x - y + 1 (line 496); coarse(i,k) = coarse(i-1,k-1) + 2 (line 504)."""
    x = fib_x(p)
    c = {}
    for i in range(2, p + 1):
        c[(i, 1)] = x - _fib_y(i) + 1
    for k in range(2, min(p, q) + 1):
        for i in range(k + 1, p + 1):
            c[(i, k)] = c[(i - 1, k - 1)] + 2
    return c


def _pair_bunches(coarse, p, k):
    """Pairing rule (lines 497-502): the z tiles zeroed at one step, rows a..a+z-1,
    use the z rows right above them: piv(a+j) = a+j-z."""
    piv = {}
    rows = list(range(k + 1, p + 1))
    by_step = {}
    for i in rows:
        by_step.setdefault(coarse[(i, k)], []).append(i)
    for s, grp in by_step.items():
        grp.sort()
        z = len(grp)
        a = grp[0]
        assert grp == list(range(a, a + z)), "a bunch must be consecutive rows"
        for j in range(z):
            piv[a + j] = a + j - z
    return piv


def _sorted_by_steps(coarse, pivots):
    items = [(coarse[(i, k)], k, i, pivots[(i, k)]) for (i, k) in coarse]
    items.sort()
    return [(i, pv, k) for (s, k, i, pv) in items]


def fib_list(p: int, q: int):
    c = fib_coarse(p, q)
    piv = {}
    for k in range(1, min(p, q) + 1):
        for i, pv in _pair_bunches(c, p, k).items():
            piv[(i, k)] = pv
    return _sorted_by_steps(c, piv)


# ----------------------------------------------------------------------------
# Greedy (lines 507-512): at each step, in each column, eliminate as many tiles
# as possible, starting with the bottom rows; pairing as for Fibonacci.
# ----------------------------------------------------------------------------
def greedy_coarse_and_pivots(p: int, q: int):
    kmax = min(p, q)
    zero_step = {}          # (i,k) -> step at which tile (i,k) is zeroed
    piv = {}
    s = 0
    remaining = sum(p - k for k in range(1, kmax + 1))
    while remaining > 0:
        s += 1
        new = []
        for k in range(1, kmax + 1):
            # rows r >= k ready for column k: all tiles left of column k zeroed
            # at a step < s (the coarse model's readiness, lines 362-366).
            avail = []
            for r in range(k, p + 1):
                if (r, k) in zero_step:
                    continue
                if k == 1 or zero_step.get((r, k - 1), s) < s:
                    avail.append(r)
            z = len(avail) // 2
            if z == 0:
                continue
            # avail is a contiguous range of rows (proved in DESIGN.md R3)
            assert avail == list(range(avail[0], avail[0] + len(avail)))
            elim = avail[len(avail) - z:]
            pivs = avail[len(avail) - 2 * z:len(avail) - z]
            for r, pv in zip(elim, pivs):
                new.append((r, k, pv))
        for r, k, pv in new:
            zero_step[(r, k)] = s
            piv[(r, k)] = pv
            remaining -= 1
    return zero_step, piv


def greedy_coarse(p: int, q: int):
    return greedy_coarse_and_pivots(p, q)[0]


def greedy_list(p: int, q: int):
    c, piv = greedy_coarse_and_pivots(p, q)
    return _sorted_by_steps(c, piv)


# ----------------------------------------------------------------------------
# BinaryTree (lines 914-918): binary reduction in each column; in round r the
# survivors at distance 2^(r-1) are paired, the upper row survives.
# ----------------------------------------------------------------------------
def _lowbit(d: int) -> int:
    return d & (-d)


def binary_list(p: int, q: int):
    out = []
    for k in range(1, min(p, q) + 1):
        items = []
        for i in range(k + 1, p + 1):
            lb = _lowbit(i - k)
            items.append((lb.bit_length(), i, i - lb))
        items.sort()
        out += [(i, pv, k) for (_, i, pv) in items]
    return out


# ----------------------------------------------------------------------------
# PlasmaTree(BS) (lines 936-953): domains of BS consecutive rows starting at the
# diagonal row k; flat tree inside each domain (its first row is the local
# panel); binary tree over the domain heads; the bottom domain shrinks as k
# grows (R4, fixed by Table 3(e)).
# ----------------------------------------------------------------------------
def plasma_list(p: int, q: int, bs: int):
    assert 1 <= bs
    out = []
    for k in range(1, min(p, q) + 1):
        heads = list(range(k, p + 1, bs))
        flat = []
        for h in heads:
            for i in range(h + 1, min(h + bs, p + 1)):
                flat.append((i, h, k))
        flat.sort(key=lambda t: t[0])
        merge = []
        for d in range(1, len(heads)):
            lb = _lowbit(d)
            merge.append((lb.bit_length(), heads[d], heads[d - lb]))
        merge.sort()
        out += flat + [(i, pv, k) for (_, i, pv) in merge]
    return out


# ----------------------------------------------------------------------------
def elim_list(tree: str, p: int, q: int, bs: int = 1):
    assert p >= q >= 1
    if tree == "flat":
        return flat_list(p, q)
    if tree == "fibonacci":
        return fib_list(p, q)
    if tree == "greedy":
        return greedy_list(p, q)
    if tree == "binary":
        return binary_list(p, q)
    if tree == "plasma":
        return plasma_list(p, q, bs)
    raise ValueError(tree)


def coarse_asap(lst):
    """Coarse-grain ASAP time-steps of any list (lines 466-471): an elimination
    takes one step and may run once both rows finished their previous
    eliminations (list order). Used as the coarse schedule of binary/plasma,
    which the paper defines only as tiled algorithms (R5)."""
    last = {}
    steps = {}
    for (i, pv, k) in lst:
        s = 1 + max(last.get(i, 0), last.get(pv, 0))
        steps[(i, k)] = s
        last[i] = s
        last[pv] = s
    return steps


def coarse_steps(tree: str, p: int, q: int, bs: int = 1):
    if tree == "flat":
        return flat_coarse(p, q)
    if tree == "fibonacci":
        return fib_coarse(p, q)
    if tree == "greedy":
        return greedy_coarse(p, q)
    return coarse_asap(elim_list(tree, p, q, bs))


# ----------------------------------------------------------------------------
# Validity of a list (§2.2)
# ----------------------------------------------------------------------------
def validate(lst, p: int, q: int):
    """Return a list of violation strings (empty == valid)."""
    bad = []
    kmax = min(p, q)
    seen = set()
    for (i, pv, k) in lst:
        if not (1 <= k <= kmax and k < i <= p and k <= pv <= p and pv != i):
            bad.append(f"range elim({i},{pv},{k})")
        if (i, k) in seen:
            bad.append(f"duplicate tile ({i},{k})")
        seen.add((i, k))
    need = {(i, k) for k in range(1, kmax + 1) for i in range(k + 1, p + 1)}
    if seen != need:
        bad.append(f"coverage: missing {sorted(need - seen)[:5]} extra {sorted(seen - need)[:5]}")
    zeroed = set()
    for (i, pv, k) in lst:
        for r in (i, pv):
            for kk in range(1, k):
                if (r, kk) not in zeroed:
                    bad.append(f"row {r} not ready for elim({i},{pv},{k}): ({r},{kk}) nonzero")
                    break
        if (pv, k) in zeroed:
            bad.append(f"pivot ({pv},{k}) already zeroed in elim({i},{pv},{k})")
        zeroed.add((i, k))
    return bad
