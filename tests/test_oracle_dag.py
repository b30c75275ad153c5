"""Pins of oracle/dag.py (task expansion + discrete-event critical paths) against
the values and closed forms PAPER.md prints (no GPU)."""
import random

import pytest

from oracle import schemes, dag

TABLE3 = [("flat", "flat", 1), ("fibonacci", "fibonacci", 1), ("greedy", "greedy", 1),
          ("binary", "binary", 1), ("plasma_bs5", "plasma", 5)]


@pytest.mark.parametrize("name,tree,bs", TABLE3)
def test_table3_tiled_15x6(name, tree, bs, golden_matrix):
    """Table 3 (lines 622-649): all 69 printed TT zeroing times of the 15x6 example."""
    g = golden_matrix(f"table3_tiled_{name}_15x6.csv")
    assert len(g) == 69
    tasks = dag.expand(schemes.elim_list(tree, 15, 6, bs), 15, 6, "TT")
    _, fin = dag.simulate(tasks)
    z = dag.zero_times(tasks, fin)
    assert {k: z[k] for k in g} == g


def test_table4a_greedy_15x3(golden_matrix):
    """Table 4(a) (lines 694-719) Greedy column and 'Greedy finishes at time-step 64' (line 691)."""
    g = golden_matrix("table4_greedy_15x3.csv")
    tasks = dag.expand(schemes.greedy_list(15, 3), 15, 3, "TT")
    _, fin = dag.simulate(tasks)
    z = dag.zero_times(tasks, fin)
    assert {k: z[k] for k in g} == g
    assert max(fin) == 64


def test_table6_greedy_fibonacci(golden_rows):
    """Table 6 (lines 1317-1368): Greedy and Fibonacci TT critical paths, p=40, q=1..40."""
    for row in golden_rows("table6_p40.csv"):
        p, q, g, fb = int(row[0]), int(row[1]), int(row[2]), int(row[7])
        assert dag.critical_path(schemes.greedy_list(p, q), p, q) == g, q
        assert dag.critical_path(schemes.fib_list(p, q), p, q) == fb, q
        # overhead / gain columns are ratios of the printed integers (4 decimals)
        assert abs(fb / g - float(row[8])) < 5e-5
        assert abs(1 - g / fb - float(row[9])) < 5e-5


@pytest.mark.parametrize("q", [1, 2, 3, 6, 11, 40])
def test_table6_plasma_best_domain(q, golden_rows):
    """Table 6 PlasmaTree (TT) column: best critical path over BS = 1..p and its
    smallest argmin BS."""
    row = [r for r in golden_rows("table6_p40.csv") if int(r[1]) == q][0]
    p = 40
    cps = [(dag.critical_path(schemes.plasma_list(p, q, bs), p, q), bs) for bs in range(1, p + 1)]
    best = min(cps)
    assert best == (int(row[3]), int(row[4]))
    assert abs(best[0] / int(row[2]) - float(row[5])) < 5e-5


def test_table5b_greedy(golden_rows):
    """Table 5(b) (lines 721-745), Greedy column, p, q <= 64 (128 in the slow test)."""
    for r in golden_rows("table5b_greedy_asap_cp.csv"):
        p, q, g = int(r[0]), int(r[1]), int(r[2])
        if p <= 64:
            assert dag.critical_path(schemes.greedy_list(p, q), p, q) == g


@pytest.mark.slow
def test_table5b_greedy_128(golden_rows):
    for r in golden_rows("table5b_greedy_asap_cp.csv"):
        p, q, g = int(r[0]), int(r[1]), int(r[2])
        if p == 128:
            assert dag.critical_path(schemes.greedy_list(p, q), p, q) == g


def test_single_elimination_parallel_time():
    """§2.1: one elimination with updates costs 4+6+12 = 22 (TS, line 286) and
    4+6+6 = 16 (TT, line 330) time-units on unbounded processors."""
    lst = [(2, 1, 1)]
    tt = dag.expand(lst, 2, 2, "TT")
    ts = dag.expand(lst, 2, 2, "TS")
    # drop the final diagonal GEQRT(2,2)/its chain: measure the elimination itself
    _, f = dag.simulate(tt)
    assert max(f[t.idx] for t in tt if t.k == 1) == 16
    _, f = dag.simulate(ts)
    assert max(f[t.idx] for t in ts if t.k == 1) == 22


def test_theorem1_flat_tt_closed_form():
    """Theorem 1(1) (lines 762-767) for every 1 <= q <= p <= 30, and the proof's
    per-tile times 2i+2 (q=1 column) and 6i + 16k - 22 (lines 787-802)."""
    for p in range(1, 31):
        for q in range(1, p + 1):
            tasks = dag.expand(schemes.flat_list(p, q), p, q, "TT")
            _, fin = dag.simulate(tasks)
            assert max(fin) == dag.flat_tt_cp_formula(p, q), (p, q)
            z = dag.zero_times(tasks, fin)
            for (i, k), t in z.items():
                if k == 1:
                    assert t == 2 * i + 2
                elif p > q or k < q:
                    assert t == 6 * i + 16 * k - 22


def test_proposition2_flat_ts_closed_form():
    """Proposition 2 (lines 965-972) and its proof's 12i + 18k - 32 (line 986)."""
    for p in range(1, 31):
        for q in range(1, p + 1):
            tasks = dag.expand(schemes.flat_list(p, q), p, q, "TS")
            _, fin = dag.simulate(tasks)
            assert max(fin) == dag.flat_ts_cp_formula(p, q), (p, q)
            z = dag.zero_times(tasks, fin)
            for (i, k), t in z.items():
                if k >= 2:
                    assert t == 12 * i + 18 * k - 32


def test_proposition1_binary_closed_form():
    """Proposition 1 proof (line 928): (10 + 6 log2 p) q - 4 log2 p - 6 for powers of two q < p."""
    for lp in range(1, 7):
        p = 1 << lp
        for lq in range(0, lp):
            q = 1 << lq
            assert dag.critical_path(schemes.binary_list(p, q), p, q) == dag.binary_tt_cp_formula(p, q), (p, q)


def test_ts_never_beats_tt_on_flat():
    """§3.2: converting TS to TT increases parallelism."""
    for p in range(1, 20):
        for q in range(1, p + 1):
            lst = schemes.flat_list(p, q)
            assert dag.critical_path(lst, p, q, "TT") <= dag.critical_path(lst, p, q, "TS")


def test_total_weight_identity():
    """Line 375-382: the total weight is 6pq^2 - 2q^3 for every list and both kernel families."""
    rnd = random.Random(7)
    shapes = [(rnd.randint(1, 24), None) for _ in range(60)]
    for p, _ in shapes:
        q = rnd.randint(1, p)
        for tree, bs in [("flat", 1), ("fibonacci", 1), ("greedy", 1), ("binary", 1), ("plasma", rnd.randint(1, p))]:
            lst = schemes.elim_list(tree, p, q, bs)
            for fam in ("TT", "TS"):
                assert dag.total_weight(dag.expand(lst, p, q, fam)) == dag.total_weight_formula(p, q)
    assert dag.total_weight_formula(40, 40) == 256000 and dag.total_weight_formula(1, 1) == 4


def test_theorem1_bounds():
    """Theorem 1(2) upper bounds, and Theorem 1(3)'s lower bound 22q - 30 where the
    paper is consistent with itself: its own Table 6 prints Greedy (40,37..40) = 780,
    796, 812, 826 < 22q - 30, so the bound is checked for p - q >= 4 only
    (reading R7; test_theorem1_3_contradiction pins the conflict)."""
    for p in range(1, 29):
        for q in range(1, p + 1):
            g = dag.critical_path(schemes.greedy_list(p, q), p, q)
            f = dag.critical_path(schemes.fib_list(p, q), p, q)
            assert g <= dag.greedy_cp_upper(p, q)
            assert f <= dag.fib_cp_upper(p, q)
            if q >= 2 and p - q >= 4:
                assert g >= 22 * q - 30 and f >= 22 * q - 30


def test_theorem1_3_contradiction(golden_rows):
    """The printed Table 6 values themselves fall below 22q - 30 at q = 37..40."""
    rows = {int(r[1]): int(r[2]) for r in golden_rows("table6_p40.csv")}
    assert [q for q in rows if rows[q] < 22 * q - 30] == [37, 38, 39, 40]


def test_bounded_processors():
    """Makespan(unbounded) <= makespan(P) <= makespan(1) = total weight."""
    for tree in ("greedy", "flat", "fibonacci"):
        p, q = 10, 4
        tasks = dag.expand(schemes.elim_list(tree, p, q), p, q)
        _, f_inf = dag.simulate(tasks)
        prev = None
        for P in (1, 2, 4, 16, 10 ** 6):
            s, f = dag.simulate_bounded(tasks, P)
            for t in tasks:
                assert all(s[t.idx] >= f[d] for d in t.deps)
            if P == 1:
                assert max(f) == dag.total_weight_formula(p, q)
            if prev is not None:
                assert max(f) <= prev
            prev = max(f)
        assert prev == max(f_inf)


def test_predict_formula():
    """§4 (line 1071) with Table 6's cp and γ_seq = 3.1860 (line 1075): work bound regime."""
    T = dag.total_weight_formula(40, 40)
    assert abs(dag.predict_gflops(3.1860, T, 826, 48) - 3.1860 * 48) < 1e-9
    assert abs(dag.predict_gflops(3.1860, 238, 16, 48) - 3.1860 * 238 / 16) < 1e-9
