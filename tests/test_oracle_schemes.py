"""Pins of oracle/schemes.py against PAPER.md §2-§3.1 (no GPU)."""
import itertools

import pytest

from oracle import schemes, dag

TREES = [("flat", 1), ("fibonacci", 1), ("greedy", 1), ("binary", 1),
         ("plasma", 1), ("plasma", 2), ("plasma", 3), ("plasma", 5)]


@pytest.mark.parametrize("tree", ["flat", "fibonacci", "greedy"])
def test_table2_coarse_15x6(tree, golden_matrix):
    """Table 2 (lines 515-542): every printed coarse time-step, 3 x 75 entries."""
    g = golden_matrix(f"table2_coarse_{tree}_15x6.csv")
    c = schemes.coarse_steps(tree, 15, 6)
    assert len(g) == 15 * 6 - 21
    assert {k: c[k] for k in g} == g


def test_paper_example_lists_p6():
    """§2: both example lists for p=6 are valid; elim(6,5,2)
    must follow elim(6,4,1) and elim(5,4,1)."""
    alg1 = [(2, 1, 1), (3, 1, 1), (4, 1, 1), (5, 1, 1), (6, 1, 1)]
    other = [(3, 1, 1), (6, 4, 1), (2, 1, 1), (5, 4, 1), (4, 1, 1)]
    assert schemes.validate(alg1, 6, 1) == []
    assert schemes.validate(other, 6, 1) == []
    assert schemes.flat_list(6, 1) == alg1
    bad = [(3, 1, 1), (6, 4, 1), (6, 5, 2), (2, 1, 1), (5, 4, 1), (4, 1, 1)]
    v = schemes.validate(bad, 6, 2)
    assert any("row 5 not ready" in s for s in v)


def test_invalid_pivot_already_zeroed():
    """Condition 2 of §2.2 (lines 367-369): the pivot must still be a potential annihilator."""
    v = schemes.validate([(2, 1, 1), (3, 2, 1)], 3, 1)
    assert any("already zeroed" in s for s in v)
    v = schemes.validate([(2, 1, 1)], 3, 1)
    assert any("coverage" in s for s in v)


@pytest.mark.parametrize("tree,bs", TREES)
def test_all_lists_valid(tree, bs):
    """Every generated list obeys §2.2 for all 1 <= q <= p <= 20, and uses piv < i (Lemma 1 form)."""
    for p in range(1, 21):
        for q in range(1, p + 1):
            lst = schemes.elim_list(tree, p, q, bs)
            assert schemes.validate(lst, p, q) == [], (tree, bs, p, q)
            assert all(pv < i for (i, pv, k) in lst)


def test_fibonacci_closed_forms():
    """§3.1: coarse critical path x + 2q - 2 (p > q), x + 2q - 4 (p = q);
    Sameh-Kuck p + q - 2 and 2q - 3; column shift identity coarse(i,k) = coarse(i-1,k-1)+2."""
    for p in range(2, 40):
        x = schemes.fib_x(p)
        assert x * (x + 1) // 2 >= p - 1 and (x - 1) * x // 2 < p - 1
        for q in range(1, p + 1):
            cf = schemes.fib_coarse(p, q)
            cs = schemes.flat_coarse(p, q)
            if p > q:
                assert max(cf.values()) == x + 2 * q - 2
                assert max(cs.values()) == p + q - 2
            elif q >= 2:
                assert max(cf.values()) == x + 2 * q - 4
                assert max(cs.values()) == 2 * q - 3
            for (i, k), s in cf.items():
                if k >= 2:
                    assert s == cf[(i - 1, k - 1)] + 2


def test_fibonacci_first_column_counts():
    """Line 493-495: p=15 first column has one 5, two 4's, three 3's, four 2's, four 1's."""
    c = schemes.fib_coarse(15, 1)
    counts = {s: list(c.values()).count(s) for s in set(c.values())}
    assert counts == {5: 1, 4: 2, 3: 3, 2: 4, 1: 4}
    c16 = schemes.fib_coarse(16, 1)
    assert list(c16.values()).count(1) == 5


def test_greedy_is_coarse_optimal_vs_fibonacci():
    """Greedy is optimal in the coarse model (line 548): its critical path never
    exceeds Fibonacci's or Sameh-Kuck's, and its time-steps are entrywise <= Fibonacci's."""
    for p in range(2, 33):
        for q in range(1, p + 1):
            g = schemes.greedy_coarse(p, q)
            f = schemes.fib_coarse(p, q)
            assert max(g.values()) <= max(f.values())
            assert max(g.values()) <= p + q - 2
            assert all(g[t] <= f[t] for t in g)


def test_greedy_coarse_is_asap_of_its_list():
    """Greedy eliminates as many tiles as possible at each step (line 508), so its
    steps coincide with the coarse ASAP steps of its own list."""
    for p in range(2, 25):
        for q in range(1, p + 1):
            assert schemes.coarse_asap(schemes.greedy_list(p, q)) == schemes.greedy_coarse(p, q)


def test_plasma_limits():
    """Lines 948-950: BS=1 is the binary tree on the whole column, BS=p a flat tree."""
    for p in range(1, 20):
        for q in range(1, p + 1):
            assert schemes.plasma_list(p, q, 1) == schemes.binary_list(p, q)
            assert sorted(schemes.plasma_list(p, q, p), key=lambda t: (t[2], t[0])) == schemes.flat_list(p, q)


def test_binary_pairing_15():
    """Table 3(d) column 1 structure: distances double each round, upper row survives."""
    lst = schemes.binary_list(15, 1)
    assert (2, 1, 1) in lst and (15, 13, 1) in lst and (9, 1, 1) in lst and (13, 9, 1) in lst


def test_total_coverage_and_count():
    for (tree, bs) in TREES:
        for p, q in itertools.product(range(1, 13), range(1, 13)):
            if q > p:
                continue
            lst = schemes.elim_list(tree, p, q, bs)
            assert len(lst) == sum(p - k for k in range(1, q + 1))
