"""Host logic of the product library (no GPU): the C ABI loads and exports
every symbol include/tiledqr.h declares, and the C elimination-list / schedule
generator is bit-exact against the oracle and the paper's printed values."""
import os
import re

import numpy as np
import pytest

import paper_1104_4475_b200 as tq
from oracle import dag, schemes
from tests.conftest import ROOT

TREES = [("flat", 1), ("fibonacci", 1), ("greedy", 1), ("binary", 1),
         ("plasma", 1), ("plasma", 2), ("plasma", 3), ("plasma", 5)]


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "tiledqr.h")).read()
    decl = re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(\w+)\s*\(", hdr, re.M)
    decl = [d for d in decl if d not in ("if", "while")]
    assert {"elim_list", "critical_path", "tiled_times", "tiled_qr", "apply_qt", "apply_q",
            "tiled_qr_host"} <= set(decl)
    L = tq.lib()
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(tq.EXPORTS)
    assert L.tqr_version() >= 100


def _oracle_list(tree, p, q, bs):
    if tree == "greedy":      # one simulation gives both the list and its steps
        steps, piv = schemes.greedy_coarse_and_pivots(p, q)
        lst = sorted(((steps[(i, k)], k, i, piv[(i, k)]) for (i, k) in steps))
        return [(i, pv, k, s) for (s, k, i, pv) in lst]
    lst = schemes.elim_list(tree, p, q, bs)
    steps = schemes.coarse_steps(tree, p, q, bs)
    return [(i, pv, k, steps[(i, k)]) for (i, pv, k) in lst]


@pytest.mark.parametrize("tree,bs", TREES)
def test_elim_list_bit_exact(tree, bs):
    for p in range(1, 25):
        for q in range(1, p + 1):
            if tree == "plasma" and bs > p:
                continue
            i, piv, k, st = tq.elim_list(p, q, tree, bs)
            got = list(zip(i.tolist(), piv.tolist(), k.tolist(), st.tolist()))
            assert got == _oracle_list(tree, p, q, bs), (tree, bs, p, q)


@pytest.mark.parametrize("p,q", [(1000, 100), (1000, 1), (333, 77)])
def test_elim_list_large(p, q):
    """configs[4]: list generation up to p = 1000, q = 100."""
    trees = [("greedy", 1), ("fibonacci", 1), ("flat", 1), ("binary", 1), ("plasma", 10)]
    for tree, bs in trees:
        i, piv, k, st = tq.elim_list(p, q, tree, bs)
        got = list(zip(i.tolist(), piv.tolist(), k.tolist(), st.tolist()))
        assert got == _oracle_list(tree, p, q, bs), (tree, p, q)


def test_table2_from_product(golden_matrix):
    """Table 2 coarse steps straight from the C generator."""
    for tree in ("flat", "fibonacci", "greedy"):
        g = golden_matrix(f"table2_coarse_{tree}_15x6.csv")
        i, piv, k, st = tq.elim_list(15, 6, tree)
        got = {(a, b): s for a, b, s in zip(i.tolist(), k.tolist(), st.tolist())}
        assert {key: got[key] for key in g} == g


@pytest.mark.parametrize("name,tree,bs", [("flat", "flat", 1), ("fibonacci", "fibonacci", 1),
                                          ("greedy", "greedy", 1), ("binary", "binary", 1),
                                          ("plasma_bs5", "plasma", 5)])
def test_table3_from_product(name, tree, bs, golden_matrix):
    """Table 3 (lines 622-649) tile zeroing times from the C simulator."""
    g = golden_matrix(f"table3_tiled_{name}_15x6.csv")
    _, z = tq.tiled_times(15, 6, tree, bs)
    assert {key: int(z[key[0] - 1, key[1] - 1]) for key in g} == g


def test_table6_from_product(golden_rows):
    """Table 6 (lines 1317-1368): Greedy, Fibonacci and best-BS PlasmaTree (TT) critical paths."""
    for row in golden_rows("table6_p40.csv"):
        p, q = int(row[0]), int(row[1])
        assert tq.critical_path(p, q, "greedy") == int(row[2])
        assert tq.critical_path(p, q, "fibonacci") == int(row[7])
        best = min((tq.critical_path(p, q, "plasma", bs), bs) for bs in range(1, p + 1))
        assert best == (int(row[3]), int(row[4])), q


def test_table5b_from_product(golden_rows):
    for r in golden_rows("table5b_greedy_asap_cp.csv"):
        p, q, g = int(r[0]), int(r[1]), int(r[2])
        assert tq.critical_path(p, q, "greedy") == g


@pytest.mark.parametrize("family", ["TT", "TS"])
def test_critical_path_matches_oracle_des(family):
    for p in range(1, 16):
        for q in range(1, p + 1):
            for tree, bs in TREES:
                if tree == "plasma" and bs > p:
                    continue
                lst = schemes.elim_list(tree, p, q, bs)
                assert tq.critical_path(p, q, tree, bs, family) == dag.critical_path(lst, p, q, family)


def test_closed_forms_from_product():
    """Theorem 1(1) and Proposition 2 closed forms; Proposition 1's power-of-two formula."""
    for p in range(1, 41):
        for q in range(1, p + 1):
            assert tq.critical_path(p, q, "flat", 1, "TT") == dag.flat_tt_cp_formula(p, q)
            assert tq.critical_path(p, q, "flat", 1, "TS") == dag.flat_ts_cp_formula(p, q)
    for lp in range(1, 8):
        for lq in range(0, lp):
            p, q = 1 << lp, 1 << lq
            assert tq.critical_path(p, q, "binary") == dag.binary_tt_cp_formula(p, q)


def test_bad_arguments_raise():
    with pytest.raises(tq.TiledQRError):
        tq.elim_list(3, 4, "greedy")
    with pytest.raises(tq.TiledQRError):
        tq.elim_list(5, 2, "plasma", 0)
    with pytest.raises(tq.TiledQRError):
        tq.critical_path(5, 2, 9)
    assert "p >= q" in tq.lib().tqr_last_error().decode() or tq.lib().tqr_last_error()


def _oracle_des(args):
    """Oracle critical path and tiled zeroing times of one (tree, family) case (worker process)."""
    p, q, tree, bs, family = args
    tasks = dag.expand(schemes.elim_list(tree, p, q, bs), p, q, family)
    _, fin = dag.simulate(tasks)
    return max(fin), dag.zero_times(tasks, fin)


def test_configs4_large_des_matches_oracle():
    """configs[4]: the product's critical_path and tiled_times (C++ DES of the Algorithm 2/3
    expansion, §3) equal the oracle DES bit for bit at (p, q) =
    (1000, 100), (1000, 1) and (333, 77), for every tree and both kernel families. The oracle
    needs ~35 s and 2.5 GB per (1000, 100) case, so the cases run in a 4-process pool."""
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    trees = [("flat", 1), ("fibonacci", 1), ("greedy", 1), ("binary", 1), ("plasma", 10)]
    cases = [(p, q, tree, bs, fam) for (p, q) in [(1000, 100), (333, 77), (1000, 1)]
             for tree, bs in trees for fam in ("TT", "TS")]
    with ProcessPoolExecutor(max_workers=4, mp_context=mp.get_context("spawn")) as ex:
        results = list(ex.map(_oracle_des, cases))
    for (p, q, tree, bs, fam), (cp, zt) in zip(cases, results):
        assert tq.critical_path(p, q, tree, bs, fam) == cp, (p, q, tree, bs, fam)
        got_cp, z = tq.tiled_times(p, q, tree, bs, fam)
        assert got_cp == cp
        assert {(i, k): int(z[i - 1, k - 1]) for (i, k) in zt} == zt, (p, q, tree, bs, fam)
        assert int(np.count_nonzero(z)) == len(zt)
