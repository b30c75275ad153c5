"""Pins of oracle/asap.py (tiled ASAP and Grasap(k), §3.2 lines
666-692) against the paper's printed values (no GPU), and the C++ generator
against the oracle."""
import pytest

import paper_1104_4475_b200 as tq
from oracle import asap, dag, schemes


def test_table4b_asap_15x3(golden_matrix):
    """Table 4(b): all 39 printed ASAP zeroing times of the 15 x 3 example."""
    g = golden_matrix("table4_asap_15x3.csv")
    assert len(g) == 39
    z = asap.zero_times(15, 3, 3)
    assert {k: z[k] for k in g} == g


def test_table4c_grasap1_15x3(golden_matrix):
    """Table 4(c) Grasap(1): 'Grasap(1) finishes at time-step 62, while Greedy
    finishes at time-step 64' (line 691); 38 of the 39 printed zeroing times
    agree. Tile (7,3) is checked against the printed value in the xfail test below."""
    g = golden_matrix("table4_grasap1_15x3.csv")
    z = asap.zero_times(15, 3, 1)
    assert {k: z[k] for k in g if k != (7, 3)} == {k: v for k, v in g.items() if k != (7, 3)}
    assert asap.critical_path(15, 3, 1) == 62
    assert asap.critical_path(15, 3, 0) == 64


@pytest.mark.xfail(strict=True, reason="DESIGN.md reading R11: the tiled ASAP reading gives 52 for tile (7,3) "
                                        "of Table 4(c); the printed value is 56")
def test_table4c_grasap1_tile_7_3_printed(golden_matrix):
    g = golden_matrix("table4_grasap1_15x3.csv")
    assert asap.zero_times(15, 3, 1)[(7, 3)] == g[(7, 3)] == 56


def test_grasap0_is_greedy_and_lists_valid():
    for p in range(2, 14):
        for q in range(1, p + 1):
            assert asap.grasap_list(p, q, 0)[0] == schemes.greedy_list(p, q)
            for ka in range(0, q + 1):
                lst = asap.grasap_list(p, q, ka)[0]
                assert schemes.validate(lst, p, q) == []
                # the incremental DES agrees with the plain expansion of its own list
                assert asap.critical_path(p, q, ka) == dag.critical_path(lst, p, q)


def test_asap_vs_greedy_15x2_15x3():
    """Lines 666-681: for 15 x 2 ASAP beats Greedy; for 15 x 3 Greedy beats ASAP."""
    assert asap.critical_path(15, 2, 2) < dag.critical_path(schemes.greedy_list(15, 2), 15, 2)
    assert asap.critical_path(15, 3, 3) > dag.critical_path(schemes.greedy_list(15, 3), 15, 3)


def test_table5b_asap(golden_rows):
    """Table 5(b) ASAP column (lines 721-745): 9 of the 10 printed critical paths;
    128 x 64 gives 1734 against the printed 1748 (reading R11). The
    128 x 128 case runs in the slow test."""
    for r in golden_rows("table5b_greedy_asap_cp.csv"):
        p, q, a = int(r[0]), int(r[1]), int(r[3])
        if p == 128 and q >= 64:
            continue
        assert asap.critical_path(p, q, q) == a, (p, q)


@pytest.mark.slow
def test_table5b_asap_128_128():
    assert asap.critical_path(128, 128, 128) == 2756


@pytest.mark.slow
@pytest.mark.xfail(strict=True, reason="DESIGN.md reading R11: the tiled ASAP reading gives 1734 for 128 x 64; "
                                        "Table 5(b) prints 1748")
def test_table5b_asap_128_64_printed():
    assert asap.critical_path(128, 64, 64) == 1748


@pytest.mark.parametrize("tree", ["asap", "grasap"])
def test_cpp_asap_bit_exact(tree):
    for p in range(2, 22):
        for q in range(1, p + 1, 2):
            for ka in ([q] if tree == "asap" else sorted({0, 1, q // 2, q})):
                i, piv, k, _ = tq.elim_list(p, q, tree, ka)
                got = list(zip(i.tolist(), piv.tolist(), k.tolist()))
                assert got == asap.grasap_list(p, q, ka)[0], (p, q, ka)
    for (p, q) in [(40, 10), (64, 16), (32, 32)]:
        ka = q if tree == "asap" else 2
        assert tq.critical_path(p, q, tree, ka) == asap.critical_path(p, q, ka)
