"""Pins of oracle/numeric.py: the fp64 tiled QR is checked against the
mathematics (A = QR, Q^T Q = I, triangularity), a hand-worked reflector,
LAPACK's QR (numpy) and an independent unblocked Householder QR (no GPU)."""
import itertools

import numpy as np
import pytest

import qrinputs
from oracle import numeric as nu
from oracle import schemes

TREES = [("flat", 1), ("fibonacci", 1), ("greedy", 1), ("binary", 1), ("plasma", 2), ("plasma", 3)]


def test_house_hand_example():
    """xLARFG on [3; 4]: beta = -5, tau = (beta - alpha)/beta = 1.6, v = 4/(3+5) = 0.5."""
    beta, tau, v = nu.house(3.0, np.array([4.0]))
    assert beta == -5.0 and abs(tau - 1.6) < 1e-15 and abs(v[0] - 0.5) < 1e-15
    beta, tau, v = nu.house(-2.0, np.array([0.0, 0.0]))
    assert beta == -2.0 and tau == 0.0          # nothing to annihilate: H = I


def test_ttqrt_scalar_tiles_closed_form():
    """nb = 1: tiles are scalars; TT elimination of [3; 4] gives R = -5 and the
    reflector of the example above, stored in the eliminated tile."""
    A = np.array([[3.0], [4.0]])
    F = nu.tiled_qr(A, 1, 1, schemes.flat_list(2, 1), "TT")
    assert F.A[0, 0] == -5.0 and abs(F.A[1, 0] - 0.5) < 1e-15
    assert abs(F.tau[(1, 2, 1)][0] - 1.6) < 1e-15
    assert F.tau[(0, 1, 1)][0] == 0.0 and F.tau[(0, 2, 1)][0] == 0.0


@pytest.mark.parametrize("tree,bs", TREES)
def test_scalar_tiles_column_norm(tree, bs):
    """nb = 1, q = 1: |R_11| is the 2-norm of the column, for every tree."""
    a = qrinputs.gaussian(13, 1, 3)
    for fam in ("TT", "TS"):
        F = nu.tiled_qr(a, 1, 1, schemes.elim_list(tree, 13, 1, bs), fam)
        assert abs(abs(F.A[0, 0]) - np.linalg.norm(a)) < 1e-13 * np.linalg.norm(a)


def _check_factor(A, F, tol=1e-13):
    m, n = A.shape
    R = F.R()
    assert np.allclose(np.tril(R, -1), 0)
    Q = nu.apply_q(F, np.eye(m, n))
    assert np.linalg.norm(np.eye(n) - Q.T @ Q) < tol * 10
    assert np.linalg.norm(A - Q @ R) / np.linalg.norm(A) < tol
    QtA = nu.apply_qt(F, A)
    assert np.linalg.norm(QtA[:n] - R) / np.linalg.norm(R) < tol
    assert np.linalg.norm(QtA[n:]) / np.linalg.norm(R) < tol
    # numpy / LAPACK dgeqrf and the unblocked textbook QR agree up to row signs
    Rl = np.linalg.qr(A, mode="r")
    Ru, _ = nu.householder_qr(A)
    Rs = nu.sign_normalise(R)
    assert np.linalg.norm(Rs - nu.sign_normalise(Rl)) / np.linalg.norm(Rl) < tol
    assert np.linalg.norm(Rs - nu.sign_normalise(Ru)) / np.linalg.norm(Ru) < tol


@pytest.mark.parametrize("tree,bs", TREES)
@pytest.mark.parametrize("family", ["TT", "TS"])
def test_tiled_qr_identities(tree, bs, family):
    for (p, q, nb, ib) in [(6, 3, 8, 3), (5, 5, 6, 4), (7, 1, 5, 5), (4, 2, 9, 2)]:
        A = qrinputs.gaussian(p * nb, q * nb, 100 + p * q)
        F = nu.tiled_qr(A, nb, ib, schemes.elim_list(tree, p, q, bs), family)
        _check_factor(A, F)


def test_householder_qr_vs_lapack():
    A = qrinputs.gaussian(40, 17, 5)
    Ru, Qu = nu.householder_qr(A)
    assert np.linalg.norm(A - Qu @ Ru) / np.linalg.norm(A) < 1e-14
    Rl = np.linalg.qr(A, mode="r")
    assert np.linalg.norm(nu.sign_normalise(Ru) - nu.sign_normalise(Rl)) / np.linalg.norm(Rl) < 1e-14


def test_compact_wy_T_blocks():
    """Every ib x ib block T satisfies I - V T V^T = H_j0 ... H_j1-1 (the compact
    WY identity, line 62-66), for GEQRT, TTQRT and TSQRT tiles."""
    p, q, nb, ib = 3, 2, 7, 3
    A = qrinputs.gaussian(p * nb, q * nb, 11)
    for fam in ("TT", "TS"):
        F = nu.tiled_qr(A, nb, ib, schemes.greedy_list(p, q), fam)
        for (slot, i, k), taus in F.tau.items():
            off = (((k - 1) * p + (i - 1)) * 2 + slot) * ib * nb
            Tbuf = F.T[off:off + ib * nb].reshape((ib, nb), order="F")
            tile = F.tile(i, k)
            for j0 in range(0, nb, ib):
                j1 = min(j0 + ib, nb)
                if slot == 0:       # GEQRT: v_c = e_c + strict lower part of column c
                    V = np.zeros((nb, j1 - j0))
                    for c in range(j0, j1):
                        V[c, c - j0] = 1.0
                        V[c + 1:, c - j0] = tile[c + 1:, c]
                else:               # TxQRT: v_c = [e_c ; v2_c], stacked over 2 nb rows
                    tri = any(t.kind == "TTQRT" and (t.i, t.k) == (i, k) for t in F.tasks)
                    V = np.zeros((2 * nb, j1 - j0))
                    for c in range(j0, j1):
                        V[c, c - j0] = 1.0
                        rows = c + 1 if tri else nb
                        V[nb:nb + rows, c - j0] = tile[:rows, c]
                mdim = V.shape[0]
                H = np.eye(mdim)
                for c in range(j1 - j0):
                    H = H @ (np.eye(mdim) - taus[j0 + c] * np.outer(V[:, c], V[:, c]))
                T = Tbuf[:j1 - j0, j0:j1]
                assert np.allclose(np.tril(T, -1), 0)
                assert np.linalg.norm(H - (np.eye(mdim) - V @ T @ V.T)) < 1e-13


def test_all_trees_same_R_up_to_signs():
    p, q, nb, ib = 8, 4, 6, 3
    A = qrinputs.gaussian(p * nb, q * nb, 42)
    Rs = []
    for (tree, bs), fam in itertools.product(TREES, ("TT", "TS")):
        Rs.append(nu.sign_normalise(nu.tiled_qr(A, nb, ib, schemes.elim_list(tree, p, q, bs), fam).R()))
    for R in Rs[1:]:
        assert np.linalg.norm(R - Rs[0]) / np.linalg.norm(Rs[0]) < 1e-13


def test_flops_formula():
    """Line 378: (6pq^2 - 2q^3) nb^3/3 = 2mn^2 - 2/3 n^3."""
    for p, q, nb in [(40, 10, 200), (8, 4, 32), (2048, 16, 256)]:
        m, n = p * nb, q * nb
        assert abs((6 * p * q * q - 2 * q ** 3) * nb ** 3 / 3 - nu.flops_qr(m, n)) < 1e-6 * nu.flops_qr(m, n)
