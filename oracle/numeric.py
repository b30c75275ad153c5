"""ORACLE (test infrastructure only) — fp64 tiled QR written as textbook Householder.

Each tile kernel of Table 1 is written out reflector
by reflector, unblocked, exactly as its name says:
  GEQRT  "factor square into triangle"         (line 245)
  TSQRT  "zero square with triangle on top"    (line 246)
  TTQRT  "zero triangle with triangle on top"  (line 247)
  UNMQR / TSMQR / TTMQR apply the transposed reflectors to the trailing tiles.
Reflectors follow LAPACK's xLARFG convention (H = I - tau v v^T, v(0) = 1,
beta = -sign(alpha) ||x||, tau = 0 when the part below alpha is zero), which
is the convention of the GEQRT kernel named at line 62.

Compact-WY T factors, inner blocking ib (line 62-66 "compact WY representation
to apply a sequence of i_b Householder reflections"; line 1031 "inner blocking
parameter of i_b=32"): for every block of ib consecutive reflectors the ib x ib
upper-triangular T with H_j0 ... H_j1-1 = I - V T V^T is built by the forward
column-wise recurrence T[:j,j] = -tau_j T[:j,:j] (V[:,:j]^T v_j), T[j,j] = tau_j.
The oracle APPLIES reflectors one at a time with their tau (it never uses T);
T is produced only as an output to compare with the GPU's T.

Storage (shared API layout): A in tiled layout as a (p*nb, q*nb)
column-major array; tile (i,k) holds R / V exactly as LAPACK GEQRT/TPQRT do:
  after GEQRT(r,k):   upper triangle incl. diagonal = R, strict lower = V
  after TTQRT(i,p,k): upper triangle incl. diagonal of tile (i,k) = V2
  after TSQRT(i,p,k): whole tile (i,k) = V2
T buffer: p*q*2 slots of ib x nb column-major (ld = ib); slot 0 of tile (i,k)
= GEQRT T, slot 1 = TTQRT/TSQRT T; block b occupies columns b*ib .. b*ib+ib-1.
"""
from __future__ import annotations

import math

import numpy as np

from . import dag


# ----------------------------------------------------------------------------
# Householder reflector (xLARFG)
# ----------------------------------------------------------------------------
def house(alpha: float, x: np.ndarray):
    """Return (beta, tau, v) with (I - tau [1;v][1;v]^T) [alpha; x] = [beta; 0]."""
    xnorm = float(np.sqrt(np.dot(x, x))) if x.size else 0.0
    if xnorm == 0.0:
        return alpha, 0.0, np.zeros_like(x)
    beta = -math.copysign(math.hypot(alpha, xnorm), alpha)
    tau = (beta - alpha) / beta
    v = x / (alpha - beta)
    return beta, tau, v


def t_block(Vfull: np.ndarray, taus: np.ndarray) -> np.ndarray:
    """Forward column-wise T of reflectors whose FULL vectors are the columns of Vfull."""
    b = Vfull.shape[1]
    T = np.zeros((b, b))
    for j in range(b):
        T[j, j] = taus[j]
        if j:
            T[:j, j] = -taus[j] * (T[:j, :j] @ (Vfull[:, :j].T @ Vfull[:, j]))
    return T


# ----------------------------------------------------------------------------
# Panel kernels. Each returns tau (length nb) and T (ib x nb, LAPACK layout).
# ----------------------------------------------------------------------------
def geqrt(A: np.ndarray, ib: int):
    """In place on the nb x nb tile A."""
    mb, nb = A.shape
    taus = np.zeros(nb)
    for i in range(min(mb, nb)):
        beta, tau, v = house(A[i, i], A[i + 1:, i].copy())
        A[i, i] = beta
        A[i + 1:, i] = v
        taus[i] = tau
        if tau != 0.0 and i + 1 < nb:
            w = A[i, i + 1:] + v @ A[i + 1:, i + 1:]
            A[i, i + 1:] -= tau * w
            A[i + 1:, i + 1:] -= tau * np.outer(v, w)
    T = np.zeros((ib, nb))
    for j0 in range(0, nb, ib):
        j1 = min(j0 + ib, nb)
        Vf = np.zeros((mb, j1 - j0))
        for c in range(j0, j1):
            Vf[c, c - j0] = 1.0
            Vf[c + 1:, c - j0] = A[c + 1:, c]
        T[:j1 - j0, j0:j1] = t_block(Vf, taus[j0:j1])
    return taus, T


def _tpqrt(A1: np.ndarray, A2: np.ndarray, ib: int, tri: bool):
    """Shared body of TTQRT (tri=True: A2 upper triangular) and TSQRT (tri=False).
    Zeroes A2 against the upper-triangular A1, column by column; reflector j is
    [e_j ; v2_j] with v2_j = A2[0:j+1, j] (TT) or A2[:, j] (TS)."""
    nb = A1.shape[1]
    mb2 = A2.shape[0]
    taus = np.zeros(nb)
    for j in range(nb):
        rows = j + 1 if tri else mb2
        beta, tau, v = house(A1[j, j], A2[:rows, j].copy())
        A1[j, j] = beta
        A2[:rows, j] = v
        taus[j] = tau
        if tau != 0.0 and j + 1 < nb:
            w = A1[j, j + 1:] + v @ A2[:rows, j + 1:]
            A1[j, j + 1:] -= tau * w
            A2[:rows, j + 1:] -= tau * np.outer(v, w)
    T = np.zeros((ib, nb))
    for j0 in range(0, nb, ib):
        j1 = min(j0 + ib, nb)
        # the e_j parts are orthonormal and distinct, so only the V2 parts
        # contribute to the off-diagonal inner products
        Vf = np.zeros((mb2, j1 - j0))
        for c in range(j0, j1):
            rows = c + 1 if tri else mb2
            Vf[:rows, c - j0] = A2[:rows, c]
        T[:j1 - j0, j0:j1] = t_block(Vf, taus[j0:j1])
    return taus, T


def ttqrt(A1, A2, ib):
    return _tpqrt(A1, A2, ib, tri=True)


def tsqrt(A1, A2, ib):
    return _tpqrt(A1, A2, ib, tri=False)


# ----------------------------------------------------------------------------
# Update kernels: apply H_{nb-1} ... H_1 H_0 (trans=True, i.e. Q^T) or
# H_0 H_1 ... H_{nb-1} (trans=False, i.e. Q) with the reflectors of a panel.
# ----------------------------------------------------------------------------
def unmqr(V: np.ndarray, taus: np.ndarray, C: np.ndarray, trans: bool = True):
    nb = V.shape[1]
    order = range(nb) if trans else range(nb - 1, -1, -1)
    for i in order:
        if taus[i] == 0.0:
            continue
        v = np.concatenate(([1.0], V[i + 1:, i]))
        w = v @ C[i:, :]
        C[i:, :] -= taus[i] * np.outer(v, w)


def _tpmqr(V2, taus, C1, C2, tri, trans):
    nb = V2.shape[1]
    mb2 = V2.shape[0]
    order = range(nb) if trans else range(nb - 1, -1, -1)
    for j in order:
        if taus[j] == 0.0:
            continue
        rows = j + 1 if tri else mb2
        v2 = V2[:rows, j]
        w = C1[j, :] + v2 @ C2[:rows, :]
        C1[j, :] -= taus[j] * w
        C2[:rows, :] -= taus[j] * np.outer(v2, w)


def ttmqr(V2, taus, C1, C2, trans=True):
    _tpmqr(V2, taus, C1, C2, True, trans)


def tsmqr(V2, taus, C1, C2, trans=True):
    _tpmqr(V2, taus, C1, C2, False, trans)


# ----------------------------------------------------------------------------
# Tiled QR driven by an elimination list (Algorithms 2-3 via dag.expand)
# ----------------------------------------------------------------------------
class Factor:
    """Result of tiled_qr: factored tiles + taus + T buffer (API layout)."""

    def __init__(self, A, p, q, nb, ib, tasks):
        self.A, self.p, self.q, self.nb, self.ib, self.tasks = A, p, q, nb, ib, tasks
        self.tau = {}                                   # (slot, i, k) -> taus
        self.T = np.zeros(p * q * 2 * ib * nb)

    def tile(self, i, k, M=None):
        nb = self.nb
        M = self.A if M is None else M
        return M[(i - 1) * nb:i * nb, (k - 1) * nb:k * nb]

    def put_T(self, slot, i, k, T):
        off = (((k - 1) * self.p + (i - 1)) * 2 + slot) * self.ib * self.nb
        self.T[off:off + self.ib * self.nb] = T.ravel(order="F")

    def R(self):
        n = self.q * self.nb
        return np.triu(self.A[:n, :n])


def tiled_qr(A: np.ndarray, nb: int, ib: int, lst, family: str = "TT") -> Factor:
    """Factor a copy of A (m x n, m = p nb, n = q nb) with elimination list lst."""
    m, n = A.shape
    p, q = m // nb, n // nb
    assert p * nb == m and q * nb == n and p >= q
    F = Factor(np.array(A, dtype=np.float64, order="F", copy=True), p, q, nb, ib,
               dag.expand(lst, p, q, family))
    for t in F.tasks:
        if t.kind == "GEQRT":
            taus, T = geqrt(F.tile(t.i, t.k), ib)
            F.tau[(0, t.i, t.k)] = taus
            F.put_T(0, t.i, t.k, T)
        elif t.kind == "UNMQR":
            unmqr(F.tile(t.i, t.k), F.tau[(0, t.i, t.k)], F.tile(t.i, t.j))
        elif t.kind in ("TTQRT", "TSQRT"):
            f = ttqrt if t.kind == "TTQRT" else tsqrt
            taus, T = f(F.tile(t.piv, t.k), F.tile(t.i, t.k), ib)
            F.tau[(1, t.i, t.k)] = taus
            F.put_T(1, t.i, t.k, T)
        else:
            f = ttmqr if t.kind == "TTMQR" else tsmqr
            f(F.tile(t.i, t.k), F.tau[(1, t.i, t.k)], F.tile(t.piv, t.j), F.tile(t.i, t.j))
    return F


def apply_qt(F: Factor, C: np.ndarray) -> np.ndarray:
    """Return Q^T C: replay the panel kernels in emission order on the rows of C."""
    C = np.array(C, dtype=np.float64, order="F", copy=True)
    nb = F.nb
    rows = lambda r: C[(r - 1) * nb:r * nb, :]
    for t in F.tasks:
        if t.kind == "GEQRT":
            unmqr(F.tile(t.i, t.k), F.tau[(0, t.i, t.k)], rows(t.i), trans=True)
        elif t.kind in ("TTQRT", "TSQRT"):
            f = ttmqr if t.kind == "TTQRT" else tsmqr
            f(F.tile(t.i, t.k), F.tau[(1, t.i, t.k)], rows(t.piv), rows(t.i), trans=True)
    return C


def apply_q(F: Factor, C: np.ndarray) -> np.ndarray:
    """Return Q C: the transposed replay in reverse emission order."""
    C = np.array(C, dtype=np.float64, order="F", copy=True)
    nb = F.nb
    rows = lambda r: C[(r - 1) * nb:r * nb, :]
    for t in reversed(F.tasks):
        if t.kind == "GEQRT":
            unmqr(F.tile(t.i, t.k), F.tau[(0, t.i, t.k)], rows(t.i), trans=False)
        elif t.kind in ("TTQRT", "TSQRT"):
            f = ttmqr if t.kind == "TTQRT" else tsmqr
            f(F.tile(t.i, t.k), F.tau[(1, t.i, t.k)], rows(t.piv), rows(t.i), trans=False)
    return C


# ----------------------------------------------------------------------------
# Independent reference: unblocked Householder QR of the whole matrix
# (§1, line 59-61: "One elementary Householder reflection ...
# the whole triangularization requires n Householder reflections")
# ----------------------------------------------------------------------------
def householder_qr(A: np.ndarray):
    """Return (R n x n, Q m x n) of the unblocked Householder QR."""
    A = np.array(A, dtype=np.float64, copy=True)
    m, n = A.shape
    vs, taus = [], []
    for i in range(n):
        beta, tau, v = house(A[i, i], A[i + 1:, i].copy())
        full = np.concatenate(([1.0], v))
        if tau != 0.0:
            w = full @ A[i:, i:]
            A[i:, i:] -= tau * np.outer(full, w)
        A[i, i] = beta
        A[i + 1:, i] = 0.0
        vs.append(full)
        taus.append(tau)
    Q = np.eye(m, n)
    for i in range(n - 1, -1, -1):
        w = vs[i] @ Q[i:, :]
        Q[i:, :] -= taus[i] * np.outer(vs[i], w)
    return np.triu(A[:n, :n]), Q


def sign_normalise(R: np.ndarray) -> np.ndarray:
    """Flip rows so the diagonal is non-negative (R is unique up to row signs)."""
    s = np.where(np.diag(R) < 0, -1.0, 1.0)
    return R * s[:, None]


def flops_qr(m: int, n: int) -> float:
    """2 n^2 (m - n/3) (line 378: 2mn^2 - 2/3 n^3)."""
    return 2.0 * n * n * (m - n / 3.0)
