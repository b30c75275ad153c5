"""GPU parity: the CUDA tiled QR (through the C ABI) against the CPU oracle on
the same seeded inputs. Tolerances are north_star's (BASELINE.json):
||A - QR||_F / ||A||_F <= 1e-12, ||I - Q^T Q||_F <= 1e-12, and R equal to the
oracle's R after row-sign normalisation within relative Frobenius 1e-10; the
reflectors V and compact-WY T factors are compared the same way (1e-10)."""
import numpy as np
import pytest

import qrinputs
from oracle import asap
from oracle import numeric as nu
from oracle import schemes

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1104_4475_b200 as tq  # noqa: E402

DEV = "cuda:0"
TOL_R = 1e-10
TOL_QR = 1e-12


def rel(a, b):
    nb_ = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb_ if nb_ > 0 else 1.0)


def run_gpu(A, nb, ib, tree, bs, family):
    m, n = A.shape
    buf = torch.from_numpy(qrinputs.to_tiles(A, nb)).to(DEV)
    T = tq.tiled_qr(buf, m, n, nb, ib, tree, bs, family)
    torch.cuda.synchronize()
    return buf, T


def gpu_Q(buf, T, m, n, nb, ib, tree, bs, family):
    E = np.zeros((m, n))
    E[:n, :n] = np.eye(n)
    Cb = torch.from_numpy(qrinputs.to_tiles(E, nb)).to(DEV)
    tq.apply_q(buf, T, Cb, m, n, nb, ib, tree, bs, family)
    torch.cuda.synchronize()
    return qrinputs.from_tiles(Cb.cpu().numpy(), m // nb, n // nb, nb)


def oracle_list(tree, p, q, bs):
    if tree == "asap":
        return asap.grasap_list(p, q, q)[0]
    if tree == "grasap":
        return asap.grasap_list(p, q, bs)[0]
    return schemes.elim_list(tree, p, q, bs)


def compare_with_oracle(A, nb, ib, tree, bs, family, tol=TOL_R):
    m, n = A.shape
    p, q = m // nb, n // nb
    buf, T = run_gpu(A, nb, ib, tree, bs, family)
    F = nu.tiled_qr(A, nb, ib, oracle_list(tree, p, q, bs), family)
    got = qrinputs.from_tiles(buf.cpu().numpy(), p, q, nb)
    # R (north_star: after row-sign normalisation)
    Rg = np.triu(got[:n, :n])
    assert rel(nu.sign_normalise(Rg), nu.sign_normalise(F.R())) <= tol
    # the whole factored buffer (R + V) and the T factors, element by element
    assert rel(got, F.A) <= tol
    assert np.max(np.abs(got - F.A)) <= tol * max(1.0, np.max(np.abs(F.A)))
    Tg = T.cpu().numpy()
    assert rel(Tg, F.T) <= tol
    return buf, T, F


CASES = [
    # (p, q, nb, ib) — several tiles, ragged inner blocks, nb not a multiple of 8
    (8, 4, 32, 32),     # configs[0]
    (6, 3, 20, 8),
    (5, 5, 12, 5),
    (7, 2, 24, 32),
    (4, 1, 16, 16),
    # nb > ws = ib = 32: panels split into per-inner-block tasks (+ ragged last block)
    (4, 2, 72, 32),
    (3, 3, 64, 32),
]
TREES = [("flat", 1), ("fibonacci", 1), ("greedy", 1), ("binary", 1), ("plasma", 2), ("plasma", 3)]


@pytest.mark.parametrize("family", ["TT", "TS"])
@pytest.mark.parametrize("tree,bs", TREES)
def test_factor_parity_small(tree, bs, family):
    for (p, q, nb, ib) in CASES:
        if tree == "plasma" and bs > p:
            continue
        A = qrinputs.gaussian(p * nb, q * nb, 1000 + 7 * p + q)
        compare_with_oracle(A, nb, ib, tree, bs, family)


# Production tile sizes (BASELINE.json configs[1]/[2]: nb = 200; configs[3]: nb = 256; ib = 32,
# PAPER.md lines 1029-1031): several tiles per dimension, 7-8 inner blocks per panel, the
# ragged last inner block of nb = 200 (bw = 8) and the last strip of width 8.
PROD_CASES = [(4, 2, 200, 32), (3, 3, 200, 32), (3, 2, 256, 32), (5, 3, 256, 32)]
PROD_TREES = [("flat", 1), ("fibonacci", 1), ("greedy", 1), ("plasma", 2)]


@pytest.mark.parametrize("family", ["TT", "TS"])
@pytest.mark.parametrize("tree,bs", PROD_TREES)
@pytest.mark.parametrize("p,q,nb,ib", PROD_CASES)
def test_factor_parity_production_tiles(p, q, nb, ib, tree, bs, family):
    """Element-wise parity of R+V and T with the oracle at the benchmarked tile
    sizes (max-abs and relative Frobenius, 1e-10)."""
    A = qrinputs.gaussian(p * nb, q * nb, 500 + 3 * p + q + nb)
    compare_with_oracle(A, nb, ib, tree, bs, family)


@pytest.mark.parametrize("p,q,nb,tree,family", [(4, 2, 200, "greedy", "TT"), (3, 2, 256, "flat", "TS"),
                                                (3, 3, 200, "fibonacci", "TS")])
def test_apply_parity_production_tiles(p, q, nb, tree, family):
    """apply_qt / apply_q at nb = 200 / 256 against the oracle's reflector-by-reflector apply."""
    ib = 32
    m, n = p * nb, q * nb
    A = qrinputs.gaussian(m, n, 41 + nb)
    buf, T, F = compare_with_oracle(A, nb, ib, tree, 1, family)
    C = qrinputs.gaussian(m, 2 * nb, 42 + nb)
    for trans in (True, False):
        Cb = torch.from_numpy(qrinputs.to_tiles(C, nb)).to(DEV)
        (tq.apply_qt if trans else tq.apply_q)(buf, T, Cb, m, n, nb, ib, tree, 1, family)
        got = qrinputs.from_tiles(Cb.cpu().numpy(), p, 2, nb)
        ref = (nu.apply_qt if trans else nu.apply_q)(F, C)
        assert rel(got, ref) <= TOL_R
        assert np.max(np.abs(got - ref)) <= TOL_R * max(1.0, np.max(np.abs(ref)))


def test_config3_tiles_q_properties():
    """configs[3] tile size on a slice of the tall matrix (p = 64, q = 16, nb = 256,
    Greedy TT, ib = 32): the stored Q (V and T at nb = 256) reproduces A and is
    orthonormal, checked on the device with apply_q (cuBLAS fp64 matmuls of the test only)."""
    p, q, nb, ib = 64, 16, 256, 32
    m, n = p * nb, q * nb
    g = torch.Generator(device=DEV).manual_seed(3)
    A = torch.randn(m * n, dtype=torch.float64, device=DEV, generator=g)
    Ad = tq.from_tiled(A, m, n, nb).clone()
    T = tq.tiled_qr(A, m, n, nb, ib, "greedy")
    R = torch.triu(tq.from_tiled(A, m, n, nb)[:n])
    E = torch.zeros(m, n, dtype=torch.float64, device=DEV)
    E[:n] = torch.eye(n, dtype=torch.float64, device=DEV)
    Qb = tq.to_tiled(E, nb)
    tq.apply_q(A, T, Qb, m, n, nb, ib, "greedy")
    Q = tq.from_tiled(Qb, m, n, nb)
    assert (torch.linalg.norm(Ad - Q @ R) / torch.linalg.norm(Ad)).item() <= TOL_QR
    assert torch.linalg.norm(torch.eye(n, dtype=torch.float64, device=DEV) - Q.T @ Q).item() <= TOL_QR
    # Q^T A = [R; 0] through apply_qt
    Cb = tq.to_tiled(Ad, nb)
    tq.apply_qt(A, T, Cb, m, n, nb, ib, "greedy")
    QtA = tq.from_tiled(Cb, m, n, nb)
    assert (torch.linalg.norm(QtA[:n] - R) / torch.linalg.norm(R)).item() <= TOL_QR
    assert (torch.linalg.norm(QtA[n:]) / torch.linalg.norm(R)).item() <= TOL_QR


@pytest.mark.parametrize("tree,family", [("greedy", "TT"), ("flat", "TS"), ("plasma", "TT")])
def test_monolithic_panels_match(tree, family, monkeypatch):
    """TQR_SPLIT=0 runs every panel kernel as one task; results equal the oracle too."""
    monkeypatch.setenv("TQR_SPLIT", "0")
    for (p, q, nb, ib) in [(4, 2, 72, 32), (3, 3, 64, 32)]:
        A = qrinputs.gaussian(p * nb, q * nb, 77 + p)
        compare_with_oracle(A, nb, ib, tree, 2 if tree == "plasma" else 1, family)


def test_config0_greedy_full_checks():
    """configs[0]: Greedy, p=8 x q=4 tiles of nb=32, ib=32, TT kernels."""
    p, q, nb, ib = 8, 4, 32, 32
    m, n = p * nb, q * nb
    A = qrinputs.gaussian(m, n, 0)
    buf, T, F = compare_with_oracle(A, nb, ib, "greedy", 1, "TT")
    Q = gpu_Q(buf, T, m, n, nb, ib, "greedy", 1, "TT")
    R = np.triu(qrinputs.from_tiles(buf.cpu().numpy(), p, q, nb)[:n, :n])
    assert np.linalg.norm(A - Q @ R) / np.linalg.norm(A) <= TOL_QR
    assert np.linalg.norm(np.eye(n) - Q.T @ Q) <= TOL_QR
    # independent unblocked Householder QR (oracle) and LAPACK agree too
    Ru, _ = nu.householder_qr(A)
    assert rel(nu.sign_normalise(R), nu.sign_normalise(Ru)) <= TOL_R


@pytest.mark.parametrize("tree,bs", [("asap", 0), ("grasap", 1)])
def test_factor_parity_asap(tree, bs):
    """The ASAP / Grasap(1) lists (decided by the tiled execution, §3.2) drive the
    same kernels; parity with the oracle on the same lists."""
    for (p, q, nb, ib) in [(8, 4, 32, 32), (6, 3, 20, 8), (4, 2, 72, 32), (3, 3, 64, 32)]:
        A = qrinputs.gaussian(p * nb, q * nb, 4000 + p + q)
        compare_with_oracle(A, nb, ib, tree, bs, "TT")


@pytest.mark.parametrize("tree,bs,family", [("greedy", 1, "TT"), ("fibonacci", 1, "TS"), ("plasma", 3, "TT")])
def test_apply_parity(tree, bs, family):
    p, q, nb, ib = 6, 3, 16, 8
    m, n = p * nb, q * nb
    A = qrinputs.gaussian(m, n, 5)
    buf, T, F = compare_with_oracle(A, nb, ib, tree, bs, family)
    C = qrinputs.gaussian(m, 2 * nb, 6)
    for trans in (True, False):
        Cb = torch.from_numpy(qrinputs.to_tiles(C, nb)).to(DEV)
        (tq.apply_qt if trans else tq.apply_q)(buf, T, Cb, m, n, nb, ib, tree, bs, family)
        got = qrinputs.from_tiles(Cb.cpu().numpy(), p, 2, nb)
        ref = (nu.apply_qt if trans else nu.apply_q)(F, C)
        assert rel(got, ref) <= TOL_R


def test_edge_cases():
    # single tile (GEQRT only), a column of tiles (q=1), nb=1 scalars, zero matrix (tau = 0)
    for (p, q, nb, ib, tree) in [(1, 1, 16, 8, "greedy"), (9, 1, 8, 4, "greedy"), (7, 3, 1, 1, "fibonacci"),
                                 (5, 2, 3, 2, "binary")]:
        A = qrinputs.gaussian(p * nb, q * nb, 11 + p)
        compare_with_oracle(A, nb, ib, tree, 1, "TT")
    Z = np.zeros((4 * 8, 2 * 8))
    buf, T, F = compare_with_oracle(Z, 8, 4, "greedy", 1, "TT")
    assert np.all(T.cpu().numpy() == 0)


def test_structured_zero_columns():
    """Exactly zero columns make x = 0 exactly for some reflectors (tau = 0 path,
    xLARFG's H = I); R stays unique, so it is compared with the oracle. (A
    duplicated column would make the trailing R depend on rounding noise.)"""
    p, q, nb, ib = 4, 2, 8, 4
    A = qrinputs.gaussian(p * nb, q * nb, 3)
    A[:, 3] = 0.0
    A[:, 12] = 0.0
    for tree, fam in (("greedy", "TT"), ("flat", "TS"), ("binary", "TT")):
        buf, T, F = compare_with_oracle(A, nb, ib, tree, 1, fam)
        assert any(np.any(t == 0.0) for t in F.tau.values())


def test_repeat_launch_epochs():
    """The plan's completion flags are epoch-based: repeated launches stay correct."""
    p, q, nb, ib = 6, 3, 16, 8
    A = qrinputs.gaussian(p * nb, q * nb, 9)
    for _ in range(3):
        compare_with_oracle(A, nb, ib, "greedy", 1, "TT")


@pytest.mark.parametrize("tree,bs,family", [("greedy", 1, "TT"), ("fibonacci", 1, "TT"), ("flat", 1, "TT"),
                                            ("plasma", 5, "TT"), ("flat", 1, "TS"), ("plasma", 10, "TS"),
                                            ("asap", 10, "TT")])
def test_config1_full_size_properties(tree, bs, family):
    """configs[1] at full size in the bench's launch configuration: 8000 x 2000,
    nb = 200, ib = 32. The oracle cannot factor it in seconds, so check
    properties that hold at any size plus LAPACK's R (a library special case)."""
    p, q, nb, ib = 40, 10, 200, 32
    m, n = p * nb, q * nb
    A = qrinputs.gaussian(m, n, 2024)
    buf, T = run_gpu(A, nb, ib, tree, bs, family)
    got = qrinputs.from_tiles(buf.cpu().numpy(), p, q, nb)
    R = np.triu(got[:n, :n])
    Rl = np.linalg.qr(A, mode="r")
    assert rel(nu.sign_normalise(R), nu.sign_normalise(Rl)) <= TOL_R
    # A - QR and orthogonality on the device, through apply_q
    Q = gpu_Q(buf, T, m, n, nb, ib, tree, bs, family)
    assert np.linalg.norm(A - Q @ R) / np.linalg.norm(A) <= TOL_QR
    assert np.linalg.norm(np.eye(n) - Q.T @ Q) <= TOL_QR


@pytest.mark.parametrize("q,nb,ib,family", [(3, 64, 32, "TT"), (2, 24, 8, "TT"), (3, 40, 32, "TS"),
                                            (2, 256, 32, "TT"), (3, 200, 32, "TT")])
def test_merge_kernel(q, nb, ib, family):
    """TT merge of two stacked tile-triangular R factors (tree "merge", used by the
    cross-GPU reduction): R equals LAPACK's R of [R1; R2] up to row signs, and
    the stored Q reproduces the input (apply_q on the device)."""
    n = q * nb
    R1 = np.triu(qrinputs.gaussian(n, n, 5))
    R2 = np.triu(qrinputs.gaussian(n, n, 6))
    S = np.asfortranarray(np.vstack([R1, R2]))
    buf, T = run_gpu(S, nb, ib, "merge", 1, family)
    got = qrinputs.from_tiles(buf.cpu().numpy(), 2 * q, q, nb)
    R = np.triu(got[:n])
    Rl = np.linalg.qr(S, mode="r")
    assert rel(nu.sign_normalise(R), nu.sign_normalise(Rl)) <= TOL_R
    Q = gpu_Q(buf, T, 2 * n, n, nb, ib, "merge", 1, family)
    assert np.linalg.norm(S - Q @ R) / np.linalg.norm(S) <= TOL_QR
    assert np.linalg.norm(np.eye(n) - Q.T @ Q) <= TOL_QR


@pytest.mark.parametrize("world,tree,family", [(4, "greedy", "TT"), (3, "fibonacci", "TT"), (2, "flat", "TT"),
                                               (4, "greedy", "TS"), (2, "plasma", "TS")])
def test_tall_skinny_domains_on_one_gpu(world, tree, family):
    """The configs[3] algorithm with `world` domains executed one after another on
    one GPU (independent launches, no inter-kernel waiting): local tiled QR per
    domain, then the binary merge tree of paper_1104_4475_b200.dist; the final R
    equals LAPACK's R of the whole matrix."""
    from paper_1104_4475_b200 import dist as tdist
    p, q, nb, ib = 9, 2, 64, 32
    A = qrinputs.gaussian(p * nb, q * nb, 99)
    Rs = []
    for r in range(world):
        r0, r1 = tdist.domain(p, world, r)
        loc = torch.from_numpy(qrinputs.to_tiles(np.asfortranarray(A[r0 * nb:r1 * nb]), nb)).to(DEV)
        tq.tiled_qr(loc, (r1 - r0) * nb, q * nb, nb, ib, tree, 2 if tree == "plasma" else 1, family)
        Rs.append(tdist.extract_r(loc, r1 - r0, q, nb))
    for pairs in tdist.merge_schedule(world):
        for dst, src in pairs:
            M = tdist.stack_pair(Rs[dst], Rs[src], q, nb)
            tq.tiled_qr(M, 2 * q * nb, q * nb, nb, ib, "merge", 1, "TT")
            Rs[dst] = tdist.top_r(M, q, nb)
    torch.cuda.synchronize()
    R = np.triu(qrinputs.from_tiles(Rs[0].cpu().numpy(), q, q, nb))
    Rl = np.linalg.qr(A, mode="r")
    assert rel(nu.sign_normalise(R), nu.sign_normalise(Rl)) <= TOL_R


@pytest.mark.parametrize("tma", ["0", "1"])
@pytest.mark.parametrize("tree,family", [("greedy", "TT"), ("flat", "TS")])
def test_copy_paths(tree, family, tma, monkeypatch):
    """Both copy paths of the strip updates: TMA tensor copies (default when nb % 8 == 0,
    ib % 8 == 0, nb >= 32) and cp.async (TQR_TMA=0, and every other shape) equal the oracle."""
    monkeypatch.setenv("TQR_TMA", tma)
    for (p, q, nb, ib) in [(4, 2, 72, 32), (3, 3, 64, 32), (6, 3, 40, 8), (3, 2, 200, 32), (6, 3, 20, 8)]:
        A = qrinputs.gaussian(p * nb, q * nb, 123 + p)
        compare_with_oracle(A, nb, ib, tree, 1, family)
        assert tq.last_launch_tma() == (tma == "1" and nb % 8 == 0 and ib % 8 == 0 and nb >= 32)
    A = qrinputs.gaussian(8 * 64, 3 * 64, 7)
    compare_with_oracle(A, 64, 32, "plasma", 3, "TT")


@pytest.mark.parametrize("tree,family", [("greedy", "TT"), ("fibonacci", "TT"), ("flat", "TT"), ("greedy", "TS"),
                                         ("fibonacci", "TS"), ("flat", "TS")])
def test_config2_square_full_size(tree, family):
    """configs[2]: 8000 x 8000 (p = q = 40, nb = 200), Greedy vs Fibonacci vs flat, TT and TS. Checked on the device
    (cuBLAS fp64 matmuls of the test only): ||A - QR|| / ||A||, ||I - Q^T Q||, and
    R against LAPACK's R after row-sign normalisation."""
    p = q = 40
    nb, ib = 200, 32
    m = n = p * nb
    g = torch.Generator(device=DEV).manual_seed(77)
    A = torch.randn(m, n, dtype=torch.float64, device=DEV, generator=g)
    buf = tq.to_tiled(A, nb)
    T = tq.tiled_qr(buf, m, n, nb, ib, tree, 1, family)
    R = torch.triu(tq.from_tiled(buf, m, n, nb))
    Qb = tq.to_tiled(torch.eye(m, dtype=torch.float64, device=DEV), nb)
    tq.apply_q(buf, T, Qb, m, n, nb, ib, tree, 1, family)
    Q = tq.from_tiled(Qb, m, m, nb)
    assert (torch.linalg.norm(A - Q @ R) / torch.linalg.norm(A)).item() <= TOL_QR
    assert torch.linalg.norm(torch.eye(n, dtype=torch.float64, device=DEV) - Q.T @ Q).item() <= TOL_QR
    if "cfg2" not in _LAPACK_R:                       # one LAPACK factorization for all six cases
        _LAPACK_R["cfg2"] = nu.sign_normalise(np.linalg.qr(A.cpu().numpy(), mode="r"))
    assert rel(nu.sign_normalise(R.cpu().numpy()), _LAPACK_R["cfg2"]) <= TOL_R


_LAPACK_R = {}


@pytest.mark.parametrize("family", ["TT", "TS"])
def test_config3_tall_full_size_gram(family):
    """configs[3] as `bench.py --workload tall` runs it on one GPU: 524288 x 4096
    (p = 2048, q = 16, nb = 256), Greedy, TT and TS kernels. The oracle cannot run at this size, so
    check properties that hold at any size: R^T R = A^T A (A = QR with Q
    orthonormal), and R equals the Cholesky factor of A^T A up to row signs."""
    p, q, nb, ib = 2048, 16, 256, 32
    m, n = p * nb, q * nb
    g = torch.Generator(device=DEV).manual_seed(5)
    A = torch.randn(m * n, dtype=torch.float64, device=DEV, generator=g)      # tiled buffer, i.i.d. N(0,1)
    Ad = tq.from_tiled(A, m, n, nb)
    G = Ad.T @ Ad
    del Ad
    tq.tiled_qr(A, m, n, nb, ib, "greedy", 1, family)
    R = torch.triu(tq.from_tiled(A, m, n, nb)[:n])
    err = (torch.linalg.norm(R.T @ R - G) / torch.linalg.norm(G)).item()
    assert err <= 1e-13, err
    # R equals the Cholesky factor of A^T A up to row signs
    Lc = torch.linalg.cholesky(G)
    assert rel(nu.sign_normalise(R.cpu().numpy()), Lc.T.cpu().numpy()) <= TOL_R


def test_host_async_pipeline():
    """tiled_qr_host_async: several pipelined end-to-end calls on pinned host
    buffers give the same factors as the device API (and as the oracle)."""
    p, q, nb, ib = 6, 3, 64, 32
    m, n = p * nb, q * nb
    mats = [qrinputs.gaussian(m, n, 300 + s) for s in range(3)]
    ins = [torch.from_numpy(qrinputs.to_tiles(Ad, nb)).pin_memory() for Ad in mats]
    outs = [(torch.empty(m * n, dtype=torch.float64).pin_memory(),
             torch.empty(tq.t_size(m, n, nb, ib), dtype=torch.float64).pin_memory()) for _ in mats]
    for x, (R_o, T_o), tree in zip(ins, outs, ("greedy", "flat", "fibonacci")):
        tq.tiled_qr_host_async(x.numpy(), R_o.numpy(), T_o.numpy(), m, n, nb, ib, tree)
    tq.host_wait()
    for Ad, (R_o, T_o), tree in zip(mats, outs, ("greedy", "flat", "fibonacci")):
        F = nu.tiled_qr(Ad, nb, ib, schemes.elim_list(tree, p, q), "TT")
        got = qrinputs.from_tiles(R_o.numpy(), p, q, nb)
        assert rel(got, F.A) <= TOL_R
        assert rel(T_o.numpy()[: F.T.size], F.T) <= TOL_R


SCHED_MODES = [{}, {"TQR_WORK_FIRST": "0"}, {"TQR_CHAIN_SPIN": "64"}, {"TQR_PRIO": "1"}, {"TQR_PRIO": "3"},
               {"TQR_LEVELS": "2"}, {"TQR_LOOKAHEAD": "0"}, {"TQR_GRID": "5"}, {"TQR_GRID": "1"}, {"TQR_TMA": "1"},
               {"TQR_FUSE": "1"}]


@pytest.mark.parametrize("tree,bs,family", [("greedy", 1, "TT"), ("plasma", 3, "TS"), ("asap", 1, "TT")])
def test_schedule_invariance(tree, bs, family, monkeypatch):
    """The schedule never changes the arithmetic: every tile is updated by the
    same tasks in the order the graph fixes, so A (R and V) and T must be
    bitwise identical under every scheduling mode (claim order, work-first,
    chain spin, priority rule, number of levels, grid of 1 or 5 CTAs)."""
    p, q, nb, ib = 9, 4, 72, 32
    m, n = p * nb, q * nb
    A = qrinputs.gaussian(m, n, 77)
    ref = None
    for mode in SCHED_MODES:
        for k in ("TQR_WORK_FIRST", "TQR_CHAIN_SPIN", "TQR_PRIO", "TQR_LEVELS", "TQR_LOOKAHEAD", "TQR_GRID", "TQR_TMA",
                  "TQR_FUSE"):
            monkeypatch.delenv(k, raising=False)
        for k, v in mode.items():
            monkeypatch.setenv(k, v)
        buf, T = run_gpu(A, nb, ib, tree, bs, family)
        got = (buf.cpu().numpy(), T.cpu().numpy())
        if ref is None:
            ref = got
            # and the default schedule is itself correct (vs LAPACK's R)
            R = np.triu(qrinputs.from_tiles(got[0], p, q, nb)[:n, :n])
            assert rel(nu.sign_normalise(R), nu.sign_normalise(np.linalg.qr(A, mode="r"))) <= TOL_R
        else:
            assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]), mode


@pytest.mark.parametrize("p,q,nb,tree,tma", [(6, 4, 200, "flat", "1"), (5, 4, 200, "greedy", "1"),
                                             (6, 3, 256, "fibonacci", "1"), (8, 4, 32, "flat", "1"),
                                             (7, 3, 72, "greedy", "0"), (6, 3, 50, "flat", "1"),
                                             (5, 3, 200, "flat", "0")])
def test_fused_unttmqr_bitwise(p, q, nb, tree, tma, monkeypatch):
    """UNMQR + TTMQR fusion (K_UNTTMQR, TQR_FUSE=1; off by default) runs the same
    arithmetic in the same order as the two separate tasks: A (R and V) and T
    are bitwise identical with and without it, on both copy paths, at nb with
    one inner block (32), a ragged last inner block (nb = 200, 72, 50) and nb = 256;
    and the fused result equals the oracle."""
    ib = 32
    A = qrinputs.gaussian(p * nb, q * nb, 900 + p + nb)
    monkeypatch.setenv("TQR_TMA", tma)
    monkeypatch.setenv("TQR_FUSE", "0")
    b0, T0 = run_gpu(A, nb, ib, tree, 1, "TT")
    monkeypatch.setenv("TQR_FUSE", "1")
    b1, T1 = run_gpu(A, nb, ib, tree, 1, "TT")
    assert torch.equal(b0, b1) and torch.equal(T0, T1)
    F = nu.tiled_qr(A, nb, ib, schemes.elim_list(tree, p, q), "TT")
    got = qrinputs.from_tiles(b1.cpu().numpy(), p, q, nb)
    assert rel(got, F.A) <= TOL_R and np.abs(got - F.A).max() <= TOL_R * np.abs(F.A).max()


def test_strip_width_too_wide_is_rejected(monkeypatch):
    """A forced strip width whose C strip does not fit in shared memory fails
    with TQR_EUNSUP and a message, before any launch."""
    monkeypatch.setenv("TQR_WS", "64")
    p, q, nb = 4, 2, 200
    A = torch.zeros(p * q * nb * nb, dtype=torch.float64, device=DEV)
    with pytest.raises(tq.TiledQRError, match="TQR_WS"):
        tq.tiled_qr(A, p * nb, q * nb, nb, 32, "greedy")


def test_misaligned_pointer_is_rejected():
    """A float64 view at an 8-byte (not 16-byte) offset is rejected before any
    launch (the strip loads and stores move 16-byte pairs)."""
    p, q, nb, ib = 4, 2, 16, 8
    base = torch.zeros(p * q * nb * nb + 1, dtype=torch.float64, device=DEV)
    A = base[1:]
    with pytest.raises(tq.TiledQRError, match="aligned"):
        tq.tiled_qr(A, p * nb, q * nb, nb, ib, "greedy")


def test_graph_replay_and_oversized_grid(monkeypatch):
    """The launch epoch lives on the device, so a CUDA-graph replay of a
    factorization is correct every time; a grid request beyond the co-resident
    capacity (TQR_GRID = 4 x SMs) is capped and completes."""
    p, q, nb, ib = 6, 3, 64, 32
    m, n = p * nb, q * nb
    A = qrinputs.gaussian(m, n, 21)
    F = nu.tiled_qr(A, nb, ib, schemes.elim_list("greedy", p, q), "TT")
    src = torch.from_numpy(qrinputs.to_tiles(A, nb)).to(DEV)
    buf = src.clone()
    T = torch.zeros(tq.t_size(m, n, nb, ib), dtype=torch.float64, device=DEV)
    tq.tiled_qr(buf, m, n, nb, ib, "greedy", T=T)          # plan built outside the capture
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        buf.copy_(src)
        with torch.cuda.graph(g, stream=s):
            buf.copy_(src)
            tq.tiled_qr(buf, m, n, nb, ib, "greedy", T=T, stream=s)
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        got = qrinputs.from_tiles(buf.cpu().numpy(), p, q, nb)
        assert rel(got, F.A) <= TOL_R
    monkeypatch.setenv("TQR_GRID", str(4 * torch.cuda.get_device_properties(0).multi_processor_count))
    buf2, T2 = run_gpu(A, nb, ib, "greedy", 1, "TT")
    assert rel(qrinputs.from_tiles(buf2.cpu().numpy(), p, q, nb), F.A) <= TOL_R


class _Mailbox:
    """In-process stand-in for torch.distributed point-to-point (tests only):
    rank threads exchange tensors through queues; every kernel is launched on
    the one default stream, so no kernel ever waits on another."""

    def __init__(self, world):
        import queue
        self.world = world
        self.q = {(s, d): queue.Queue() for s in range(world) for d in range(world)}

    def endpoint(self, rank):
        box = self

        class _End:
            world = box.world

            def __init__(self):
                self.rank = rank

            def send(self, t, dst):
                torch.cuda.synchronize()
                box.q[(rank, dst)].put(t.clone())

            def recv(self, t, src):
                t.copy_(box.q[(src, rank)].get(timeout=120))
                torch.cuda.synchronize()
        return _End()


@pytest.mark.parametrize("world,tree,family", [(2, "greedy", "TT"), (3, "fibonacci", "TT"), (4, "flat", "TT"),
                                               (2, "greedy", "TS"), (3, "flat", "TS")])
def test_distributed_apply_threads(world, tree, family):
    """dist.tall_skinny_qr + dist.apply_qt / apply_q with the CUDA kernels, the ranks
    run as threads on one GPU (mailbox exchange): Q^T [A | X] gives R on top and
    zeros below it for the A columns, least squares matches numpy, Q undoes Q^T."""
    import threading
    from paper_1104_4475_b200 import dist as tdist
    p, q, qc, nb, ib = 10, 2, 3, 64, 32
    n = q * nb
    A = qrinputs.gaussian(p * nb, n, 77)
    B = np.asfortranarray(np.hstack([A, qrinputs.gaussian(p * nb, (qc - q) * nb, 78)]))
    box = _Mailbox(world)
    out, errs = {}, []

    def run(rank):
        try:
            r0, r1 = tdist.domain(p, world, rank)
            A_loc = torch.from_numpy(qrinputs.to_tiles(np.asfortranarray(A[r0 * nb:r1 * nb]), nb)).to(DEV)
            B_loc = torch.from_numpy(qrinputs.to_tiles(np.asfortranarray(B[r0 * nb:r1 * nb]), nb)).to(DEV)
            comm = box.endpoint(rank)
            F = tdist.tall_skinny_qr(A_loc, p, q, nb, ib, tree, 1, family, comm=comm)
            tdist.apply_qt(F, B_loc, qc * nb, comm=comm)
            torch.cuda.synchronize()
            out[f"qtb{rank}"] = qrinputs.from_tiles(B_loc.cpu().numpy(), r1 - r0, qc, nb)
            if rank == 0:
                out["R"] = qrinputs.from_tiles(F.R.cpu().numpy(), q, q, nb)
            tdist.apply_q(F, B_loc, qc * nb, comm=comm)
            torch.cuda.synchronize()
            out[f"back{rank}"] = qrinputs.from_tiles(B_loc.cpu().numpy(), r1 - r0, qc, nb)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(300)
    assert not errs, errs
    QtB = np.vstack([out[f"qtb{r}"] for r in range(world)])
    R = np.triu(out["R"])
    assert np.linalg.norm(QtB[:n, :n] - R) <= 1e-12 * np.linalg.norm(R)
    assert np.linalg.norm(QtB[n:, :n]) <= 1e-12 * np.linalg.norm(A)
    assert np.allclose(np.linalg.norm(QtB, axis=0), np.linalg.norm(B, axis=0), rtol=1e-12)
    x = np.linalg.solve(R, QtB[:n, n:])
    x_ref = np.linalg.lstsq(A, B[:, n:], rcond=None)[0]
    assert np.linalg.norm(x - x_ref) <= 1e-10 * np.linalg.norm(x_ref)
    back = np.vstack([out[f"back{r}"] for r in range(world)])
    assert np.linalg.norm(back - B) <= 1e-12 * np.linalg.norm(B)


def test_concurrent_kernel_on_another_stream():
    """A long kernel holding SMs on another stream (an fp64 GEMM issued just
    before) does not stall the factorization: the first CTA to arrive seeds the
    roots, so the dataflow progresses with whatever CTAs are resident, and the
    result equals the oracle's."""
    p, q, nb, ib = 6, 3, 64, 32
    m, n = p * nb, q * nb
    A = qrinputs.gaussian(m, n, 23)
    F = nu.tiled_qr(A, nb, ib, schemes.elim_list("greedy", p, q), "TT")
    X = torch.randn(6144, 6144, dtype=torch.float64, device=DEV)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    buf = torch.from_numpy(qrinputs.to_tiles(A, nb)).to(DEV)
    T = torch.zeros(tq.t_size(m, n, nb, ib), dtype=torch.float64, device=DEV)
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        Y = X @ X
    with torch.cuda.stream(s2):
        tq.tiled_qr(buf, m, n, nb, ib, "greedy", T=T, stream=s2)
    torch.cuda.synchronize()
    assert torch.isfinite(Y).all()
    assert rel(qrinputs.from_tiles(buf.cpu().numpy(), p, q, nb), F.A) <= TOL_R
