"""Multi-GPU tall-skinny path: domain split, binary merge
schedule, R extraction / stacking, and the full send/recv reduction over
gloo with world_size 2 and 3 on CPU (no GPU). The local factorizations and
merges are injected as oracle computations (test-only), so these tests check
the distributed logic; the CUDA merge kernel is checked in test_gpu_parity."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import qrinputs
from oracle import numeric as nu
from oracle import schemes
from paper_1104_4475_b200 import dist as tdist


def test_domains_partition():
    for p in (1, 7, 40, 2048):
        for world in (1, 2, 3, 4, 8):
            if world > p:
                continue
            doms = [tdist.domain(p, world, r) for r in range(world)]
            assert doms[0][0] == 0 and doms[-1][1] == p
            assert all(doms[r][1] == doms[r + 1][0] for r in range(world - 1))
            sizes = [b - a for a, b in doms]
            assert max(sizes) - min(sizes) <= 1


def test_merge_schedule_is_a_binary_tree():
    for world in range(1, 17):
        sched = tdist.merge_schedule(world)
        alive = set(range(world))
        for pairs in sched:
            for dst, src in pairs:
                assert dst in alive and src in alive and dst < src
                alive.remove(src)
        assert alive == {0}
        assert len(sched) == (world - 1).bit_length()


def test_extract_and_stack_layout():
    p_loc, q, nb = 5, 3, 4
    A = torch.arange(p_loc * q * nb * nb, dtype=torch.float64)
    R = tdist.extract_r(A, p_loc, q, nb)
    dense_A = qrinputs.from_tiles(A.numpy(), p_loc, q, nb)
    dense_R = qrinputs.from_tiles(R.numpy(), q, q, nb)
    assert np.array_equal(dense_R, np.triu(dense_A[:q * nb]))
    M = tdist.stack_pair(R, 2 * R, q, nb)
    dense_M = qrinputs.from_tiles(M.numpy(), 2 * q, q, nb)
    assert np.array_equal(dense_M[:q * nb], dense_R) and np.array_equal(dense_M[q * nb:], 2 * dense_R)
    assert torch.equal(tdist.top_r(M, q, nb), R)


def merge_list(q):
    """The TT merge scheme of the library (tree "merge"), restated for the oracle."""
    return [(q + t, k, k) for k in range(1, q + 1) for t in range(1, k + 1)]


def oracle_factor(A, m, n, nb, ib, tree, bs, family):
    """Test-only compute backend: the CPU oracle on the tiled buffer, in place."""
    p, q = m // nb, n // nb
    lst = merge_list(q) if tree == "merge" else schemes.elim_list(tree, p, q, bs)
    F = nu.tiled_qr(qrinputs.from_tiles(A.numpy(), p, q, nb), nb, ib, lst, family)
    A.copy_(torch.from_numpy(qrinputs.to_tiles(F.A, nb)))
    return torch.from_numpy(F.T)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, q, nb, ib, tree, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = qrinputs.gaussian(p * nb, q * nb, 31)
        r0, r1 = tdist.domain(p, world, rank)
        A_loc = torch.from_numpy(qrinputs.to_tiles(np.asfortranarray(A[r0 * nb:r1 * nb]), nb))
        out = tdist.tall_skinny_qr(A_loc, p, q, nb, ib, tree, 1, "TT", factor=oracle_factor)
        if rank == 0:
            result["R"] = qrinputs.from_tiles(out.R.numpy(), q, q, nb)
        result[f"merges{rank}"] = len(out.merges)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,tree", [(2, "greedy"), (3, "fibonacci")])
def test_gloo_tall_skinny_reduction(world, tree):
    p, q, nb, ib = 7, 2, 6, 3
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), p, q, nb, ib, tree, result), nprocs=world, join=True)
    A = qrinputs.gaussian(p * nb, q * nb, 31)
    Ru, _ = nu.householder_qr(A)
    R = np.triu(result["R"])
    assert np.linalg.norm(nu.sign_normalise(R) - nu.sign_normalise(Ru)) / np.linalg.norm(Ru) < 1e-12
    assert result["merges0"] == (world - 1).bit_length()


class _OracleQ:
    """Test-only factor handle: the oracle's Factor (its taus replay Q)."""

    def __init__(self, F):
        self.F = F


def oracle_factor_q(A, m, n, nb, ib, tree, bs, family):
    p, q = m // nb, n // nb
    lst = merge_list(q) if tree == "merge" else schemes.elim_list(tree, p, q, bs)
    F = nu.tiled_qr(qrinputs.from_tiles(A.numpy(), p, q, nb), nb, ib, lst, family)
    A.copy_(torch.from_numpy(qrinputs.to_tiles(F.A, nb)))
    return _OracleQ(F)


def oracle_apply(A, H, C, m, n, nb, ib, tree, bs, family, trans):
    """Test-only apply backend: the oracle's apply_qt / apply_q on the tiled C, in place."""
    p = m // nb
    qc = C.numel() // (m * nb)
    dense = qrinputs.from_tiles(C.numpy(), p, qc, nb)
    out = (nu.apply_qt if trans else nu.apply_q)(H.F, dense)
    C.copy_(torch.from_numpy(qrinputs.to_tiles(np.asfortranarray(out), nb)))


def _apply_worker(rank, world, port, p, q, qc, nb, ib, tree, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = qrinputs.gaussian(p * nb, q * nb, 41)
        B = np.asfortranarray(np.hstack([A, qrinputs.gaussian(p * nb, (qc - q) * nb, 42)]))
        r0, r1 = tdist.domain(p, world, rank)
        A_loc = torch.from_numpy(qrinputs.to_tiles(np.asfortranarray(A[r0 * nb:r1 * nb]), nb))
        B_loc = torch.from_numpy(qrinputs.to_tiles(np.asfortranarray(B[r0 * nb:r1 * nb]), nb))
        F = tdist.tall_skinny_qr(A_loc, p, q, nb, ib, tree, 1, "TT", factor=oracle_factor_q)
        tdist.apply_qt(F, B_loc, qc * nb, apply=oracle_apply)
        result[f"qtb{rank}"] = qrinputs.from_tiles(B_loc.numpy(), r1 - r0, qc, nb)
        if rank == 0:
            result["R"] = qrinputs.from_tiles(F.R.numpy(), q, q, nb)
        tdist.apply_q(F, B_loc, qc * nb, apply=oracle_apply)
        result[f"back{rank}"] = qrinputs.from_tiles(B_loc.numpy(), r1 - r0, qc, nb)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,tree", [(2, "greedy"), (3, "flat"), (4, "fibonacci")])
def test_gloo_distributed_apply(world, tree):
    """Q^T and Q of the distributed factor (local factors + merge tree) over gloo:
    Q^T [A | X] puts R in rank 0's top tile rows and zeros below it for the A
    columns (A = QR), preserves column norms (Q orthogonal),
    solves least squares (R x = (Q^T b)[:n] equals numpy's lstsq), and Q undoes Q^T."""
    p, q, qc, nb, ib = 9, 2, 3, 6, 3
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_apply_worker, args=(world, _free_port(), p, q, qc, nb, ib, tree, result), nprocs=world, join=True)
    A = qrinputs.gaussian(p * nb, q * nb, 41)
    B = np.hstack([A, qrinputs.gaussian(p * nb, (qc - q) * nb, 42)])
    QtB = np.vstack([result[f"qtb{r}"] for r in range(world)])
    # rows of Q^T B in the order of the distributed Q: rank 0's top q tile rows are (Q^T B)[:n]
    n = q * nb
    R = np.triu(result["R"])
    top = QtB[:n]
    assert np.linalg.norm(top[:, :n] - R) <= 1e-12 * np.linalg.norm(R)
    rest = np.vstack([QtB[n:]])
    assert np.linalg.norm(rest[:, :n]) <= 1e-12 * np.linalg.norm(A)
    assert np.allclose(np.linalg.norm(QtB, axis=0), np.linalg.norm(B, axis=0), rtol=1e-12)
    x = np.linalg.solve(R, top[:, n:])
    x_ref = np.linalg.lstsq(A, B[:, n:], rcond=None)[0]
    assert np.linalg.norm(x - x_ref) <= 1e-10 * np.linalg.norm(x_ref)
    back = np.vstack([result[f"back{r}"] for r in range(world)])
    assert np.linalg.norm(back - B) <= 1e-12 * np.linalg.norm(B)
