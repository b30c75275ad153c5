"""Multi-GPU tall-skinny tiled QR (BASELINE.json configs[3]).

One process per GPU. The p x q tile matrix is split into contiguous tile-row
domains, one per rank; every rank factors its domain locally with the chosen
tree (`tiled_qr`, no communication). The q x q tile-upper-triangular R factors
of the domains are then reduced by a binary tree across ranks: at level l,
rank r (r mod 2^(l+1) == 0) receives R from rank r + 2^l over NCCL (the only
exchange step of the path) and factors the stacked [R_r; R_src] with the TT
merge scheme (`tiled_qr(..., tree="merge")`, PAPER.md's TT kernels on a
2q x q tile matrix whose lower tiles are structural zeros). Rank 0 ends with
the R of the whole matrix; Q stays distributed (local V/T on every rank plus
the merge V/T on the receiving ranks). `apply_qt` / `apply_q` apply that
distributed Q to a right-hand side B whose tile rows are split by the same
domains (least squares: Q is the product of
the local transformations and the merge transformations, so Q^T B is the
local Q^T on every rank followed by the merge Q^T of each level on the stacked
top q tile rows of the two ranks; Q X runs the same steps in reverse).

This module is marshalling and scheduling only: the factorizations run in
libtiledqr.so. The compute callables are parameters so that the schedule and
the communication can be tested on CPU with the gloo backend.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch
import torch.distributed as dist


def domain(p: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous tile-row domain [r0, r1) of `rank` (sizes differ by at most one)."""
    base, extra = divmod(p, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def merge_schedule(world: int) -> list[list[tuple[int, int]]]:
    """Binary reduction tree over ranks: per level, the (receiver, sender) pairs."""
    levels, step = [], 1
    while step < world:
        levels.append([(r, r + step) for r in range(0, world, 2 * step) if r + step < world])
        step *= 2
    return levels


def extract_r(A_local: torch.Tensor, p_loc: int, q: int, nb: int) -> torch.Tensor:
    """R (top q x q tiles) of a factored local domain as a q x q tiled block, with
    the reflectors below it (strict lower part of diagonal tiles, tiles below
    the diagonal) replaced by the structural zeros the merge expects."""
    tiles = A_local.view(q, p_loc, nb, nb)[:, :q]          # [k][i][c][r] (column-major tiles)
    R = torch.zeros((q, q, nb, nb), dtype=A_local.dtype, device=A_local.device)
    for k in range(q):
        R[k, :k] = tiles[k, :k]
        R[k, k] = torch.tril(tiles[k, k])                 # r <= c in the [c][r] view = upper triangle
    return R.reshape(-1)


def stack_pair(R_top: torch.Tensor, R_bot: torch.Tensor, q: int, nb: int) -> torch.Tensor:
    """[R_top; R_bot] as a 2q x q tiled matrix (tile (i,k) at (k*2q + i)*nb^2)."""
    M = torch.empty((q, 2 * q, nb * nb), dtype=R_top.dtype, device=R_top.device)
    M[:, :q] = R_top.view(q, q, nb * nb)
    M[:, q:] = R_bot.view(q, q, nb * nb)
    return M.reshape(-1)


def top_r(M: torch.Tensor, q: int, nb: int) -> torch.Tensor:
    return M.view(q, 2 * q, nb * nb)[:, :q].contiguous().reshape(-1)


def top_rows(B: torch.Tensor, p_loc: int, q: int, qc: int, nb: int) -> torch.Tensor:
    """The top q tile rows of a p_loc x qc tiled block (a q x qc tiled block, copied)."""
    return B.view(qc, p_loc, nb * nb)[:, :q].contiguous().reshape(-1)


def set_top_rows(B: torch.Tensor, X: torch.Tensor, p_loc: int, q: int, qc: int, nb: int) -> None:
    B.view(qc, p_loc, nb * nb)[:, :q] = X.view(qc, q, nb * nb)


def stack_rows(X_top: torch.Tensor, X_bot: torch.Tensor, q: int, qc: int, nb: int) -> torch.Tensor:
    """[X_top; X_bot] (each q x qc tiles) as a 2q x qc tiled block."""
    M = torch.empty((qc, 2 * q, nb * nb), dtype=X_top.dtype, device=X_top.device)
    M[:, :q] = X_top.view(qc, q, nb * nb)
    M[:, q:] = X_bot.view(qc, q, nb * nb)
    return M.reshape(-1)


def split_rows(M: torch.Tensor, q: int, qc: int, nb: int) -> tuple[torch.Tensor, torch.Tensor]:
    V = M.view(qc, 2 * q, nb * nb)
    return V[:, :q].contiguous().reshape(-1), V[:, q:].contiguous().reshape(-1)


@dataclass
class DistFactor:
    rank: int
    rows: tuple[int, int]                      # tile-row domain
    p: int = 0
    q: int = 0
    nb: int = 0
    ib: int = 32
    tree: str = "greedy"
    bs: int = 1
    family: str = "TT"
    A_local: torch.Tensor | None = None        # the factored local domain (R/V tiles)
    T_local: torch.Tensor | None = None
    merges: list = field(default_factory=list)  # (level, src, M, T) on receiving ranks
    R: torch.Tensor | None = None              # q x q tiled R (rank 0 only, after the reduction)


class DistComm:
    """Point-to-point exchange of the reduction (torch.distributed: NCCL on the
    GPUs, gloo in the CPU tests). Any object with rank, world, send(t, dst) and
    recv(t, src) can stand in (tests/test_gpu_parity.py runs the ranks as
    threads on one GPU with an in-process mailbox)."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def send(self, t, dst):
        dist.send(t, dst, group=self.group)

    def recv(self, t, src):
        dist.recv(t, src, group=self.group)


def _cuda_factor(A, m, n, nb, ib, tree, bs, family):
    from . import tiled_qr
    return tiled_qr(A, m, n, nb, ib, tree, bs, family)


def _cuda_apply(A, T, C, m, n, nb, ib, tree, bs, family, trans):
    from . import apply_q, apply_qt
    (apply_qt if trans else apply_q)(A, T, C, m, n, nb, ib, tree, bs, family)


def tall_skinny_qr(A_local: torch.Tensor, p: int, q: int, nb: int, ib: int = 32, tree="greedy", bs: int = 1,
                   family="TT", group=None, factor=None, sync=None, comm=None) -> DistFactor:
    """Distributed tiled QR of a p x q tile matrix whose tile rows domain(p, world, rank)
    this rank holds in `A_local` (tiled layout with p_loc tile rows)."""
    factor = factor or _cuda_factor
    comm = comm or DistComm(group)
    world, rank = comm.world, comm.rank
    r0, r1 = domain(p, world, rank)
    p_loc = r1 - r0
    assert p_loc >= q, "every domain needs at least q tile rows"
    out = DistFactor(rank=rank, rows=(r0, r1), p=p, q=q, nb=nb, ib=ib, tree=tree, bs=bs, family=family,
                     A_local=A_local)
    out.T_local = factor(A_local, p_loc * nb, q * nb, nb, ib, tree, bs, family)
    R = extract_r(A_local, p_loc, q, nb)
    for level, pairs in enumerate(merge_schedule(world)):
        for dst, src in pairs:
            if rank == src:
                if sync:
                    sync()
                comm.send(R, dst)
                return out
            if rank == dst:
                R_src = torch.empty_like(R)
                comm.recv(R_src, src)
                M = stack_pair(R, R_src, q, nb)
                Tm = factor(M, 2 * q * nb, q * nb, nb, ib, "merge", 1, family)
                out.merges.append((level, src, M, Tm))
                R = top_r(M, q, nb)
    if rank == 0:
        out.R = R
    return out


def _merge_of(F: DistFactor, level: int, src: int):
    for lv, s, M, Tm in F.merges:
        if lv == level and s == src:
            return M, Tm
    raise KeyError(f"rank {F.rank} holds no merge factor for level {level}, source {src}")


def apply_qt(F: DistFactor, B_local: torch.Tensor, nrhs: int, group=None, apply=None, sync=None,
             comm=None) -> torch.Tensor:
    """B <- Q^T B for the distributed factor F (in place on every rank's rows).

    B_local holds this rank's tile rows F.rows of B (tiled, p_loc x qc tiles,
    nrhs = qc nb). Steps: the local Q^T of the domain (apply_qt with the local
    tree); then, level by level of merge_schedule, the sender ships its top q
    tile rows to the receiver, which applies that level's merge Q^T to the
    stacked 2q x qc block, keeps the top half and returns the bottom half (the
    sender's rows of the result). Afterwards rank 0's top q tile rows hold
    (Q^T B)[:n], the rows that meet R in a least-squares solve."""
    apply = apply or _cuda_apply
    comm = comm or DistComm(group)
    world, rank = comm.world, F.rank
    q, nb = F.q, F.nb
    p_loc = F.rows[1] - F.rows[0]
    qc = nrhs // nb
    assert qc * nb == nrhs and B_local.numel() == p_loc * qc * nb * nb
    apply(F.A_local, F.T_local, B_local, p_loc * nb, q * nb, nb, F.ib, F.tree, F.bs, F.family, True)
    top = top_rows(B_local, p_loc, q, qc, nb)
    for level, pairs in enumerate(merge_schedule(world)):
        for dst, src in pairs:
            if rank == src:
                if sync:
                    sync()
                comm.send(top, dst)
                comm.recv(top, dst)
                set_top_rows(B_local, top, p_loc, q, qc, nb)
                return B_local
            if rank == dst:
                other = torch.empty_like(top)
                comm.recv(other, src)
                M, Tm = _merge_of(F, level, src)
                S = stack_rows(top, other, q, qc, nb)
                apply(M, Tm, S, 2 * q * nb, q * nb, nb, F.ib, "merge", 1, F.family, True)
                top, bottom = split_rows(S, q, qc, nb)
                if sync:
                    sync()
                comm.send(bottom, src)
    set_top_rows(B_local, top, p_loc, q, qc, nb)
    return B_local


def apply_q(F: DistFactor, X_local: torch.Tensor, nrhs: int, group=None, apply=None, sync=None,
             comm=None) -> torch.Tensor:
    """X <- Q X for the distributed factor F: the steps of apply_qt in reverse
    order with Q instead of Q^T (merge levels from the last to the first, then
    the local Q of every domain)."""
    apply = apply or _cuda_apply
    comm = comm or DistComm(group)
    world, rank = comm.world, F.rank
    q, nb = F.q, F.nb
    p_loc = F.rows[1] - F.rows[0]
    qc = nrhs // nb
    assert qc * nb == nrhs and X_local.numel() == p_loc * qc * nb * nb
    top = top_rows(X_local, p_loc, q, qc, nb)
    sched = merge_schedule(world)
    for level in range(len(sched) - 1, -1, -1):
        for dst, src in sched[level]:
            if rank == src:
                if sync:
                    sync()
                comm.send(top, dst)
                comm.recv(top, dst)
            elif rank == dst:
                other = torch.empty_like(top)
                comm.recv(other, src)
                M, Tm = _merge_of(F, level, src)
                S = stack_rows(top, other, q, qc, nb)
                apply(M, Tm, S, 2 * q * nb, q * nb, nb, F.ib, "merge", 1, F.family, False)
                top, bottom = split_rows(S, q, qc, nb)
                if sync:
                    sync()
                comm.send(bottom, src)
    set_top_rows(X_local, top, p_loc, q, qc, nb)
    apply(F.A_local, F.T_local, X_local, p_loc * nb, q * nb, nb, F.ib, F.tree, F.bs, F.family, False)
    return X_local
