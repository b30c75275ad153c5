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
the merge V/T on the receiving ranks).

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


@dataclass
class DistFactor:
    rank: int
    rows: tuple[int, int]                      # tile-row domain
    T_local: torch.Tensor | None = None
    merges: list = field(default_factory=list)  # (level, src, M, T) on receiving ranks
    R: torch.Tensor | None = None              # q x q tiled R (rank 0 only, after the reduction)


def _cuda_factor(A, m, n, nb, ib, tree, bs, family):
    from . import tiled_qr
    return tiled_qr(A, m, n, nb, ib, tree, bs, family)


def tall_skinny_qr(A_local: torch.Tensor, p: int, q: int, nb: int, ib: int = 32, tree="greedy", bs: int = 1,
                   family="TT", group=None, factor=None, sync=None) -> DistFactor:
    """Distributed tiled QR of a p x q tile matrix whose tile rows domain(p, world, rank)
    this rank holds in `A_local` (tiled layout with p_loc tile rows)."""
    factor = factor or _cuda_factor
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    r0, r1 = domain(p, world, rank)
    p_loc = r1 - r0
    assert p_loc >= q, "every domain needs at least q tile rows"
    out = DistFactor(rank=rank, rows=(r0, r1))
    out.T_local = factor(A_local, p_loc * nb, q * nb, nb, ib, tree, bs, family)
    R = extract_r(A_local, p_loc, q, nb)
    for level, pairs in enumerate(merge_schedule(world)):
        for dst, src in pairs:
            if rank == src:
                if sync:
                    sync()
                dist.send(R, dst, group=group)
                return out
            if rank == dst:
                R_src = torch.empty_like(R)
                dist.recv(R_src, src, group=group)
                M = stack_pair(R, R_src, q, nb)
                Tm = factor(M, 2 * q * nb, q * nb, nb, ib, "merge", 1, family)
                out.merges.append((level, src, M, Tm))
                R = top_r(M, q, nb)
    if rank == 0:
        out.R = R
    return out
