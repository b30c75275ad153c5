"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no Householder, no trees, no
schedules): it only draws the i.i.d. N(0,1) fp64 matrices that BASELINE.json's
configs name ("entries i.i.d. N(0,1) from seed") and converts between the
LAPACK column-major view and the tiled view, which is pure data movement.

Tiled layout: tile (i,k) (0-based) of a p x q tile matrix with
tile size nb is stored contiguously, column-major inside the tile, at element
offset (k*p + i) * nb*nb.
"""
from __future__ import annotations

import numpy as np


def gaussian(m: int, n: int, seed: int) -> np.ndarray:
    """m x n fp64 matrix, entries i.i.d. N(0,1), Fortran (column-major) order."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.asfortranarray(rng.standard_normal((m, n)))


def to_tiles(a: np.ndarray, nb: int) -> np.ndarray:
    """Column-major m x n matrix -> flat tiled buffer (p*q*nb*nb,) as described above."""
    m, n = a.shape
    assert m % nb == 0 and n % nb == 0
    p, q = m // nb, n // nb
    out = np.empty(p * q * nb * nb, dtype=np.float64)
    for k in range(q):
        for i in range(p):
            off = (k * p + i) * nb * nb
            out[off:off + nb * nb] = a[i * nb:(i + 1) * nb, k * nb:(k + 1) * nb].ravel(order="F")
    return out


def from_tiles(t: np.ndarray, p: int, q: int, nb: int) -> np.ndarray:
    """Inverse of to_tiles."""
    a = np.empty((p * nb, q * nb), dtype=np.float64, order="F")
    for k in range(q):
        for i in range(p):
            off = (k * p + i) * nb * nb
            a[i * nb:(i + 1) * nb, k * nb:(k + 1) * nb] = t[off:off + nb * nb].reshape((nb, nb), order="F")
    return a
