"""B200-native tiled QR of arXiv:1104.4475 — thin Python binding of libtiledqr.so.

Argument marshalling only: every step of the factorization runs in the CUDA
kernels behind the C ABI declared in include/tiledqr.h. There is no CPU
fallback — if the shared library is missing, importing the compute entry
points raises.

Names follow the paper: elim_list (§2.2), critical_path / tiled_times
(§3, Tables 3 and 6), tiled_qr (Algorithm 1 with the TT/TS kernels of
Algorithms 2-3), apply_qt / apply_q.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = [
    "TREES", "FAMILIES", "lib", "elim_list", "critical_path", "tiled_times", "tiled_qr",
    "apply_qt", "apply_q", "tiled_qr_host", "tiled_qr_host_async", "host_wait", "to_tiled", "from_tiled", "t_size", "last_launch_count",
]

TREES = {"flat": 0, "fibonacci": 1, "greedy": 2, "binary": 3, "plasma": 4, "merge": 5, "asap": 6, "grasap": 7}
FAMILIES = {"TT": 0, "TS": 1}

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtiledqr.so")
_lib = None

_I32P = ctypes.POINTER(ctypes.c_int32)
_VP = ctypes.c_void_p
_SIGS = {
    "elim_list": (ctypes.c_int, [ctypes.c_int] * 4 + [_I32P] * 4 + [ctypes.c_int64]),
    "critical_path": (ctypes.c_int64, [ctypes.c_int] * 5),
    "tiled_times": (ctypes.c_int64, [ctypes.c_int] * 5 + [_I32P]),
    "tiled_qr": (ctypes.c_int, [ctypes.c_int] * 7 + [_VP, _VP, _VP]),
    "apply_qt": (ctypes.c_int, [ctypes.c_int] * 7 + [_VP, _VP, _VP, ctypes.c_int, _VP]),
    "apply_q": (ctypes.c_int, [ctypes.c_int] * 7 + [_VP, _VP, _VP, ctypes.c_int, _VP]),
    "tiled_qr_host": (ctypes.c_int, [ctypes.c_int] * 7 + [_VP, _VP, _VP]),
    "tqr_trace_enable": (ctypes.c_int, [ctypes.c_int]),
    "tqr_trace_fetch": (ctypes.c_int64, [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int64]),
    "tqr_trace_graph": (ctypes.c_int64, [_I32P, _I32P, ctypes.c_int64]),
    "tqr_plan_graph": (ctypes.c_int64, [ctypes.c_int] * 9 + [_I32P, ctypes.c_int64, _I32P, _I32P, ctypes.c_int64]),
    "tiled_qr_host_async": (ctypes.c_int, [ctypes.c_int] * 7 + [_VP, _VP, _VP, _VP]),
    "tqr_host_wait": (ctypes.c_int, []),
    "tqr_last_launch_count": (ctypes.c_int, []),
    "tqr_last_launch_tma": (ctypes.c_int, []),
    "tqr_release_plans": (None, []),
    "tqr_last_error": (ctypes.c_char_p, []),
    "tqr_version": (ctypes.c_int, []),
}
EXPORTS = tuple(_SIGS)


class TiledQRError(RuntimeError):
    pass


def lib():
    """Load libtiledqr.so (built in-tree by __graft_entry__.build()). Raises if absent.
    TQR_LIB names another in-tree build of the same library (A/B timing of kernel variants)."""
    global _lib
    if _lib is None:
        path = os.environ.get("TQR_LIB") or LIB_PATH
        if not os.path.exists(path):
            raise TiledQRError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc < 0:
        raise TiledQRError(f"libtiledqr error {rc}: {lib().tqr_last_error().decode()}")
    return rc


def _tree(tree):
    return TREES[tree] if isinstance(tree, str) else int(tree)


def _fam(family):
    return FAMILIES[family] if isinstance(family, str) else int(family)


def _ptr(a):
    return ctypes.cast(a.ctypes.data, _I32P)


# ---------------------------------------------------------------------------
# host-side schemes
# ---------------------------------------------------------------------------
def elim_list(p: int, q: int, tree="greedy", bs: int = 1):
    """Elimination list of `tree` (1-based): arrays i, piv, k, coarse step (include/tiledqr.h)."""
    cap = sum(p - k for k in range(1, min(p, q) + 1))
    i, piv, k, st = (np.zeros(max(cap, 1), np.int32) for _ in range(4))
    n = _check(lib().elim_list(p, q, _tree(tree), bs, _ptr(i), _ptr(piv), _ptr(k), _ptr(st), cap))
    return i[:n], piv[:n], k[:n], st[:n]


def critical_path(p: int, q: int, tree="greedy", bs: int = 1, family="TT") -> int:
    return _check(lib().critical_path(p, q, _tree(tree), bs, _fam(family)))


def tiled_times(p: int, q: int, tree="greedy", bs: int = 1, family="TT"):
    """(critical path, zero_time[p, q]) — Table 3's per-tile zeroing times (0-based array)."""
    z = np.zeros(p * q, np.int32)
    cp = _check(lib().tiled_times(p, q, _tree(tree), bs, _fam(family), _ptr(z)))
    return cp, z.reshape((q, p)).T.copy()


# ---------------------------------------------------------------------------
# device computation (torch CUDA tensors as device memory)
# ---------------------------------------------------------------------------
def t_size(m: int, n: int, nb: int, ib: int) -> int:
    return (m // nb) * (n // nb) * 2 * ib * nb


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dev(t):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TiledQRError("expected a contiguous float64 CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def to_tiled(M, nb: int):
    """Logical m x n torch tensor -> flat tiled buffer (tile (i,k) at (k*p+i)*nb^2, column-major)."""
    m, n = M.shape
    p, q = m // nb, n // nb
    return M.reshape(p, nb, q, nb).permute(2, 0, 3, 1).contiguous().reshape(-1)


def from_tiled(buf, m: int, n: int, nb: int):
    p, q = m // nb, n // nb
    return buf.reshape(q, p, nb, nb).permute(1, 3, 0, 2).reshape(m, n)


def tiled_qr(A, m: int, n: int, nb: int, ib: int = 32, tree="greedy", bs: int = 1, family="TT", T=None,
             stream=None):
    """Factor the tiled fp64 CUDA buffer A (m x n) in place; returns the T buffer."""
    import torch
    if T is None:
        T = torch.zeros(t_size(m, n, nb, ib), dtype=torch.float64, device=A.device)
    _check(lib().tiled_qr(m, n, nb, ib, _tree(tree), bs, _fam(family), _dev(A), _dev(T), _stream(stream)))
    return T


def apply_qt(A, T, C, m: int, n: int, nb: int, ib: int = 32, tree="greedy", bs: int = 1, family="TT",
             nrhs: int | None = None, stream=None):
    nrhs = C.numel() // m if nrhs is None else nrhs
    _check(lib().apply_qt(m, n, nb, ib, _tree(tree), bs, _fam(family), _dev(A), _dev(T), _dev(C), nrhs,
                          _stream(stream)))
    return C


def apply_q(A, T, C, m: int, n: int, nb: int, ib: int = 32, tree="greedy", bs: int = 1, family="TT",
            nrhs: int | None = None, stream=None):
    nrhs = C.numel() // m if nrhs is None else nrhs
    _check(lib().apply_q(m, n, nb, ib, _tree(tree), bs, _fam(family), _dev(A), _dev(T), _dev(C), nrhs,
                         _stream(stream)))
    return C


def tiled_qr_host(A_host: np.ndarray, m: int, n: int, nb: int, ib: int = 32, tree="greedy", bs: int = 1,
                  family="TT", T_host: np.ndarray | None = None, stream=None):
    """End-to-end call on host buffers (tiled layout, float64, C-contiguous 1-D)."""
    if T_host is None:
        T_host = np.empty(t_size(m, n, nb, ib), np.float64)
    assert A_host.dtype == np.float64 and A_host.flags.c_contiguous
    s = _stream(stream) if stream is not None else ctypes.c_void_p(0)
    _check(lib().tiled_qr_host(m, n, nb, ib, _tree(tree), bs, _fam(family), ctypes.c_void_p(A_host.ctypes.data),
                               ctypes.c_void_p(T_host.ctypes.data), s))
    return T_host


def trace_enable(on: bool = True):
    """Diagnostics: record per-task timestamps of subsequent launches."""
    lib().tqr_trace_enable(1 if on else 0)


KIND_NAMES = ["GEQRT", "UNMQR", "TTQRT", "TTMQR", "TSQRT", "TSMQR", "AP_UNMQR", "AP_TTMQR", "AP_TSMQR",
              "GEQRT_B", "GEQRT_U", "TTQRT_B", "TTQRT_U", "TSQRT_B", "TSQRT_U", "UNTTMQR"]


PHASES = ["load", "fix", "mma1", "tri", "mma3", "panel", "trec", "store"]


def trace_fetch():
    """Per-task trace of the last traced launch: structured numpy array."""
    cap = 16 * 4_000_000
    buf = np.zeros(cap, np.uint64)
    n = _check(lib().tqr_trace_fetch(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), cap))
    r = buf[: 16 * n].reshape(n, 16).astype(np.int64)
    dt = [("taken", "i8"), ("ready", "i8"), ("done", "i8"), ("sm", "i4"), ("kind", "i4"), ("i", "i4"),
          ("piv", "i4"), ("k", "i4"), ("j", "i4"), ("s", "i4")] + [(f"c_{p}", "i8") for p in PHASES]
    out = np.zeros(n, dtype=dt)
    out["taken"], out["ready"], out["done"], out["sm"], out["kind"] = r[:, 0], r[:, 1], r[:, 2], r[:, 3], r[:, 4]
    out["i"], out["piv"] = r[:, 5] & 0xFFFF, (r[:, 5] >> 16) & 0xFFFF
    out["k"], out["j"], out["s"] = r[:, 6] & 0xFFFF, (r[:, 6] >> 16) & 0xFFFF, r[:, 7]
    for x, p in enumerate(PHASES):
        out[f"c_{p}"] = r[:, 8 + x]
    return out


def trace_graph(ntask: int):
    """Successor CSR (ptr, idx) of the last traced plan (diagnostics)."""
    cap = max(ntask + 1, 8 * ntask + 16)
    ptr = np.zeros(cap, np.int32)
    idx = np.zeros(cap, np.int32)
    n = _check(lib().tqr_trace_graph(_ptr(ptr), _ptr(idx), cap))
    return ptr[: ntask + 1].copy(), idx[:n].copy()


def plan_graph(m: int, n: int, nb: int, ib: int = 32, tree="greedy", bs: int = 1, family="TT", ws: int = 0,
               split: bool = True, mstrip: int = 0, fuse=None):
    """Host-only diagnostic: the device task graph (tasks[ntask, 8], succ_ptr, succ).
    tasks[:, 5] = strip | (strips of the task << 16); mstrip = strips per update task (0: the default);
    fuse = UNMQR + TTMQR fusion (None: the library default, TQR_FUSE)."""
    fz = 0 if fuse is None else (2 if fuse else 4)
    args = (m, n, nb, ib, _tree(tree), bs, _fam(family), ws, (1 if split else 0) | fz | (mstrip << 8))
    nt = _check(lib().tqr_plan_graph(*args, None, 0, None, None, 0))
    tasks = np.zeros(8 * nt, np.int32)
    ptr = np.zeros(nt + 1, np.int32)
    cap = 16 * nt + 16
    succ = np.zeros(cap, np.int32)
    _check(lib().tqr_plan_graph(*args, _ptr(tasks), tasks.size, _ptr(ptr), _ptr(succ), cap))
    return tasks.reshape(nt, 8), ptr, succ[: ptr[-1]].copy()


def tiled_qr_host_async(A_host: np.ndarray, R_host: np.ndarray, T_host: np.ndarray, m: int, n: int, nb: int,
                        ib: int = 32, tree="greedy", bs: int = 1, family="TT", stream=None):
    """Pipelined end-to-end call (pinned host buffers): upload, factor, download, no wait."""
    for b in (A_host, R_host, T_host):
        assert b.dtype == np.float64 and b.flags.c_contiguous
    s = _stream(stream) if stream is not None else ctypes.c_void_p(0)
    _check(lib().tiled_qr_host_async(m, n, nb, ib, _tree(tree), bs, _fam(family), ctypes.c_void_p(A_host.ctypes.data),
                                     ctypes.c_void_p(R_host.ctypes.data), ctypes.c_void_p(T_host.ctypes.data), s))


def host_wait():
    _check(lib().tqr_host_wait())


def last_launch_count() -> int:
    return lib().tqr_last_launch_count()


def last_launch_tma() -> bool:
    return bool(lib().tqr_last_launch_tma())
