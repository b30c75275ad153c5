// Device side of the tiled QR: the persistent dataflow kernel and the tile
// kernels of Table 1 as CTA-wide routines.
//
// Conventions: tile (i,k) (0-based) of the p x q tile matrix starts at
// element (k*p + i)*nb*nb and is column-major (ld = nb). Reflectors follow
// LAPACK xLARFG: H = I - tau v v^T, beta = -sign(alpha) ||(alpha, x)||,
// tau = (beta - alpha)/beta, v = x / (alpha - beta); tau = 0 when x = 0.
// A block of <= ib reflectors is applied in compact-WY form
// Q_b = I - V T V^T (lines 62-66; forward column-wise T).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "plan.h"

namespace tqr {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxNb = 256;
constexpr int kMaxIb = 32;
constexpr size_t kMaxSmem = 227 * 1024 - 512;   // dynamic smem budget (opt-in max minus static)
constexpr int kTld = 33;                    // ld of the 32 x 32 smem T / top / G blocks
constexpr int kPanelScratch = 2 * 32 * kTld + kWarps * 32 + 4 * 32 + 8;

struct RunArgs {
  const DevTask *tasks;
  const int32_t *deps;
  int ntask;
  int *done;     // per-task completion epoch
  int *ctrl;     // [0] next task, [1] exited CTAs
  int epoch;
  int nctas;
  double *A, *T, *C;
  int p, q, nb, ib, ws, trans;
};

struct SmemLayout {
  int ldc, ldv;
  size_t offC, offV, offW, offT, total;   // in doubles
};

__host__ __device__ inline int odd_ld(int n) { return n | 1; }

__host__ __device__ inline SmemLayout smem_layout(int nb, int ib, int ws) {
  SmemLayout s;
  s.ldc = odd_ld(2 * nb);
  s.ldv = odd_ld(nb);
  size_t c = (size_t)s.ldc * ws;
  size_t v = (size_t)s.ldv * ib;
  size_t w = (size_t)2 * 32 * ws;
  if (w < (size_t)kPanelScratch) w = kPanelScratch;
  s.offC = 0;
  s.offV = c;
  s.offW = c + v;
  s.offT = c + v + w;
  s.total = s.offT + 32 * kTld;
  return s;
}

inline size_t smem_bytes(int nb, int ib, int ws) { return smem_layout(nb, ib, ws).total * sizeof(double); }

#ifdef __CUDACC__

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double *tile_ptr(double *base, int p, int nb, int i, int k) {
  return base + ((size_t)k * p + i) * (size_t)nb * nb;
}
__device__ __forceinline__ double *tslot_ptr(double *T, int p, int nb, int ib, int i, int k, int s) {
  return T + (((size_t)k * p + i) * 2 + s) * (size_t)ib * nb;
}

// ---- strip movement: rows [r0, r1) of tile columns [c0, c0+wsz) <-> buf rows (off + r)
__device__ __forceinline__ void load_rows(double *buf, int ldc, int off, const double *tile, int nb,
                                          int r0, int r1, int c0, int wsz) {
  const int nr = r1 - r0;
  for (int idx = threadIdx.x; idx < nr * wsz; idx += kThreads) {
    int r = r0 + idx % nr, c = idx / nr;
    buf[off + r + c * ldc] = __ldcg(tile + r + (size_t)(c0 + c) * nb);
  }
}
__device__ __forceinline__ void store_rows(const double *buf, int ldc, int off, double *tile, int nb,
                                           int r0, int r1, int c0, int wsz) {
  const int nr = r1 - r0;
  for (int idx = threadIdx.x; idx < nr * wsz; idx += kThreads) {
    int r = r0 + idx % nr, c = idx / nr;
    tile[r + (size_t)(c0 + c) * nb] = buf[off + r + c * ldc];
  }
}

// V of a GEQRT block (columns j0..j0+bw-1 of tile X): rows j0..nb-1, unit
// diagonal, zeros above; stored at Vbuf[(r - j0) + l*ldv].
__device__ __forceinline__ void load_v_geqrt(double *V, int ldv, const double *X, int nb, int j0, int bw) {
  const int nr = nb - j0;
  for (int idx = threadIdx.x; idx < nr * bw; idx += kThreads) {
    int rr = idx % nr, l = idx / nr;
    double v = 0.0;
    if (rr == l) v = 1.0;
    else if (rr > l) v = __ldcg(X + (j0 + rr) + (size_t)(j0 + l) * nb);
    V[rr + l * ldv] = v;
  }
}
// V2 of a TTQRT (tri) / TSQRT block: rows 0..R2-1 of tile X, R2 = j0+bw (TT) or nb (TS);
// in TT only the upper triangle (r <= j0+l) belongs to the reflectors.
__device__ __forceinline__ void load_v_tp(double *V, int ldv, const double *X, int nb, int j0, int bw, bool tri) {
  const int nr = tri ? j0 + bw : nb;
  for (int idx = threadIdx.x; idx < nr * bw; idx += kThreads) {
    int r = idx % nr, l = idx / nr;
    V[r + l * ldv] = (!tri || r <= j0 + l) ? __ldcg(X + r + (size_t)(j0 + l) * nb) : 0.0;
  }
}
__device__ __forceinline__ void load_t(double *Ts, const double *Tslot, int ib, int j0, int bw) {
  for (int idx = threadIdx.x; idx < bw * bw; idx += kThreads) {
    int l = idx % bw, c = idx / bw;
    Ts[l + c * kTld] = l <= c ? __ldcg(Tslot + l + (size_t)(j0 + c) * ib) : 0.0;
  }
}

// ---- apply one compact-WY block to a strip held in shared memory ----------
// W = [Ctop +] V^T Cv ; W2 = op(T) W ; Cv -= V W2 ; [Ctop -= W2]
// trans: op(T) = T^T (applies Q_b^T), else T (applies Q_b).
// Ctop (bw rows, may be null) carries the implicit identity part of
// V = [I; V2] (TT/TS kernels). All arrays in smem, column-major.
__device__ void apply_block(double *Ctop, double *Cv, int ldc, int nrows, const double *V, int ldv,
                            const double *Ts, int bw, int wsz, bool trans, double *W, double *W2) {
  for (int idx = threadIdx.x; idx < bw * wsz; idx += kThreads) {
    int l = idx % bw, c = idx / bw;
    double s = Ctop ? Ctop[l + c * ldc] : 0.0;
    const double *v = V + l * ldv;
    const double *cc = Cv + c * ldc;
    for (int r = 0; r < nrows; ++r) s = fma(v[r], cc[r], s);
    W[l + c * 32] = s;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < bw * wsz; idx += kThreads) {
    int l = idx % bw, c = idx / bw;
    double s = 0.0;
    if (trans) {
      for (int m = 0; m <= l; ++m) s = fma(Ts[m + l * kTld], W[m + c * 32], s);
    } else {
      for (int m = l; m < bw; ++m) s = fma(Ts[l + m * kTld], W[m + c * 32], s);
    }
    W2[l + c * 32] = s;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nrows * wsz; idx += kThreads) {
    int r = idx % nrows, c = idx / nrows;
    double s = 0.0;
    for (int l = 0; l < bw; ++l) s = fma(V[r + l * ldv], W2[l + c * 32], s);
    Cv[r + c * ldc] -= s;
  }
  if (Ctop) {
    for (int idx = threadIdx.x; idx < bw * wsz; idx += kThreads) {
      int l = idx % bw, c = idx / bw;
      Ctop[l + c * ldc] -= W2[l + c * 32];
    }
  }
  __syncthreads();
}

// ---- warp reduce-scatter: lane l ends with sum over lanes of v[l] (v[0]) ----
template <int OFF>
__device__ __forceinline__ void rs_step(double (&v)[32], int lane) {
  const bool hi = lane & OFF;
#pragma unroll
  for (int i = 0; i < OFF; ++i) {
    double keep = hi ? v[i + OFF] : v[i];
    double send = hi ? v[i] : v[i + OFF];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);
  }
}

// ---- panel factorization of one inner block --------------------------------
// MODE 0 = GEQRT on tile X (rows j0..nb-1, pivot row j0+c for column c)
// MODE 1 = TTQRT: pivot rows = A1 rows j0..j0+bw-1 (triangle), eliminated
//          rows = A2 rows 0..j0+c (triangle)           (Table 1)
// MODE 2 = TSQRT: eliminated rows = all nb rows of A2 (line 246)
// Each thread owns one eliminated row in registers; one fused block
// reduction per column produces ||x||^2, the dot products of the update and
// the V^T v column of the T recurrence. Writes R/V back (only the parts this
// kernel owns), fills Vbuf (for the trailing update) and Ts, stores T.
template <int MODE>
__device__ void panel_block(double *X, double *A1, double *Tslot, int nb, int ib, int j0, int bw,
                            double *Vbuf, int ldv, double *Ts, double *scratch) {
  double *top = scratch;               // 32 x 33 (TT/TS pivot rows)
  double *G = top + 32 * kTld;         // 32 x 33, G[m + c*33] = V_m^T v_c
  double *red = G + 32 * kTld;         // kWarps x 32
  double *prow = red + kWarps * 32;    // pivot row (GEQRT)
  double *wv = prow + 32;
  double *taus = wv + 32;
  double *sc = taus + 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row = MODE == 0 ? j0 + tid : tid;
  const bool valid = MODE == 0 ? row < nb : (MODE == 1 ? row < j0 + bw : row < nb);

  double a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    a[c] = 0.0;
    if (valid && c < bw && (MODE != 1 || row <= j0 + c)) a[c] = __ldcg(X + row + (size_t)(j0 + c) * nb);
  }
  if (MODE != 0) {
    for (int idx = tid; idx < 32 * 32; idx += kThreads) {
      int l = idx & 31, c = idx >> 5;
      top[l + c * kTld] = (l < bw && c < bw && l <= c) ? __ldcg(A1 + (j0 + l) + (size_t)(j0 + c) * nb) : 0.0;
    }
  }
  __syncthreads();

#pragma unroll
  for (int c = 0; c < 32; ++c) {
    if (c < bw) {
      const int pr = j0 + c;
      if (MODE == 0 && row == pr) {
#pragma unroll
        for (int l = 0; l < 32; ++l) prow[l] = a[l];
      }
      const bool part = valid && (MODE == 0 ? row > pr : (MODE == 1 ? row <= pr : true));
      const double x = part ? a[c] : 0.0;
      double v[32];
#pragma unroll
      for (int l = 0; l < 32; ++l) v[l] = x * a[l];
      rs_step<16>(v, lane);
      rs_step<8>(v, lane);
      rs_step<4>(v, lane);
      rs_step<2>(v, lane);
      rs_step<1>(v, lane);
      red[warp * 32 + lane] = v[0];
      __syncthreads();
      if (warp == 0) {
        double tot = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) tot += red[w * 32 + lane];
        const double Pl = MODE == 0 ? prow[lane] : top[c + lane * kTld];
        const double alpha = __shfl_sync(0xffffffffu, Pl, c);
        const double xn2 = __shfl_sync(0xffffffffu, tot, c);
        double tau, scale, beta;
        if (xn2 == 0.0) {
          tau = 0.0; scale = 0.0; beta = alpha;
        } else {
          const double xn = sqrt(xn2);
          beta = -copysign(hypot(alpha, xn), alpha);
          tau = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
        if (lane > c && lane < bw) {
          const double w = Pl + scale * tot;
          wv[lane] = w;
          if (MODE != 0) top[c + lane * kTld] = Pl - tau * w;
        }
        if (lane < c) G[lane + c * kTld] = (MODE == 0 ? Pl : 0.0) + scale * tot;
        if (lane == c) {
          taus[c] = tau;
          sc[0] = scale; sc[1] = tau; sc[2] = beta;
          if (MODE != 0) top[c + c * kTld] = beta;
        }
      }
      __syncthreads();
      const double scale = sc[0], tau = sc[1];
      if (part) {
        const double vr = scale * x;
        const double tv = tau * vr;
        a[c] = vr;
#pragma unroll
        for (int l = c + 1; l < 32; ++l)
          if (l < bw) a[l] -= tv * wv[l];
      } else if (MODE == 0 && row == pr) {
        a[c] = sc[2];
#pragma unroll
        for (int l = c + 1; l < 32; ++l)
          if (l < bw) a[l] -= tau * wv[l];
      }
    }
  }

  // write back what this kernel owns + the V buffer of the trailing update
  if (valid) {
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      if (c < bw) {
        if (MODE == 0) {
          X[row + (size_t)(j0 + c) * nb] = a[c];
          const int rr = row - j0;
          Vbuf[rr + c * ldv] = rr == c ? 1.0 : (rr > c ? a[c] : 0.0);
        } else {
          if (MODE == 2 || row <= j0 + c) X[row + (size_t)(j0 + c) * nb] = a[c];
          Vbuf[row + c * ldv] = a[c];
        }
      }
    }
  }
  if (MODE != 0) {
    for (int idx = tid; idx < bw * bw; idx += kThreads) {
      int l = idx % bw, c = idx / bw;
      if (l <= c) A1[(j0 + l) + (size_t)(j0 + c) * nb] = top[l + c * kTld];
    }
  }
  // T recurrence: T[c][c] = tau_c, T[0:c, c] = -tau_c T[0:c, 0:c] G[0:c, c]
  if (warp == 0) {
    for (int c = 0; c < bw; ++c) {
      double t = 0.0;
      if (lane < c)
        for (int m = lane; m < c; ++m) t = fma(Ts[lane + m * kTld], G[m + c * kTld], t);
      __syncwarp();
      if (lane < c) Ts[lane + c * kTld] = -taus[c] * t;
      else if (lane == c) Ts[c + c * kTld] = taus[c];
      else Ts[lane + c * kTld] = 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
  for (int idx = tid; idx < ib * bw; idx += kThreads) {
    int l = idx % ib, c = idx / ib;
    Tslot[l + (size_t)(j0 + c) * ib] = (l < bw && l <= c) ? Ts[l + c * kTld] : 0.0;
  }
}

// ---- panel kernels: GEQRT / TTQRT / TSQRT on whole tiles ------------------
template <int MODE>
__device__ void panel_task(double *X, double *A1, double *Tslot, int nb, int ib, int ws, double *smem,
                           const SmemLayout &L) {
  double *Cb = smem + L.offC, *Vb = smem + L.offV, *Wb = smem + L.offW, *Ts = smem + L.offT;
  for (int j0 = 0; j0 < nb; j0 += ib) {
    const int bw = min(ib, nb - j0);
    panel_block<MODE>(X, A1, Tslot, nb, ib, j0, bw, Vb, L.ldv, Ts, Wb);
    // trailing update of columns j0+bw..nb-1 with Q_b^T
    for (int cs = j0 + bw; cs < nb; cs += ws) {
      const int wsz = min(ws, nb - cs);
      __syncthreads();
      if (MODE == 0) {
        load_rows(Cb, L.ldc, 0, X, nb, j0, nb, cs, wsz);
        __syncthreads();
        apply_block(nullptr, Cb + j0, L.ldc, nb - j0, Vb, L.ldv, Ts, bw, wsz, true, Wb, Wb + 32 * ws);
        store_rows(Cb, L.ldc, 0, X, nb, j0, nb, cs, wsz);
      } else {
        const int r2 = MODE == 1 ? j0 + bw : nb;
        load_rows(Cb, L.ldc, 0, A1, nb, j0, j0 + bw, cs, wsz);
        load_rows(Cb, L.ldc, nb, X, nb, 0, r2, cs, wsz);
        __syncthreads();
        apply_block(Cb + j0, Cb + nb, L.ldc, r2, Vb, L.ldv, Ts, bw, wsz, true, Wb, Wb + 32 * ws);
        store_rows(Cb, L.ldc, 0, A1, nb, j0, j0 + bw, cs, wsz);
        store_rows(Cb, L.ldc, nb, X, nb, 0, r2, cs, wsz);
      }
    }
    __syncthreads();
  }
}

// ---- update kernels on one column strip -----------------------------------
// UNMQR: C (tile strip) <- Q^T C with the GEQRT reflectors of tile Vt
__device__ void unmqr_strip(const double *Vt, const double *Tslot, double *Ct, int nb, int ib, int cs,
                            int wsz, bool trans, int ws, double *smem, const SmemLayout &L) {
  double *Cb = smem + L.offC, *Vb = smem + L.offV, *Wb = smem + L.offW, *Ts = smem + L.offT;
  load_rows(Cb, L.ldc, 0, Ct, nb, 0, nb, cs, wsz);
  const int nblk = (nb + ib - 1) / ib;
  for (int t = 0; t < nblk; ++t) {
    const int b = trans ? t : nblk - 1 - t;
    const int j0 = b * ib, bw = min(ib, nb - j0);
    load_v_geqrt(Vb, L.ldv, Vt, nb, j0, bw);
    load_t(Ts, Tslot, ib, j0, bw);
    __syncthreads();
    apply_block(nullptr, Cb + j0, L.ldc, nb - j0, Vb, L.ldv, Ts, bw, wsz, trans, Wb, Wb + 32 * ws);
  }
  store_rows(Cb, L.ldc, 0, Ct, nb, 0, nb, cs, wsz);
}

// TTMQR / TSMQR: [C1; C2] <- Q^T [C1; C2] with the TTQRT/TSQRT reflectors V2 of tile Vt
__device__ void tpmqr_strip(const double *Vt, const double *Tslot, double *C1, double *C2, int nb, int ib,
                            int cs, int wsz, bool tri, bool trans, int ws, double *smem, const SmemLayout &L) {
  double *Cb = smem + L.offC, *Vb = smem + L.offV, *Wb = smem + L.offW, *Ts = smem + L.offT;
  load_rows(Cb, L.ldc, 0, C1, nb, 0, nb, cs, wsz);
  load_rows(Cb, L.ldc, nb, C2, nb, 0, nb, cs, wsz);
  const int nblk = (nb + ib - 1) / ib;
  for (int t = 0; t < nblk; ++t) {
    const int b = trans ? t : nblk - 1 - t;
    const int j0 = b * ib, bw = min(ib, nb - j0);
    load_v_tp(Vb, L.ldv, Vt, nb, j0, bw, tri);
    load_t(Ts, Tslot, ib, j0, bw);
    __syncthreads();
    apply_block(Cb + j0, Cb + nb, L.ldc, tri ? j0 + bw : nb, Vb, L.ldv, Ts, bw, wsz, trans, Wb, Wb + 32 * ws);
  }
  store_rows(Cb, L.ldc, 0, C1, nb, 0, nb, cs, wsz);
  store_rows(Cb, L.ldc, nb, C2, nb, 0, nb, cs, wsz);
}

__device__ void run_task(const RunArgs &a, const DevTask &t, double *smem, const SmemLayout &L) {
  const int p = a.p, nb = a.nb, ib = a.ib, ws = a.ws;
  switch (t.kind) {
    case K_GEQRT:
      panel_task<0>(tile_ptr(a.A, p, nb, t.i, t.k), nullptr, tslot_ptr(a.T, p, nb, ib, t.i, t.k, 0), nb, ib, ws,
                    smem, L);
      break;
    case K_TTQRT:
      panel_task<1>(tile_ptr(a.A, p, nb, t.i, t.k), tile_ptr(a.A, p, nb, t.piv, t.k),
                    tslot_ptr(a.T, p, nb, ib, t.i, t.k, 1), nb, ib, ws, smem, L);
      break;
    case K_TSQRT:
      panel_task<2>(tile_ptr(a.A, p, nb, t.i, t.k), tile_ptr(a.A, p, nb, t.piv, t.k),
                    tslot_ptr(a.T, p, nb, ib, t.i, t.k, 1), nb, ib, ws, smem, L);
      break;
    case K_UNMQR:
    case K_AP_UNMQR: {
      double *Cbase = t.kind == K_UNMQR ? a.A : a.C;
      const int cs = t.s * ws, wsz = min(ws, nb - cs);
      unmqr_strip(tile_ptr(a.A, p, nb, t.i, t.k), tslot_ptr(a.T, p, nb, ib, t.i, t.k, 0),
                  tile_ptr(Cbase, p, nb, t.i, t.j), nb, ib, cs, wsz, a.trans != 0, ws, smem, L);
      break;
    }
    case K_TTMQR:
    case K_TSMQR:
    case K_AP_TTMQR:
    case K_AP_TSMQR: {
      const bool ap = t.kind == K_AP_TTMQR || t.kind == K_AP_TSMQR;
      const bool tri = t.kind == K_TTMQR || t.kind == K_AP_TTMQR;
      double *Cbase = ap ? a.C : a.A;
      const int cs = t.s * ws, wsz = min(ws, nb - cs);
      tpmqr_strip(tile_ptr(a.A, p, nb, t.i, t.k), tslot_ptr(a.T, p, nb, ib, t.i, t.k, 1),
                  tile_ptr(Cbase, p, nb, t.piv, t.j), tile_ptr(Cbase, p, nb, t.i, t.j), nb, ib, cs, wsz, tri,
                  a.trans != 0, ws, smem, L);
      break;
    }
    default:
      break;
  }
}

// ---- the persistent dataflow kernel ----------------------------------------
// Tasks are taken in the host's topological priority order through one global
// counter; a task waits on the completion flags of its predecessors (all of
// which were taken earlier by running CTAs, so the wait always ends), runs on
// the whole CTA, then publishes its own flag (release / acquire at gpu scope).
__global__ void __launch_bounds__(kThreads, 1) tqr_persistent(RunArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_task;
  const SmemLayout L = smem_layout(a.nb, a.ib, a.ws);
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(&a.ctrl[0], 1);
    __syncthreads();
    const int t = s_task;
    if (t >= a.ntask) break;
    const DevTask tk = a.tasks[t];
    for (int d = tk.dep_begin + threadIdx.x; d < tk.dep_end; d += kThreads) {
      const int *f = a.done + a.deps[d];
      while (ld_acquire(f) != a.epoch) __nanosleep(32);
    }
    __threadfence();
    __syncthreads();
    run_task(a, tk, smem, L);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      st_release(a.done + t, a.epoch);
    }
  }
  if (threadIdx.x == 0) {
    const int n = atomicAdd(&a.ctrl[1], 1);
    if (n == a.nctas - 1) {
      a.ctrl[0] = 0;
      a.ctrl[1] = 0;
      __threadfence();
    }
  }
}

#endif  // __CUDACC__

}  // namespace tqr
