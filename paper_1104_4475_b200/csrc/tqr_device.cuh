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
constexpr int kTld = 33;
constexpr int kTraceWords = 13;             // per-task trace record (diagnostics): 4 stamps/ids, 8 phases, push time
// scheduler control words (ints; each on its own 128-byte line): per priority
// level l a queue head at kCtrlHead + 64 l, its tail at kCtrlTail + 64 l and
// its count of published, unclaimed tasks at kCtrlLevel + 32 l
// kCtrlEpoch holds the launch epoch (1 after upload; the last CTA of a launch
// advances it), kCtrlStart the arrival ticket whose first holder seeds the roots.
constexpr int kCtrlHead = 0, kCtrlTail = 32, kCtrlDone = 64 * kLevels, kCtrlExit = 64 * kLevels + 32,
              kCtrlLevel = 64 * kLevels + 96, kCtrlEpoch = 96 * kLevels + 96, kCtrlStart = 96 * kLevels + 128,
              kCtrlWords = 96 * kLevels + 160;
constexpr int kPanelScratch = 2 * 32 * kTld + 2 * 256 + 8 + 32;

struct RunArgs {
  const DevTask *tasks;
  const int2 *succ;             // successor edges (task, its meta) (CSR, ranges in the task records)
  const int32_t *roots;         // tasks without predecessors
  int nroots;
  int ntask;
  unsigned *cnt;                // per-task arrivals, accumulated over launches (epoch * indegree when ready)
  unsigned long long *queue;    // kLevels ready queues (level kLevels-1 = most critical); level l
                                // owns slots [qoff[l], qoff[l+1]) = one per task of that level
  int qoff[kLevels + 1];
  int *ctrl;                    // kCtrl* counters (incl. the launch epoch, kept on the device so that a
                                // launch that never started, or a graph replay, cannot desynchronise it)
  int nctas;
  double *A, *T, *C;
  int p, q, nb, ib, ws, trans;
  int tma;                     // 1: move C strips and V blocks with 1-D TMA bulk copies
  int work_first;              // 1: a CTA runs the most urgent successor it made ready (not queued)
  int chain_spin;              // polls (128 ns apart) for a chained successor's other inputs
  unsigned long long *trace;   // optional: kTraceWords u64 per task (taken, ready, done, smid<<32|kind, 8 phase cycle counters)
};

struct SmemLayout {
  int ldc, ldv, ldw, wcols, nvb;
  size_t offC, offV[2], offW, offT[2], total;   // in doubles
};

// Leading dimensions are = 4 (mod 16) doubles: the DMMA fragment loads of a
// warp (lanes 4g+t reading element t + g*ld or g + t*ld) then hit 16 distinct
// 8-byte bank pairs per half-warp (conflict-free).
__host__ __device__ inline int ld4(int n) { return n + ((4 - n % 16) + 16) % 16; }
__host__ __device__ inline int round_up(int n, int m) { return (n + m - 1) / m * m; }

// C buffer rows: single-tile strips (UNMQR, GEQRT trailing) use rows 0..nb-1;
// two-tile strips (TTMQR/TSMQR) keep C2 at rows kWinRows.. and stream the 32
// C1 rows of each inner block through two windows at rows 0 and 32.
constexpr int kWinRows = 64;

__host__ __device__ inline SmemLayout smem_layout(int nb, int ib, int ws) {
  SmemLayout s;
  s.wcols = round_up(ws, 8);
  s.ldc = ld4(nb + kWinRows + 16);
  s.ldv = ld4(round_up(nb, 16));
  s.ldw = 36;
  const size_t c = (size_t)s.ldc * s.wcols;
  const size_t v = (size_t)s.ldv * 32;
  size_t w = (size_t)2 * s.ldw * s.wcols;
  if (w < (size_t)kPanelScratch) w = kPanelScratch;
  const size_t tt = 32 * kTld;
  s.nvb = (c + 2 * v + w + 2 * tt) * sizeof(double) <= kMaxSmem ? 2 : 1;   // double-buffer V/T if it fits
  s.offC = 0;
  s.offV[0] = c;
  s.offV[1] = c + v;
  s.offW = c + s.nvb * v;
  s.offT[0] = s.offW + w;
  s.offT[1] = s.offT[0] + tt;
  s.total = s.offT[0] + s.nvb * tt;
  if (s.nvb == 1) { s.offV[1] = s.offV[0]; s.offT[1] = s.offT[0]; }
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

// ---- optional in-task phase profiling (diagnostic tracer) -------------------
// Thread 0 attributes the cycles since the previous mark to a phase slot;
// marks sit right after CTA-wide barriers, so they measure the whole CTA.
__shared__ unsigned long long s_prof[8];
__shared__ unsigned long long s_prof_last;
__shared__ int s_prof_on;
enum { PH_LOAD = 0, PH_FIX, PH_MMA1, PH_TRI, PH_MMA3, PH_PANEL, PH_TREC, PH_STORE };
#ifdef TQR_PANEL_PROF
#define PPROF(slot) prof_mark(slot)
#else
#define PPROF(slot)
#endif
__device__ __forceinline__ void prof_mark(int slot) {
  if (threadIdx.x == 0 && s_prof_on) {
    unsigned long long now = clock64();
    s_prof[slot] += now - s_prof_last;
    s_prof_last = now;
  }
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
__device__ __forceinline__ unsigned smid() {
  unsigned v;
  asm volatile("mov.u32 %0, %smid;" : "=r"(v));
  return v;
}

__device__ __forceinline__ double *tile_ptr(double *base, int p, int nb, int i, int k) {
  return base + ((size_t)k * p + i) * (size_t)nb * nb;
}
__device__ __forceinline__ double *tslot_ptr(double *T, int p, int nb, int ib, int i, int k, int s) {
  return T + (((size_t)k * p + i) * 2 + s) * (size_t)ib * nb;
}

// ---- asynchronous global -> shared copies (LDGSTS) ---------------------------
// All tile data reaches shared memory through cp.async so that every load of a
// task is in flight at once (a scalar load loop is L2-latency bound). The .cg
// (16 B) form bypasses L1; the 8 B form is used only for odd sizes. Writers of
// a tile are ordered before readers by the release/acquire flags plus a
// gpu-scope fence, which also invalidates L1.
__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(double *dst, const double *src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }



// copy rows [r0, r1) of columns [c0, c0+ncol) of a column-major global array
// (leading dimension ldg) to shared dst[(r - r0) + c*lds]
__device__ __forceinline__ void async_block(double *dst, int lds, const double *src, int ldg, int r0, int r1,
                                            int c0, int ncol) {
  const int nr = r1 - r0;
  if (nr <= 0 || ncol <= 0) return;
  const double *g = src + r0 + (size_t)c0 * ldg;
  const bool v16 = ((nr | lds | ldg) & 1) == 0 && ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (v16 && nr <= 4 * 64 && ncol <= 4 * kWarps) {
    // warps over columns, lanes over 16-byte row pairs; nr <= 256 and ncol <= 32
    // always hold here (nb <= kMaxNb), so both loops unroll into predicated
    // copies with constant offsets from one base address per thread
    double *d0 = dst + 2 * lane + warp * lds;
    const double *g0 = g + 2 * lane + (size_t)warp * ldg;
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) {
      if (warp + ci * kWarps < ncol) {
        double *d = d0 + ci * kWarps * lds;
        const double *gs = g0 + (size_t)ci * kWarps * ldg;
#pragma unroll
        for (int ri = 0; ri < 4; ++ri)
          if (2 * lane + 64 * ri < nr) cp_async16(d + 64 * ri, gs + 64 * ri);
      }
    }
  } else if (v16) {   // warps over columns, lanes over 16-byte row pairs (no integer division)
    for (int c = warp; c < ncol; c += kWarps)
      for (int r = 2 * lane; r < nr; r += 64) cp_async16(dst + r + c * lds, g + r + (size_t)c * ldg);   // dst row 0 = r0
  } else {
    for (int c = warp; c < ncol; c += kWarps)
      for (int r = lane; r < nr; r += 32) cp_async8(dst + r + c * lds, g + r + (size_t)c * ldg);
  }
}

// ---- TMA (1-D bulk copies) with an mbarrier transaction count --------------
// One cp.async.bulk per tile column (global column segment -> smem column),
// issued by the lanes of warp 0; completion is tracked by the CTA's mbarrier
// (expect_tx per issue, one arrival per batch, parity wait). The SASS shows
// UBLKCP. Sizes/addresses that are not 16-byte multiples fall back to cp.async.
__shared__ __align__(8) unsigned long long s_mbar;

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init() {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_mbar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// issue column copies rows [r0, r1) of columns [c0, c0+ncol): TMA when every
// column segment is 16-byte aligned and a multiple of 16 bytes, else cp.async
__device__ __forceinline__ void tma_block(double *dst, int lds, const double *src, int ldg, int r0, int r1,
                                          int c0, int ncol, bool use_tma) {
  const int nr = r1 - r0;
  if (nr <= 0 || ncol <= 0) return;
  const double *g = src + r0 + (size_t)c0 * ldg;
  const bool ok = use_tma && ((nr | lds | ldg) & 1) == 0 &&
                  ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (!ok) {
    async_block(dst, lds, src, ldg, r0, r1, c0, ncol);
    return;
  }
  if (threadIdx.x < 32) {
    const unsigned bytes = (unsigned)nr * 8u;
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async;" ::: "memory");
      asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&s_mbar)),
                   "r"(bytes * (unsigned)ncol) : "memory");
    }
    __syncwarp();
    for (int c = threadIdx.x; c < ncol; c += 32)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(dst + c * lds)), "l"(g + (size_t)c * ldg), "r"(bytes), "r"(smem_u32(&s_mbar))
                   : "memory");
  }
}

// wait for every outstanding copy of this batch: cp.async groups and the TMA
// transactions (one arrival + parity wait; `phase` is the per-thread parity)
__device__ __forceinline__ void async_wait(unsigned &phase) {
  cp_async_wait_all();
  if (threadIdx.x == 0) {
    unsigned long long st;
    asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(smem_u32(&s_mbar)) : "memory");
  }
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "TQR_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TQR_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(&s_mbar)), "r"(phase) : "memory");
  phase ^= 1u;
}

// ---- strip movement: rows [r0, r1) of tile columns [c0, c0+wsz) <-> buf rows (off + r)
__device__ __forceinline__ void load_rows(double *buf, int ldc, int off, const double *tile, int nb,
                                          int r0, int r1, int c0, int wsz) {
  async_block(buf + off + r0, ldc, tile, nb, r0, r1, c0, wsz);
}
__device__ __forceinline__ void store_rows(const double *buf, int ldc, int off, double *tile, int nb,
                                           int r0, int r1, int c0, int wsz) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if ((((r1 - r0) | ldc | nb | r0 | off) & 1) == 0 && r1 - r0 <= 4 * 64 && wsz <= 4 * kWarps) {
    // same unrolled, predicated form as async_block (rows <= 256, columns <= 32)
    const int nr = r1 - r0;
    const double *b0 = buf + off + r0 + 2 * lane + warp * ldc;
    double *t0 = tile + r0 + 2 * lane + (size_t)(c0 + warp) * nb;
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) {
      if (warp + ci * kWarps < wsz) {
        const double *b = b0 + ci * kWarps * ldc;
        double *tt = t0 + (size_t)ci * kWarps * nb;
#pragma unroll
        for (int ri = 0; ri < 4; ++ri)
          if (2 * lane + 64 * ri < nr)
            *reinterpret_cast<double2 *>(tt + 64 * ri) = *reinterpret_cast<const double2 *>(b + 64 * ri);
      }
    }
  } else if ((((r1 - r0) | ldc | nb | r0 | off) & 1) == 0) {
    for (int c = warp; c < wsz; c += kWarps)
      for (int r = r0 + 2 * lane; r < r1; r += 64)
        *reinterpret_cast<double2 *>(tile + r + (size_t)(c0 + c) * nb) =
            *reinterpret_cast<const double2 *>(buf + off + r + c * ldc);
  } else {
    for (int c = warp; c < wsz; c += kWarps)
      for (int r = r0 + lane; r < r1; r += 32) tile[r + (size_t)(c0 + c) * nb] = buf[off + r + c * ldc];
  }
}

// V of a GEQRT block (columns j0..j0+bw-1 of tile X): rows j0..nb-1 at
// Vbuf[(r - j0) + l*ldv]. Issued asynchronously; fix_v_geqrt (after the wait)
// sets the unit diagonal, zeros above it and the k4 padding rows.
__device__ __forceinline__ void issue_v_geqrt(double *V, int ldv, const double *X, int nb, int j0, int bw) {
  async_block(V, ldv, X, nb, j0, nb, j0, bw);
}
// (bw <= 32: the column loops unroll into 4 predicated steps per warp)
__device__ __forceinline__ void fix_v_geqrt(double *V, int ldv, int nb, int j0, int bw) {
  const int nr = nb - j0, pad = ((nr + 15) & ~15) - nr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int li = 0; li < 4; ++li) {
    const int l = warp + li * kWarps;
    if (l < bw) {
      if (lane <= l && lane < nr) V[lane + l * ldv] = lane == l ? 1.0 : 0.0;
      if (lane < pad) V[nr + lane + l * ldv] = 0.0;
    }
  }
}
// V2 of a TTQRT (tri) / TSQRT block: rows 0..R2-1 of tile X, R2 = j0+bw (TT) or nb (TS);
// in TT only the upper triangle (r <= j0+l) belongs to the reflectors.
__device__ __forceinline__ void issue_v_tp(double *V, int ldv, const double *X, int nb, int j0, int bw, bool tri) {
  async_block(V, ldv, X, nb, 0, tri ? j0 + bw : nb, j0, bw);
}
__device__ __forceinline__ void fix_v_tp(double *V, int ldv, int nb, int j0, int bw, bool tri) {
  const int nr = tri ? j0 + bw : nb, pad = ((nr + 15) & ~15) - nr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int li = 0; li < 4; ++li) {
    const int l = warp + li * kWarps;
    if (l < bw) {
      if (tri && lane > l && lane < bw) V[j0 + lane + l * ldv] = 0.0;
      if (lane < pad) V[nr + lane + l * ldv] = 0.0;
    }
  }
}
// zero V rows [nr, round_up(nr, 16)) of columns 0..bw-1 (K padding of the DMMA loops)
__device__ __forceinline__ void zero_vpad(double *V, int ldv, int nr, int bw) {
  const int pad = ((nr + 15) & ~15) - nr;
  if (pad > 0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int l = warp; l < bw; l += kWarps)
      if (lane < pad) V[nr + lane + l * ldv] = 0.0;
  }
}
// T block (bw x bw upper triangular) of columns j0.. of a T slot -> Ts (ld kTld);
// the rest of the 32 x 32 block is zeroed (it feeds a padded DMMA)
__device__ __forceinline__ void issue_t(double *Ts, const double *Tslot, int ib, int j0, int bw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *d0 = Ts + lane + warp * kTld;
  const double *g0 = Tslot + lane + (size_t)(j0 + warp) * ib;
#pragma unroll
  for (int ci = 0; ci < 4; ++ci) {
    const int c = warp + ci * kWarps;
    if (lane <= c && c < bw) cp_async8(d0 + ci * kWarps * kTld, g0 + (size_t)ci * kWarps * ib);
    else d0[ci * kWarps * kTld] = 0.0;
  }
}

// ---- FP64 tensor-core MMA (DMMA): D(16x8) += A(16x4) B(4x8) ------------------
// Fragments (lane = 4*g + t): a0 = A[g][t], a1 = A[g+8][t]; b0 = B[t][g];
// d0,d1 = D[g][2t, 2t+1], d2,d3 = D[g+8][2t, 2t+1].
__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// ---- apply one compact-WY block to a strip held in shared memory ----------
// W = [Ctop +] V^T Cv ; W2 = -op(T) W ; Cv += V W2 ; [Ctop += W2]
// trans: op(T) = T^T (applies Q_b^T), else T (applies Q_b).
// Ctop (bw rows, may be null) carries the implicit identity part of
// V = [I; V2] (TT/TS kernels). All arrays in smem, column-major.
// Requirements (kept by the loaders): V rows [nrows, round_up(nrows,4)) are
// zero; everything the m16/n8 padding reads is finite; W/W2 have ldw = 36.
// All three contractions run on the FP64 tensor pipe (mma.sync m16n8k4 f64).
// DMMA latency (~150 cycles) is hidden with several independent accumulator
// chains per warp: K is interleaved over 4 chains in phase 1 and 2 chains in
// phase 2, and phase 3 deals the (m16, n8) fragments round-robin over warps
// (warp w: n-tile w mod NT, m-tiles w / NT + i * 8 / NT).
// Cv += V W2 for NF fragments (m-tiles mfirst, mfirst+MSTEP, ...) of n-tile n
template <int NF, int MSTEP>
__device__ __forceinline__ void phase3_frags(double *Cv, int ldc, int nrows, const double *V, int ldv,
                                             const double *W2, int wsz, int n, int mfirst, int kpad3) {
  constexpr int ldw = 36;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int c0 = n * 8 + 2 * t;
  double acc[NF][4];
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    const int m0 = (mfirst + i * MSTEP) * 16;
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[i][e] = Cv[(m0 + g + (e >> 1) * 8) + (c0 + (e & 1)) * ldc];
  }
  // K = 32 always (W2 rows >= bw are exact zeros); loads of step k+4 overlap the DMMAs of step k
  const double *wb = W2 + t + (n * 8 + g) * ldw;
  const double *vr = V + g + t * ldv + mfirst * 16;
  double b = wb[0], a0[NF], a1[NF];
#pragma unroll
  for (int i = 0; i < NF; ++i) { a0[i] = vr[i * MSTEP * 16]; a1[i] = vr[i * MSTEP * 16 + 8]; }
#pragma unroll
  for (int k = 4; k < 32; k += 4) {
    const double nbv = wb[k];
    double n0[NF], n1[NF];
#pragma unroll
    for (int i = 0; i < NF; ++i) {
      n0[i] = vr[i * MSTEP * 16 + k * ldv];
      n1[i] = vr[i * MSTEP * 16 + 8 + k * ldv];
    }
#pragma unroll
    for (int i = 0; i < NF; ++i) dmma(acc[i], a0[i], a1[i], b);
    b = nbv;
#pragma unroll
    for (int i = 0; i < NF; ++i) { a0[i] = n0[i]; a1[i] = n1[i]; }
  }
#pragma unroll
  for (int i = 0; i < NF; ++i) dmma(acc[i], a0[i], a1[i], b);
  (void)kpad3;
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    const int m0 = (mfirst + i * MSTEP) * 16;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = m0 + g + (e >> 1) * 8, c = c0 + (e & 1);
      if (r < nrows && c < wsz) Cv[r + c * ldc] = acc[i][e];
    }
  }
}

template <int NT>
__device__ void apply_block_t(double *Ctop, double *Cv, int ldc, int nrows, const double *V, int ldv,
                              const double *Ts, int bw, int wsz, bool trans, double *W, double *W2) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  constexpr int ldw = 36;
  const int nt = (wsz + 7) >> 3;
  // phase 1: W (bw x wsz) = V^T Cv, one 16x8 fragment per warp-iteration, full K in 4 chains
  {
    const int mt = (bw + 15) >> 4;
    const int kpad = (nrows + 15) & ~15;        // V rows [nrows, kpad) are zero
    for (int f = warp; f < mt * nt; f += kWarps) {
      // bw <= 32, so mt is 1 or 2: no integer division
      const int m0 = (mt == 2 ? (f & 1) : 0) * 16, n0 = (mt == 2 ? (f >> 1) : f) * 8;
      double acc[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[u][e] = 0.0;
      const double *va = V + (m0 + g) * ldv + t;
      const double *vb = va + 8 * ldv;
      const double *cb = Cv + (n0 + g) * ldc + t;
      // branch-free, software-pipelined: the fragments of step k+16 are loaded
      // while the DMMAs of step k run (DMMAs under a branch do not overlap)
      double fa[4], fb[4], fc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { fa[u] = va[4 * u]; fb[u] = vb[4 * u]; fc[u] = cb[4 * u]; }
      for (int k = 16; k < kpad; k += 16) {
        double na[4], nb2[4], nc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { na[u] = va[k + 4 * u]; nb2[u] = vb[k + 4 * u]; nc[u] = cb[k + 4 * u]; }
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma(acc[u], fa[u], fb[u], fc[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) { fa[u] = na[u]; fb[u] = nb2[u]; fc[u] = nc[u]; }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma(acc[u], fa[u], fb[u], fc[u]);
      const int r0 = m0 + g, c0 = n0 + 2 * t;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = r0 + (e >> 1) * 8, c = c0 + (e & 1);
        double v = (acc[0][e] + acc[1][e]) + (acc[2][e] + acc[3][e]);
        if (Ctop && r < bw && c < wsz) v += Ctop[r + c * ldc];
        W[r + c * ldw] = v;
      }
    }
  }
  __syncthreads();
  prof_mark(PH_MMA1);
  // phase 2: W2 = -op(T) W on the tensor pipe (T is a zero-padded 32 x 32
  // upper triangle, so rows bw..31 of W2 come out exactly zero)
  const int kpad3 = (bw + 3) & ~3;
  for (int f = warp; f < 2 * nt; f += kWarps) {
    const int m0 = (f & 1) * 16, n0 = (f >> 1) * 8;
    double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
    // K = 32 always: T is zero beyond bw, so the padding adds exact zeros
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      double a0, a1;
      if (trans) {   // A[l][m] = T[m][l]
        a0 = Ts[(kk + t) + (m0 + g) * kTld];
        a1 = Ts[(kk + t) + (m0 + g + 8) * kTld];
      } else {       // A[l][m] = T[l][m]
        a0 = Ts[(m0 + g) + (kk + t) * kTld];
        a1 = Ts[(m0 + g + 8) + (kk + t) * kTld];
      }
      dmma(acc[(kk >> 2) & 1], a0, a1, W[(kk + t) + (n0 + g) * ldw]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = m0 + g + (e >> 1) * 8, c = n0 + 2 * t + (e & 1);
      W2[r + c * ldw] = -(acc[0][e] + acc[1][e]);
    }
  }
  __syncthreads();
  prof_mark(PH_TRI);
  // phase 3: Cv (nrows x wsz) += V W2, fragments dealt round-robin; the
  // per-warp fragment count selects a static-trip-count instance
  {
    constexpr int MSTEP = kWarps / NT;
    const int mt = (nrows + 15) >> 4;
    const int n = warp % NT, mfirst = warp / NT;
    const int nf = mt > mfirst ? (mt - mfirst + MSTEP - 1) / MSTEP : 0;
    if (n < nt && nf > 0) {
      switch (nf) {
        case 1: phase3_frags<1, MSTEP>(Cv, ldc, nrows, V, ldv, W2, wsz, n, mfirst, kpad3); break;
        case 2: phase3_frags<2, MSTEP>(Cv, ldc, nrows, V, ldv, W2, wsz, n, mfirst, kpad3); break;
        case 3: phase3_frags<3, MSTEP>(Cv, ldc, nrows, V, ldv, W2, wsz, n, mfirst, kpad3); break;
        case 4: phase3_frags<4, MSTEP>(Cv, ldc, nrows, V, ldv, W2, wsz, n, mfirst, kpad3); break;
        case 5: phase3_frags<5, MSTEP>(Cv, ldc, nrows, V, ldv, W2, wsz, n, mfirst, kpad3); break;
        case 6: phase3_frags<6, MSTEP>(Cv, ldc, nrows, V, ldv, W2, wsz, n, mfirst, kpad3); break;
        case 7: phase3_frags<7, MSTEP>(Cv, ldc, nrows, V, ldv, W2, wsz, n, mfirst, kpad3); break;
        default: phase3_frags<8, MSTEP>(Cv, ldc, nrows, V, ldv, W2, wsz, n, mfirst, kpad3); break;
      }
    }
  }
  if (Ctop) {
    for (int c = warp; c < wsz; c += kWarps)
      if (lane < bw) Ctop[lane + c * ldc] += W2[lane + c * ldw];
  }
  __syncthreads();
  prof_mark(PH_MMA3);
}

__device__ __forceinline__ void apply_block(double *Ctop, double *Cv, int ldc, int nrows, const double *V,
                                            int ldv, const double *Ts, int bw, int wsz, bool trans, double *W,
                                            double *W2) {
  if (wsz <= 32) apply_block_t<4>(Ctop, Cv, ldc, nrows, V, ldv, Ts, bw, wsz, trans, W, W2);
  else apply_block_t<8>(Ctop, Cv, ldc, nrows, V, ldv, Ts, bw, wsz, trans, W, W2);
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

// ---- Householder scalars (xLARFG) from alpha and ||x||^2 ------------------
// beta = -sign(alpha) ||(alpha, x)||, tau = (beta - alpha)/beta, scale =
// 1/(alpha - beta), evaluated with one rsqrt and one reciprocal:
// r = 1/||(alpha,x)||, tau = 1 + |alpha| r, scale = sign(alpha)/(|alpha| + ||.||).
// (Equal to the textbook formulas up to rounding; reading R8.)
__device__ __forceinline__ void larfg_scalars(double alpha, double xn2, double &beta, double &tau, double &scale) {
  if (xn2 == 0.0) {
    beta = alpha; tau = 0.0; scale = 0.0;
    return;
  }
  const double s = fma(alpha, alpha, xn2);
  const double aa = fabs(alpha);
  double nrm, r;
  if (s < 1e-290 || s > 1e290) {          // extreme range: scaled hypot
    nrm = hypot(alpha, sqrt(xn2));
    r = 1.0 / nrm;
  } else {
    r = rsqrt(s);
    nrm = s * r;
  }
  beta = alpha >= 0.0 ? -nrm : nrm;
  tau = fma(aa, r, 1.0);
  const double rs = 1.0 / (aa + nrm);
  scale = alpha >= 0.0 ? rs : -rs;
}

// ---- T from G = V^T V and tau by recursive doubling -------------------------
// Block form of the compact-WY product (lines 62-66): for Q1 Q2 with
// Q_i = I - V_i T_i V_i^T,  T = [[T1, -T1 (V1^T V2) T2], [0, T2]].
// Levels s = 1, 2, 4, 8, 16 merge adjacent diagonal blocks; every level is two
// small triangular products spread over the CTA (one entry per thread).
// Ts must hold tau on the diagonal and zeros elsewhere on entry; X is scratch.
__device__ void t_doubling(double *Ts, const double *G, double *X) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int lg = 0; lg < 5; ++lg) {                     // merge size sz = 2^lg
    const int sz = 1 << lg;
    const int u = tid >> (2 * lg), e = tid & (sz * sz - 1);
    const int i = e & (sz - 1), j = e >> lg;
    const int b0 = 2 * sz * u, b1 = b0 + sz;
    const bool act = tid < 16 * sz;                    // (16/sz) merges of sz*sz entries
    if (act) {                                         // X = G12 T22
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < sz; ++m)
        if (m <= j) acc = fma(G[(b0 + i) + (b1 + m) * kTld], Ts[(b1 + m) + (b1 + j) * kTld], acc);
      X[(b0 + i) + (b1 + j) * kTld] = acc;
    }
    __syncthreads();
    if (act) {                                         // T12 = -T11 X
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < sz; ++m)
        if (m >= i) acc = fma(Ts[(b0 + i) + (b0 + m) * kTld], X[(b0 + m) + (b1 + j) * kTld], acc);
      Ts[(b0 + i) + (b1 + j) * kTld] = -acc;
    }
    __syncthreads();
  }
}

// G (32 x 32, ld kTld) = V^T V for the 32 V columns in Vbuf (rows 0..nr4-1), DMMA
__device__ void gram_v(double *G, const double *V, int ldv, int nr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (warp & 1) * 16, n0 = (warp >> 1) * 8;   // 8 warps = 2 x 4 fragments
  const int kpad = (nr + 15) & ~15;          // rows [nr, kpad) of V are zero
  double acc0[4] = {0.0, 0.0, 0.0, 0.0}, acc1[4] = {0.0, 0.0, 0.0, 0.0};
  const double *va = V + (m0 + g) * ldv + t, *vb = va + 8 * ldv, *vc = V + (n0 + g) * ldv + t;
  for (int k = 0; k < kpad; k += 8) {
    dmma(acc0, va[k], vb[k], vc[k]);
    dmma(acc1, va[k + 4], vb[k + 4], vc[k + 4]);
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) G[(m0 + g + (e >> 1) * 8) + (n0 + 2 * t + (e & 1)) * kTld] = acc0[e] + acc1[e];
}

// ---- panel factorization of one inner block --------------------------------
// MODE 0 = GEQRT on tile X (rows j0..nb-1, pivot row j0+c for column c)
// MODE 1 = TTQRT: pivot rows = A1 rows j0..j0+bw-1 (triangle), eliminated
//          rows = A2 rows 0..j0+c (triangle)           (Table 1)
// MODE 2 = TSQRT: eliminated rows = all nb rows of A2 (line 246)
// Column-cyclic warp ownership: warp w owns panel columns w, w+8, w+16, w+24;
// lane l holds rows l, l+32, ..., l+224 of them in registers (TT/TS: lane l
// also holds pivot row l of each owned column). Reflector c is generated by
// its owner warp alone (warp-local norm, xLARFG scalars), published through
// shared memory, and after ONE barrier every warp applies it to its own
// columns > c (warp-local dot products). The owner of column c+1 can start
// as soon as its column is updated, so the per-column chain is short.
// After the columns: G = V^T V on the tensor pipe and T by recursive
// doubling. Writes R/V back (only the parts this kernel owns), fills Vbuf (for
// a trailing update), Ts and the T slot.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int MODE>
__device__ void panel_block(double *X, double *A1, double *Tslot, int nb, int ib, int j0, int bw,
                            double *Vbuf, int ldv, double *Ts, double *scratch) {
  double *top = scratch;               // 32 x kTld scratch for t_doubling
  double *G = top + 32 * kTld;         // 32 x kTld: V^T V
  double *vsh = G + 32 * kTld;         // 2 x 256: published reflector (double-buffered)
  double *scal = vsh + 2 * 256;        // 2 x 4: tau of the published reflector
  double *taus = scal + 8;             // 32
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nr = MODE == 0 ? nb - j0 : (MODE == 1 ? j0 + bw : nb);   // V rows of this block
  const int rbase = MODE == 0 ? j0 : 0;

  double a[4][8];     // a[q][s]: column warp + 8q, row rbase + lane + 32 s
  double pt[4];       // TT/TS: A1 row j0+lane of column warp + 8q (pivot rows)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int cl = warp + 8 * q;
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2) {
      const int rr = lane + 32 * s2, row = rbase + rr;
      a[q][s2] = (cl < bw && rr < nr && (MODE != 1 || row <= j0 + cl)) ? __ldcg(X + row + (size_t)(j0 + cl) * nb) : 0.0;
    }
    pt[q] = (MODE != 0 && cl < bw && lane <= cl) ? __ldcg(A1 + (j0 + lane) + (size_t)(j0 + cl) * nb) : 0.0;
  }

  double betas[4] = {0.0, 0.0, 0.0, 0.0};   // R diagonal of owned columns (lane c of owner)
  // The column loop is unrolled over the owner's slot qo (c = 8 qo + wo) so the
  // owner reads and writes its column with static register indices.
#pragma unroll
  for (int qo = 0; qo < 4; ++qo) {
#pragma unroll 1
    for (int wo = 0; wo < 8; ++wo) {
      const int c = 8 * qo + wo;
      if (c >= bw) break;
      const int pr = j0 + c;
      double *vb = vsh + (c & 1) * 256;
      if (warp == wo) {
        // ---- generate reflector c from the owned column a[qo][*] ----
        const int first = MODE == 0 ? c + 1 : 0;                 // first participating relative row
        const int last = MODE == 1 ? pr : nr - 1;                // last participating relative row
        double ss = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) {
          const int rr = lane + 32 * s2;
          if (rr >= first && rr <= last) ss = fma(a[qo][s2], a[qo][s2], ss);
        }
        const double xn2 = warp_sum(ss);
        const double alpha = __shfl_sync(0xffffffffu, MODE == 0 ? a[qo][0] : pt[qo], c);
        double beta, tau, scale;
        larfg_scalars(alpha, xn2, beta, tau, scale);
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) {
          const int rr = lane + 32 * s2;
          const bool tl = rr >= first && rr <= last;
          const double v = tl ? scale * a[qo][s2] : 0.0;
          vb[rr] = v;
          if (tl) a[qo][s2] = v;               // column now holds V below the pivot
        }
        if (lane == c) betas[qo] = beta;
        if (lane == 0) { scal[(c & 1) * 4] = tau; taus[c] = tau; }
      }
      __syncthreads();
      // ---- apply reflector c to the owned columns > c ----
      // branch-free over the 4 owned columns so the 4 warp reductions overlap
      const double tau = scal[(c & 1) * 4];
      if (warp + 8 * 3 > c && tau != 0.0) {
        double v[8];
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) v[s2] = vb[lane + 32 * s2];
        double d[4], P[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          d[q] = 0.0;
          if (q >= qo) {               // slots below qo hold finished columns (static skip)
#pragma unroll
            for (int s2 = 0; s2 < 8; ++s2) d[q] = fma(v[s2], a[q][s2], d[q]);
          }
          P[q] = MODE == 0 ? __shfl_sync(0xffffffffu, a[q][0], c) : __shfl_sync(0xffffffffu, pt[q], c);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q >= qo) d[q] += __shfl_xor_sync(0xffffffffu, d[q], o);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q < qo) continue;
          const int cl = warp + 8 * q;
          const double tw = (cl > c && cl < bw) ? tau * (P[q] + d[q]) : 0.0;
#pragma unroll
          for (int s2 = 0; s2 < 8; ++s2) a[q][s2] = fma(-tw, v[s2], a[q][s2]);
          if (lane == c) {
            if (MODE == 0) a[q][0] -= tw;
            else pt[q] -= tw;
          }
        }
      }
    }
  }
  // ---- write back the owned columns: X (R above / V below the pivot) and Vbuf ----
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int cl = warp + 8 * q;
    if (cl < bw) {
      if (MODE != 0 && lane == cl) pt[q] = betas[q];
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) {
        const int rr = lane + 32 * s2, row = rbase + rr;
        if (rr < nr) {
          if (MODE == 0) {
            const double fin = rr == cl ? betas[q] : a[q][s2];
            X[row + (size_t)(j0 + cl) * nb] = fin;
            Vbuf[rr + cl * ldv] = rr == cl ? 1.0 : (rr > cl ? a[q][s2] : 0.0);
          } else {
            const bool part = MODE == 2 || row <= j0 + cl;
            if (part) X[row + (size_t)(j0 + cl) * nb] = a[q][s2];
            Vbuf[rr + cl * ldv] = part ? a[q][s2] : 0.0;
          }
        }
      }
    }
  }
  if (MODE != 0) {     // final pivot rows (R) back to A1, upper triangle of the block
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cl = warp + 8 * q;
      if (cl < bw && lane <= cl) A1[(j0 + lane) + (size_t)(j0 + cl) * nb] = pt[q];
    }
  }
  __syncthreads();
  zero_vpad(Vbuf, ldv, nr, bw);
  for (int idx = tid; idx < 32 * 32; idx += kThreads) {     // Ts = diag(tau) (zero-padded)
    const int l = idx & 31, c = idx >> 5;
    Ts[l + c * kTld] = (l == c && c < bw) ? taus[c] : 0.0;
  }
  __syncthreads();
  prof_mark(PH_PANEL);
  gram_v(G, Vbuf, ldv, nr);
  __syncthreads();
  t_doubling(Ts, G, top);
  prof_mark(PH_TREC);
  for (int c = warp; c < bw; c += kWarps)
    if (lane < ib) Tslot[lane + (size_t)(j0 + c) * ib] = (lane < bw && lane <= c) ? Ts[lane + c * kTld] : 0.0;
}

// ---- panel kernels: GEQRT / TTQRT / TSQRT on whole tiles ------------------
template <int MODE>
__device__ void panel_task(double *X, double *A1, double *Tslot, int nb, int ib, int ws, double *smem,
                           const SmemLayout &L) {
  double *Cb = smem + L.offC, *Vb = smem + L.offV[0], *Wb = smem + L.offW, *Ts = smem + L.offT[0];
  for (int j0 = 0; j0 < nb; j0 += ib) {
    const int bw = min(ib, nb - j0);
    panel_block<MODE>(X, A1, Tslot, nb, ib, j0, bw, Vb, L.ldv, Ts, Wb);
    // trailing update of columns j0+bw..nb-1 with Q_b^T
    for (int cs = j0 + bw; cs < nb; cs += ws) {
      const int wsz = min(ws, nb - cs);
      __syncthreads();
      if (MODE == 0) {
        load_rows(Cb, L.ldc, 0, X, nb, j0, nb, cs, wsz);
        cp_async_wait_all();
        __syncthreads();
        prof_mark(PH_LOAD);
        apply_block(nullptr, Cb + j0, L.ldc, nb - j0, Vb, L.ldv, Ts, bw, wsz, true, Wb, Wb + L.ldw * L.wcols);
        store_rows(Cb, L.ldc, 0, X, nb, j0, nb, cs, wsz);
      } else {
        const int r2 = MODE == 1 ? j0 + bw : nb;
        async_block(Cb, L.ldc, A1, nb, j0, j0 + bw, cs, wsz);         // C1 rows of the block -> window 0
        load_rows(Cb, L.ldc, kWinRows, X, nb, 0, r2, cs, wsz);
        cp_async_wait_all();
        __syncthreads();
        prof_mark(PH_LOAD);
        apply_block(Cb, Cb + kWinRows, L.ldc, r2, Vb, L.ldv, Ts, bw, wsz, true, Wb, Wb + L.ldw * L.wcols);
        store_rows(Cb - j0, L.ldc, 0, A1, nb, j0, j0 + bw, cs, wsz);
        store_rows(Cb, L.ldc, kWinRows, X, nb, 0, r2, cs, wsz);
      }
    }
    __syncthreads();
  }
}

// ---- update kernels on one column strip -----------------------------------
// Inner blocks are pipelined: while block b is applied, the V / T (and C1
// rows) of the next block stream into the other buffer (when smem allows).

// UNMQR: C (tile strip) <- Q^T C (or Q C) with inner blocks [b_lo, b_hi) of the
// GEQRT reflectors of tile Vt; only rows >= b_lo*ib are touched.
__device__ void unmqr_strip(const double *Vt, const double *Tslot, double *Ct, int nb, int ib, int cs,
                            int wsz, bool trans, int b_lo, int b_hi, double *smem, const SmemLayout &L,
                            unsigned &mbph, bool tma, bool resident = false) {
  double *Cb = smem + L.offC, *Wb = smem + L.offW;
  const int r0 = b_lo * ib;
  const int nblk = b_hi - b_lo;
  auto blk = [&](int idx) { return trans ? b_lo + idx : b_hi - 1 - idx; };
  tma_block(Cb + r0, L.ldc, Ct, nb, r0, nb, cs, wsz, tma);
  if (!resident) {     // resident: the panel task just left V (unit diagonal, padded) and T in buffer 0
    const int j0 = blk(0) * ib, bw = min(ib, nb - j0);
    tma_block(smem + L.offV[0], L.ldv, Vt, nb, j0, nb, j0, bw, tma);
    issue_t(smem + L.offT[0], Tslot, ib, j0, bw);
  }
  for (int idx = 0; idx < nblk; ++idx) {
    const int cur = idx & (L.nvb - 1);
    double *Vb = smem + (cur ? L.offV[1] : L.offV[0]), *Ts = smem + (cur ? L.offT[1] : L.offT[0]);
    const int j0 = blk(idx) * ib, bw = min(ib, nb - j0);
    async_wait(mbph);
    __syncthreads();
    prof_mark(PH_LOAD);
    if (!(resident && idx == 0)) {
      fix_v_geqrt(Vb, L.ldv, nb, j0, bw);
      __syncthreads();
    }
    prof_mark(PH_FIX);
    if (L.nvb == 2 && idx + 1 < nblk) {
      const int j1 = blk(idx + 1) * ib, bw1 = min(ib, nb - j1);
      tma_block(smem + (cur ? L.offV[0] : L.offV[1]), L.ldv, Vt, nb, j1, nb, j1, bw1, tma);
      issue_t(smem + (cur ? L.offT[0] : L.offT[1]), Tslot, ib, j1, bw1);
    }
    apply_block(nullptr, Cb + j0, L.ldc, nb - j0, Vb, L.ldv, Ts, bw, wsz, trans, Wb, Wb + L.ldw * L.wcols);
    if (L.nvb == 1 && idx + 1 < nblk) {
      const int j1 = blk(idx + 1) * ib, bw1 = min(ib, nb - j1);
      tma_block(Vb, L.ldv, Vt, nb, j1, nb, j1, bw1, tma);
      issue_t(Ts, Tslot, ib, j1, bw1);
    }
  }
  store_rows(Cb, L.ldc, 0, Ct, nb, r0, nb, cs, wsz);
}

// TTMQR / TSMQR: [C1; C2] <- Q^T [C1; C2] (or Q) with inner blocks [b_lo, b_hi)
// of the TTQRT/TSQRT reflectors V2 of tile Vt. Block b touches C1 rows
// b*ib .. b*ib+bw-1 (streamed through a 32-row window) and C2 rows
// 0 .. (tri ? b*ib+bw : nb)-1 (resident).
__device__ void tpmqr_strip(const double *Vt, const double *Tslot, double *C1, double *C2, int nb, int ib,
                            int cs, int wsz, bool tri, bool trans, int b_lo, int b_hi, double *smem,
                            const SmemLayout &L, unsigned &mbph, bool tma, bool resident = false) {
  double *Cb = smem + L.offC, *Wb = smem + L.offW;
  const int r2hi = tri ? min(b_hi * ib, nb) : nb;
  const int nblk = b_hi - b_lo;
  auto blk = [&](int idx) { return trans ? b_lo + idx : b_hi - 1 - idx; };
  tma_block(Cb + kWinRows, L.ldc, C2, nb, 0, r2hi, cs, wsz, tma);
  {
    const int j0 = blk(0) * ib, bw = min(ib, nb - j0);
    if (!resident) {
      tma_block(smem + L.offV[0], L.ldv, Vt, nb, 0, tri ? j0 + bw : nb, j0, bw, tma);
      issue_t(smem + L.offT[0], Tslot, ib, j0, bw);
    }
    tma_block(Cb, L.ldc, C1, nb, j0, j0 + bw, cs, wsz, tma);
  }
  for (int idx = 0; idx < nblk; ++idx) {
    const int cur = idx & (L.nvb - 1);
    double *Vb = smem + (cur ? L.offV[1] : L.offV[0]), *Ts = smem + (cur ? L.offT[1] : L.offT[0]), *win = Cb + 32 * (idx & 1);
    const int j0 = blk(idx) * ib, bw = min(ib, nb - j0);
    async_wait(mbph);
    __syncthreads();
    prof_mark(PH_LOAD);
    if (!(resident && idx == 0)) {
      fix_v_tp(Vb, L.ldv, nb, j0, bw, tri);
      __syncthreads();
    }
    prof_mark(PH_FIX);
    if (L.nvb == 2 && idx + 1 < nblk) {
      const int j1 = blk(idx + 1) * ib, bw1 = min(ib, nb - j1);
      tma_block(smem + (cur ? L.offV[0] : L.offV[1]), L.ldv, Vt, nb, 0, tri ? j1 + bw1 : nb, j1, bw1, tma);
      issue_t(smem + (cur ? L.offT[0] : L.offT[1]), Tslot, ib, j1, bw1);
      tma_block(Cb + 32 * ((idx + 1) & 1), L.ldc, C1, nb, j1, j1 + bw1, cs, wsz, tma);
    }
    apply_block(win, Cb + kWinRows, L.ldc, tri ? j0 + bw : nb, Vb, L.ldv, Ts, bw, wsz, trans, Wb,
                Wb + L.ldw * L.wcols);
    store_rows(win - j0, L.ldc, 0, C1, nb, j0, j0 + bw, cs, wsz);
    if (L.nvb == 1 && idx + 1 < nblk) {
      __syncthreads();
      const int j1 = blk(idx + 1) * ib, bw1 = min(ib, nb - j1);
      tma_block(Vb, L.ldv, Vt, nb, 0, tri ? j1 + bw1 : nb, j1, bw1, tma);
      issue_t(Ts, Tslot, ib, j1, bw1);
      tma_block(Cb + 32 * ((idx + 1) & 1), L.ldc, C1, nb, j1, j1 + bw1, cs, wsz, tma);
    }
  }
  store_rows(Cb, L.ldc, kWinRows, C2, nb, 0, r2hi, cs, wsz);
}

__device__ void run_task(const RunArgs &a, const DevTask &t, double *smem, const SmemLayout &L, bool resident,
                         unsigned &mbph) {
  const bool tma = a.tma != 0;
  const int p = a.p, nb = a.nb, ib = a.ib, ws = a.ws;
  const int nblk = (nb + ib - 1) / ib;
  double *Vb = smem + L.offV[0], *Wb = smem + L.offW, *Ts = smem + L.offT[0];
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
    // ---- split panels: inner block s of the panel, or update of strip s by block j
    case K_GEQRT_B: {
      const int j0 = t.s * ib;
      panel_block<0>(tile_ptr(a.A, p, nb, t.i, t.k), nullptr, tslot_ptr(a.T, p, nb, ib, t.i, t.k, 0), nb, ib, j0,
                     min(ib, nb - j0), Vb, L.ldv, Ts, Wb);
      break;
    }
    case K_TTQRT_B:
    case K_TSQRT_B: {
      const int j0 = t.s * ib;
      double *X = tile_ptr(a.A, p, nb, t.i, t.k), *A1 = tile_ptr(a.A, p, nb, t.piv, t.k);
      double *Tsl = tslot_ptr(a.T, p, nb, ib, t.i, t.k, 1);
      if (t.kind == K_TTQRT_B) panel_block<1>(X, A1, Tsl, nb, ib, j0, min(ib, nb - j0), Vb, L.ldv, Ts, Wb);
      else panel_block<2>(X, A1, Tsl, nb, ib, j0, min(ib, nb - j0), Vb, L.ldv, Ts, Wb);
      break;
    }
    case K_GEQRT_U: {
      const int cs = t.s * ws, wsz = min(ws, nb - cs);
      double *X = tile_ptr(a.A, p, nb, t.i, t.k);
      unmqr_strip(X, tslot_ptr(a.T, p, nb, ib, t.i, t.k, 0), X, nb, ib, cs, wsz, true, t.j, t.j + 1, smem, L,
                  mbph, tma, resident);
      break;
    }
    case K_TTQRT_U:
    case K_TSQRT_U: {
      const int cs = t.s * ws, wsz = min(ws, nb - cs);
      double *X = tile_ptr(a.A, p, nb, t.i, t.k);
      tpmqr_strip(X, tslot_ptr(a.T, p, nb, ib, t.i, t.k, 1), tile_ptr(a.A, p, nb, t.piv, t.k), X, nb, ib, cs, wsz,
                  t.kind == K_TTQRT_U, true, t.j, t.j + 1, smem, L, mbph, tma, resident);
      break;
    }
    // ---- updates of other tiles (factorization) and of C (apply)
    case K_UNMQR:
    case K_AP_UNMQR: {
      double *Cbase = t.kind == K_UNMQR ? a.A : a.C;
      const int cs = t.s * ws, wsz = min(ws, nb - cs);
      unmqr_strip(tile_ptr(a.A, p, nb, t.i, t.k), tslot_ptr(a.T, p, nb, ib, t.i, t.k, 0),
                  tile_ptr(Cbase, p, nb, t.i, t.j), nb, ib, cs, wsz, a.trans != 0, 0, nblk, smem, L, mbph, tma);
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
                  a.trans != 0, 0, nblk, smem, L, mbph, tma);
      break;
    }
    default:
      break;
  }
}

// ---- the persistent dataflow kernel ----------------------------------------
// Dataflow with per-task dependency counters (north_star: "a persistent kernel
// gated by per-tile dependency counters"). A finished task bumps the counter
// of each successor (atom.acq_rel); the predecessor that completes a
// successor's count pushes it on the ready queue of its priority level (or
// runs it next itself: chain continuation / work-first).
// CTAs only ever take ready tasks, so no CTA idles on a specific task while
// others are runnable. Queue slots carry the launch epoch, counters
// accumulate epoch x indegree, and the last CTA to leave resets the queue
// heads/tails: nothing is cleared between launches (one launch per call).
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned *p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ int ld_relaxed(const int *p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__shared__ unsigned s_epoch;   // launch epoch, read from ctrl[kCtrlEpoch] at kernel start

__device__ __forceinline__ void push_ready(const RunArgs &a, int t) {   // (chained tasks may be queued too)
  const int q = (a.tasks[t].meta >> 16) & 15;
  const int pos = atomicAdd(&a.ctrl[kCtrlTail + 64 * q], 1);
  st_release64(a.queue + a.qoff[q] + pos, ((unsigned long long)s_epoch << 32) | (unsigned)t);
  atomicAdd(&a.ctrl[kCtrlLevel + 32 * q], 1);
  if (a.trace) a.trace[kTraceWords * (size_t)t + 12] = globaltimer();   // diagnostics: push time
}

// Claim a task of queue q, or return -1. A fetch-and-subtract on the level's
// count reserves one published task (undone if the count was not positive),
// then a fetch-and-add on the head takes the next slot; neither retries, so
// tens of idle CTAs claiming from one level do not serialise on a CAS loop.
// The slot's pusher has already taken its tail position, so at worst the pop
// waits for that store to land.
__device__ __forceinline__ int try_pop(const RunArgs &a, int q) {
  int *cnt = &a.ctrl[kCtrlLevel + 32 * q];
  if (atomicSub(cnt, 1) <= 0) { atomicAdd(cnt, 1); return -1; }
  const int h = atomicAdd(&a.ctrl[kCtrlHead + 64 * q], 1);
  const unsigned long long *slot = a.queue + a.qoff[q] + h;
  unsigned long long v;
  while (((v = ld_acquire64(slot)) >> 32) != s_epoch) __nanosleep(20);
  return (int)(v & 0xffffffffu);
}

__device__ __forceinline__ unsigned ld_acquire_u(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned need_count(const RunArgs &a, int t) {
  const int m = a.tasks[t].meta;
  return s_epoch * (unsigned)((m & 0xffff) + ((m >> 20) & 1));
}
__device__ __forceinline__ bool is_panel_block(int kind) {
  return kind == K_GEQRT_B || kind == K_TTQRT_B || kind == K_TSQRT_B;
}

__global__ void __launch_bounds__(kThreads, 1) tqr_persistent(RunArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_task, s_chain, s_resident;
  const SmemLayout L = smem_layout(a.nb, a.ib, a.ws);
  if (threadIdx.x == 0) {
    s_prof_on = 0; s_chain = -1; s_resident = 0; mbar_init();
    s_epoch = (unsigned)ld_acquire(&a.ctrl[kCtrlEpoch]);
  }
  unsigned mbph = 0u;   // parity of the CTA mbarrier (identical in every thread)
  // everything the DMMA padding may read must be finite: start from zeros
  for (size_t x = threadIdx.x; x < L.total; x += kThreads) smem[x] = 0.0;
  __syncthreads();
  // the first CTA to arrive seeds every root: progress never depends on a
  // particular CTA being resident (grids larger than the co-resident
  // capacity, or SMs held by a concurrent kernel, still complete)
  if (threadIdx.x == 0 && atomicAdd(&a.ctrl[kCtrlStart], 1) == 0)
    for (int r = 0; r < a.nroots; ++r) push_ready(a, a.roots[r]);
  for (;;) {
    if (threadIdx.x < 32) {
      // warp 0 claims the next task: lane l < kLevels reads level l's count,
      // a ballot names the non-empty levels, lane 0 claims from the highest
      const int lane = threadIdx.x;
      __syncwarp();   // s_chain was written by lane 0 at the end of the last task
      unsigned long long t_take = (a.trace && lane == 0) ? globaltimer() : 0ull;
      int t = s_chain;
      if (t < 0) {
        if (lane == 0) s_resident = 0;
        unsigned backoff = 32;
        for (;;) {
          const int c = lane < kLevels ? ld_relaxed(&a.ctrl[kCtrlLevel + 32 * lane]) : 0;
          unsigned live = __ballot_sync(0xffffffffu, c > 0);
          while (live && t < 0) {
            const int q = 31 - __clz(live);
            int got = -1;
            if (lane == 0) got = try_pop(a, q);
            t = __shfl_sync(0xffffffffu, got, 0);
            live &= ~(1u << q);
          }
          if (t >= 0) break;
          int fin = 0;
          if (lane == 0) fin = ld_relaxed(&a.ctrl[kCtrlDone]) >= a.ntask;
          if (__shfl_sync(0xffffffffu, fin, 0)) { t = -1; break; }
          __nanosleep(backoff);
          backoff = backoff < 1024 ? backoff * 2 : 1024;
        }
      }
      if (lane == 0) s_task = t;
      if (lane == 0 && a.trace && t >= 0) {
        a.trace[kTraceWords * (size_t)t] = t_take;
        a.trace[kTraceWords * (size_t)t + 1] = globaltimer();
        for (int x = 0; x < 8; ++x) s_prof[x] = 0;
        s_prof_last = clock64();
        s_prof_on = 1;
      }
    }
    __syncthreads();
    const int t = s_task;
    if (t < 0) break;
    __threadfence();
    const DevTask tk = a.tasks[t];
    // warp 0 issues the loads of its first successor edges now; they land
    // while the task runs and are consumed only when releasing
    int2 e0 = make_int2(-1, 0);
    if (threadIdx.x < 32 && tk.dep_begin + (int)threadIdx.x < tk.dep_end) e0 = __ldg(a.succ + tk.dep_begin + threadIdx.x);
    run_task(a, tk, smem, L, s_resident != 0, mbph);
    __syncthreads();
    prof_mark(PH_STORE);
    int keep = -1;   // (lane 0) successor this CTA runs next without queueing it
    if (threadIdx.x < 32) {
      // release the successors, one per lane (a panel block can have tens):
      // every lane fences the CTA's writes (ordered by the barrier above) to
      // gpu scope before its arrival, so the atomics run in parallel instead
      // of as a dependent chain of round trips on one thread
      const int lane = threadIdx.x;
      __threadfence();
      // work-first: without a chain continuation, the CTA keeps the most
      // urgent successor it made ready if no queued task is more urgent
      // (the queue probe is issued alongside the arrivals)
      const bool may_keep = tk.chain < 0 && a.work_first;
      const int qc = (may_keep && lane < kLevels) ? ld_relaxed(&a.ctrl[kCtrlLevel + 32 * lane]) : 0;
      int mine = -1, mine_lvl = -1;
      for (int x = tk.dep_begin + lane; x < tk.dep_end; x += 32) {
        const int2 e = x == tk.dep_begin + lane ? e0 : a.succ[x];
        const int sc = e.x, m = e.y;
        const unsigned need = s_epoch * (unsigned)((m & 0xffff) + ((m >> 20) & 1));
        if (atom_add_acqrel(a.cnt + sc, 1u) + 1u == need) {
          const int lvl = (m >> 16) & 15;
          if (may_keep && lvl > mine_lvl) {
            if (mine >= 0) push_ready(a, mine);
            mine = sc; mine_lvl = lvl;
          } else {
            push_ready(a, sc);
          }
        }
      }
      if (may_keep) {
        const unsigned live = __ballot_sync(0xffffffffu, qc > 0);
        const int qmax = live ? 31 - __clz(live) : -1;
        int best = mine >= 0 ? mine_lvl * 32 + lane : -1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
        const bool win = best >= 0 && (best & 31) == lane && mine_lvl >= qmax;
        if (mine >= 0 && !win) push_ready(a, mine);
        const unsigned wl = __ballot_sync(0xffffffffu, win);
        keep = __shfl_sync(0xffffffffu, mine, wl ? __ffs(wl) - 1 : 0);
        if (!wl) keep = -1;
      }
      __syncwarp();
    }
    if (threadIdx.x == 0) {
      if (a.trace) {
        unsigned long long *tr = a.trace + kTraceWords * (size_t)t;
        tr[2] = globaltimer();
        tr[3] = ((unsigned long long)smid() << 32) | (unsigned)tk.kind;
        for (int x = 0; x < 8; ++x) tr[4 + x] = s_prof[x];   // word 12 = push time
      }
      atomicAdd(&a.ctrl[kCtrlDone], 1);
      // panel chain: run the chained successor here if its other inputs are (or
      // soon become) ready; otherwise release the virtual dependency so the last
      // real predecessor queues it normally. Either way it runs exactly once.
      int nxt = -1;
      if (tk.chain >= 0) {
        const int c = tk.chain;
        const unsigned need = need_count(a, c);
        for (int it = 0; it < a.chain_spin && ld_acquire_u(a.cnt + c) + 1u < need; ++it) __nanosleep(128);
        if (atom_add_acqrel(a.cnt + c, 1u) + 1u == need) nxt = c;
      }
      s_resident = (nxt >= 0 && is_panel_block(tk.kind)) ? 1 : 0;
      s_chain = nxt >= 0 ? nxt : keep;
    }
  }
  if (threadIdx.x == 0) {
    const int n = atomicAdd(&a.ctrl[kCtrlExit], 1);
    if (n == a.nctas - 1) {
      for (int q = 0; q < kLevels; ++q)
        a.ctrl[kCtrlHead + 64 * q] = a.ctrl[kCtrlTail + 64 * q] = a.ctrl[kCtrlLevel + 32 * q] = 0;
      a.ctrl[kCtrlDone] = 0; a.ctrl[kCtrlExit] = 0; a.ctrl[kCtrlStart] = 0;
      __threadfence();
      a.ctrl[kCtrlEpoch] = (int)(s_epoch + 1u);   // the next launch (stream-ordered) runs epoch + 1
      __threadfence();
    }
  }
}

#endif  // __CUDACC__

}  // namespace tqr
