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
#include <cuda.h>
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
constexpr int kLdwP = 34;                   // partial W^T: accumulator-pattern stores and loads only (col + 2t*kLdwP conflict-free)
constexpr int kLdw = 36;                    // W^T / W2^T in smem: element (col, refl) at col + refl * kLdw
constexpr int kSlots = 8;                   // row tiles of 8 per warp in a strip update (nb <= 256)
#ifndef TQR_BOX
#define TQR_BOX 4
#endif
constexpr int kBoxTiles = TQR_BOX;          // row tiles per TMA box of a V block
#ifndef TQR_EXP
#define TQR_EXP 0                           // (timing experiments of tools/strip_bench only; 0 in the product:
                                            //  32/64 repeat phase 1/3, 128/256 drop phase 1/3's V loads)
#endif
constexpr int kTraceWords = 13;             // per-task trace record (diagnostics): 4 stamps/ids, 8 phases, push time
// scheduler control words (ints; each on its own 128-byte line): per priority
// level l a queue head at kCtrlHead + 64 l, its tail at kCtrlTail + 64 l and
// its count of published, unclaimed tasks at kCtrlLevel + 32 l
// kCtrlEpoch holds the launch epoch (1 after upload; the last CTA of a launch
// advances it), kCtrlStart the arrival ticket whose first holder seeds the roots.
constexpr int kCtrlHead = 0, kCtrlTail = 32, kCtrlDone = 64 * kLevels, kCtrlExit = 64 * kLevels + 32,
              kCtrlLevel = 64 * kLevels + 96, kCtrlEpoch = 96 * kLevels + 96, kCtrlStart = 96 * kLevels + 128,
              kCtrlWords = 96 * kLevels + 160;
// panel scratch: t_doubling temp, G = V^T V, working T (all 32 x kTld), the
// published reflector (2 x 256), its tau (2 x 4) and the block's taus (32)
constexpr int kPanelScratch = 3 * 32 * kTld + 2 * 256 + 8 + 32;

struct alignas(64) RunArgs {
  CUtensorMap mapA;             // A as (row in tile-of-8, global column, row tile): box 8 x 32 x 4 (TMA path)
  CUtensorMap mapC;             // the same view of C (apply_qt / apply_q)
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
  int tma;                     // 1: V blocks and C1 windows move by TMA tensor copies (nb, ib % 8 == 0)
  int work_first;              // 1: a CTA runs the most urgent successor it made ready (not queued)
  int chain_spin;              // polls (128 ns apart) for a chained successor's other inputs
  unsigned long long *trace;   // optional: kTraceWords u64 per task (taken, ready, done, smid<<32|kind, 8 phase cycle counters)
};

// ---- shared-memory layout ----------------------------------------------------
// Row-tile ("tile-of-8") layout of a column block: rows are grouped in tiles
// of 8; tile j holds rows 8j..8j+7 of up to 32 columns as [column][row % 8],
// 256 doubles per tile. Element (r, l) sits at (r >> 3) * 256 + l * 8 + (r & 7).
// Every fragment access of the strip update is bank-conflict-free in it: the
// 16-byte row pairs (2t, 2t+1) of lanes (g, t) land on 8 distinct 16-byte
// units per quarter warp, and the 8-byte reads (row g, column 4k + t) on 16
// distinct bank pairs per half warp.
__host__ __device__ inline int vidx(int r, int l) { return (r >> 3) * 256 + l * 8 + (r & 7); }
__host__ __device__ inline int round_up(int n, int m) { return (n + m - 1) / m * m; }

struct SmemLayout {
  int ntile;                    // ceil(nb / 8) row tiles
  size_t offV[2];               // reflector blocks V (double-buffered), ntile x 256 each, absolute rows
  size_t offWp;                 // 4 partial W^T (32 x kLdw each); the panel's scratch aliases it
  size_t offW, offW2;           // reduced W^T and W2^T (32 x kLdw each)
  size_t offT[2];               // T blocks, ld ib (double-buffered)
  size_t offC1[2];              // C1 windows of TT/TS updates: ib rows x 32 columns, row-tile layout
  size_t total;                 // in doubles
};

__host__ __device__ inline SmemLayout smem_layout(int nb, int ib, int ws) {
  (void)ib; (void)ws;
  SmemLayout s;
  s.ntile = (nb + 7) / 8;
  const size_t v = (size_t)s.ntile * 256;
  s.offV[0] = 0;
  s.offV[1] = v;
  s.offWp = 2 * v;
  const size_t wp = 4 * 32 * kLdw > kPanelScratch ? 4 * 32 * kLdw : kPanelScratch;
  s.offW = s.offWp + wp;
  s.offW2 = s.offW + 32 * kLdw;
  s.offT[0] = s.offW2 + 32 * kLdw;
  s.offT[1] = s.offT[0] + 1024;
  s.offC1[0] = s.offT[1] + 1024;
  s.offC1[1] = s.offC1[0] + 1024;
  s.total = s.offC1[1] + 1024;
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
#ifndef TQR_PROF
#define TQR_PROF 0                          // 1: in-task phase counters for the tracer (costs ~4% in the hot loops)
#endif
__device__ __forceinline__ void prof_mark(int slot) {
  if (TQR_PROF && threadIdx.x == 0 && s_prof_on) {
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
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// ---- asynchronous global -> shared copies ------------------------------------
// cp.async (LDGSTS) with zero fill: `valid` = false writes zeros without a
// global read. Completion is tracked per buffer by an mbarrier: the one warp
// that issues a buffer's copies ends with cp.async.mbarrier.arrive.noinc on
// every lane (the barrier expects those 32 arrivals, plus the TMA transaction
// bytes), so consumers wait on the mbarrier instead of a CTA-wide barrier. Writers of a tile are ordered before readers by the release/acquire
// task counters plus a gpu-scope fence.
__device__ __forceinline__ void cp_async16_zf(double *dst, const double *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async8_zf(double *dst, const double *src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__shared__ __align__(8) unsigned long long s_mbar[2];   // one per V/T/C1 buffer ("full": 32 arrivals of the issuing warp)
__shared__ int s_done[2];      // warps done with a buffer's block (the 8th refills it)

__device__ __forceinline__ void mbar_init_all() {
  for (int b = 0; b < 2; ++b)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&s_mbar[b])), "r"(32) : "memory");
  s_done[0] = s_done[1] = 0;
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// this thread's arrival on buffer b's barrier once its outstanding cp.async copies have landed
__device__ __forceinline__ void mbar_arrive_cp(int b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&s_mbar[b])) : "memory");
}
// wait for the current phase of buffer b's barrier; `ph` holds one parity bit per buffer
__device__ __forceinline__ void mbar_wait(int b, unsigned &ph) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "TQR_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TQR_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(&s_mbar[b])), "r"((ph >> b) & 1u) : "memory");
  ph ^= 1u << b;
}

// rows [row0, row0 + 8 ntl) of columns [c0, c0 + ncol) (ncol <= 32) of the
// column-major tile X (ld nb) -> row-tile layout dst (tile 0 = rows row0..row0+7);
// rows outside [0, nb) are zero-filled; columns >= ncol are left untouched.
// Issued by one warp: per (row tile, 8 columns) chunk, lane -> column lane/4, row pair lane%4.
__device__ __forceinline__ void load_tiles8(double *dst, const double *X, int nb, int row0, int ntl, int c0,
                                            int ncol) {
  const int lane = threadIdx.x & 31;
  const int cl = lane >> 2, pr = 2 * (lane & 3);
  const bool v16 = ((nb | row0) & 1) == 0;
  for (int ch = 0; ch < ntl * 4; ++ch) {
    const int tl = ch >> 2, c = 8 * (ch & 3) + cl;
    if (c < ncol) {
      const int r = row0 + 8 * tl + pr;
      double *d = dst + tl * 256 + c * 8 + pr;
      const double *s = X + (size_t)(c0 + c) * nb;
      if (v16) {
        cp_async16_zf(d, s + (r < nb ? r : 0), r < nb);
      } else {
        cp_async8_zf(d, s + (r < nb ? r : 0), r < nb);
        cp_async8_zf(d + 1, s + (r + 1 < nb ? r + 1 : 0), r + 1 < nb);
      }
    }
  }
}
// T block of inner block j0 (bw columns of a T slot, ld ib) -> dst (same layout); one warp
__device__ __forceinline__ void load_tblock(double *dst, const double *Tslot, int ib, int j0, int bw) {
  const int n = bw * ib, lane = threadIdx.x & 31;
  const double *s = Tslot + (size_t)j0 * ib;
  if ((ib & 1) == 0) {
    for (int i = 2 * lane; i < n; i += 64) cp_async16_zf(dst + i, s + i, true);
  } else {
    for (int i = lane; i < n; i += 32) cp_async8_zf(dst + i, s + i, true);
  }
}

// ---- TMA: 3-D tensor copies in the row-tile layout ---------------------------
// The host encodes A (and C) as a 3-D tensor (row within a tile of 8, global
// column (k p + i) nb + c, row tile) with strides (8 B, nb * 8 B, 64 B); a box
// of 8 x 32 x 4 lands in shared memory as 4 row tiles of 32 columns, i.e.
// exactly the row-tile layout. Rows past nb (row tiles >= nb/8) are
// out-of-bounds and filled with zeros by the copy engine.
__device__ __forceinline__ void tma_box(double *dst, const CUtensorMap *map, int col, int tile, int b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(0), "r"(col), "r"(tile), "r"(smem_u32(&s_mbar[b]))
      : "memory");
}
__device__ __forceinline__ void tma_bulk(double *dst, const double *src, unsigned bytes, int b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(&s_mbar[b]))
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(int b, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&s_mbar[b])), "r"(bytes)
               : "memory");
}
// ---- FP64 tensor-core MMA (DMMA): D(16x8) += A(16x4) B(4x8) ------------------
// Fragments (lane = 4*g + t): a0 = A[g][t], a1 = A[g+8][t]; b0 = B[t][g];
// d0,d1 = D[g][2t, 2t+1], d2,d3 = D[g+8][2t, 2t+1].
__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(b0));
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

// G (32 x 32, ld kTld) = V^T V over row tiles [tlo, thi) of a row-tile-layout V
// block (rows outside the reflectors are zero), on the tensor pipe: the two
// k-steps of a tile take rows (2t) and (2t+1), one 16-byte load per operand.
__device__ void gram_v8(double *G, const double *V, int tlo, int thi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (warp & 1) * 16, n0 = (warp >> 1) * 8;   // 8 warps = 2 x 4 fragments
  double acc0[4] = {0.0, 0.0, 0.0, 0.0}, acc1[4] = {0.0, 0.0, 0.0, 0.0};
  for (int j = tlo; j < thi; ++j) {
    const double *vt = V + j * 256 + 2 * t;
    const double2 a = *reinterpret_cast<const double2 *>(vt + (m0 + g) * 8);
    const double2 a8 = *reinterpret_cast<const double2 *>(vt + (m0 + g + 8) * 8);
    const double2 b = *reinterpret_cast<const double2 *>(vt + (n0 + g) * 8);
    dmma(acc0, a.x, a8.x, b.x);
    dmma(acc1, a.y, a8.y, b.y);
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
// doubling. Writes R/V back (only the parts this kernel owns), the T slot, and
// leaves the block's V (row-tile layout, absolute rows, zero outside the
// reflectors) in Vbuf and its T (ld ib) in Tb for a trailing update on this CTA.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

#ifndef TQR_PABL
#define TQR_PABL 0   // tools/panel_bench.cu only: timing attribution of the column chain (results are wrong)
#endif
template <int MODE>
__device__ void panel_block(double *X, double *A1, double *Tslot, int nb, int ib, int j0, int bw,
                            double *Vbuf, double *Tb, double *scratch) {
  double *top = scratch;               // 32 x kTld scratch for t_doubling
  double *G = top + 32 * kTld;         // 32 x kTld: V^T V
  double *Ts = G + 32 * kTld;          // 32 x kTld: working T
  double *vsh = Ts + 32 * kTld;        // 2 x 256: published reflector (double-buffered)
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
        const double xn2 = (TQR_PABL & 2) ? ss : warp_sum(ss);
        const double alpha = __shfl_sync(0xffffffffu, MODE == 0 ? a[qo][0] : pt[qo], c);
        double beta, tau, scale;
        if (TQR_PABL & 1) { beta = alpha; tau = 0.5; scale = 1e-3 * xn2; }
        else larfg_scalars(alpha, xn2, beta, tau, scale);
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
      if (!(TQR_PABL & 8)) __syncthreads();
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
          P[q] = (TQR_PABL & 16) ? a[q][1]
                 : MODE == 0 ? __shfl_sync(0xffffffffu, a[q][0], c) : __shfl_sync(0xffffffffu, pt[q], c);
        }
#pragma unroll
        for (int o = (TQR_PABL & 4) ? 0 : 16; o > 0; o >>= 1)
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
  // Vbuf covers the whole row tiles [vlo, vhi) of the block's V rows, zero
  // outside the reflectors (the gram product and the trailing update read
  // whole tiles).
  const int vlo = MODE == 0 ? (j0 & ~7) : 0, vhi = round_up(rbase + nr, 8);
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
            Vbuf[vidx(row, cl)] = rr == cl ? 1.0 : (rr > cl ? a[q][s2] : 0.0);
          } else {
            const bool part = MODE == 2 || row <= j0 + cl;
            if (part) X[row + (size_t)(j0 + cl) * nb] = a[q][s2];
            Vbuf[vidx(row, cl)] = part ? a[q][s2] : 0.0;
          }
        } else if (row < vhi) {
          Vbuf[vidx(row, cl)] = 0.0;
        }
      }
      if (MODE == 0 && lane < j0 - vlo) Vbuf[vidx(vlo + lane, cl)] = 0.0;
    }
  }
  if (MODE != 0) {     // final pivot rows (R) back to A1, upper triangle of the block
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cl = warp + 8 * q;
      if (cl < bw && lane <= cl) A1[(j0 + lane) + (size_t)(j0 + cl) * nb] = pt[q];
    }
  }
  for (int idx = tid; idx < 32 * 32; idx += kThreads) {     // Ts = diag(tau) (zero-padded)
    const int l = idx & 31, c = idx >> 5;
    Ts[l + c * kTld] = (l == c && c < bw) ? taus[c] : 0.0;
  }
  __syncthreads();
  prof_mark(PH_PANEL);
  gram_v8(G, Vbuf, vlo >> 3, vhi >> 3);
  __syncthreads();
  t_doubling(Ts, G, top);
  prof_mark(PH_TREC);
  for (int c = warp; c < bw; c += kWarps)
    if (lane < ib) {
      const double v = (lane < bw && lane <= c) ? Ts[lane + c * kTld] : 0.0;
      Tslot[lane + (size_t)(j0 + c) * ib] = v;
      Tb[lane + c * ib] = v;
    }
}

// ---- trailing updates on one column strip (UNMQR / TTMQR / TSMQR) -----------
// C <- Q_b^T C (or Q_b C) for the inner blocks b of a panel kernel's
// reflectors, in compact-WY form (lines 62-66): W = V^T C, W2 = -op(T) W,
// C += V W2; for TT/TS (V = [I; V2], Table 1) W = C1_b + V2^T C2,
// C1_b += W2, C2 += V2 W2.
//
// Register-resident design: the strip's C (C2 for TT/TS) lives in registers
// as fragments of C^T for the whole task; only V, T and the 32-row C1 window
// of each inner block move through shared memory (double-buffered, the next
// block's copies in flight during this block's math). Warp w = (row group
// rg = w/2, column half mh = w%2) owns columns 16 mh .. 16 mh + 15 of the row
// tiles j = rg + 4 s (s < kSlots). Per block:
//   phase 1  partial W^T over the warp's row tiles: the C^T accumulators ARE
//            the A fragments (k-steps = rows 2t and 2t+1 of a tile), V the B
//            fragments (one 16-byte load per 2 DMMAs); 4 partials -> smem
//   reduce   W^T = sum of the partials (+ C1 window for TT/TS)
//   phase 2  W2^T = -W^T op(T)^T, one 16x8 fragment per warp, + C1_b update
//   phase 3  C^T += W2^T V^T (V^T from smem, W2^T fragments held in registers)
// All contractions run on the FP64 tensor pipe (mma.sync m16n8k4 f64 = DMMA).
// The reflectors' structure (unit diagonal / zeros above it for GEQRT, the
// upper trapezoid of TTQRT) is applied as a mask on the loaded fragments of
// the <= 5 row tiles that cross the block's diagonal, so V is copied raw.
enum { SU_UN = 0, SU_TT = 1, SU_TS = 2 };

struct StripJob {
  const double *Vt;     // tile holding the reflectors (GEQRT: V below the diagonal; TT/TS: V2)
  const double *Tslot;  // its T slot (ib x nb, ld ib)
  double *C1;           // TT/TS: the pivot-row tile (rows b*ib .. b*ib + bw - 1 per block)
  double *C2;           // the updated tile
  int nb, ib, cs, wsz;  // strip = columns [cs, cs + wsz) of C1 / C2
  int b_lo, b_hi;       // inner blocks applied (ascending for Q^T, descending for Q)
  bool trans, resident; // resident: block b_lo's V and T are already in buffer 0 (panel chain)
  const CUtensorMap *mV, *mC1;  // TMA path: tensor maps (boxes of kBoxTiles / 4 row tiles) of the V tile's and the
                                // C1 tile's matrix (null: cp.async)
  int vcol, c1col;              // global column of the V tile's and the C1 tile's first column
};

// row tiles a block touches: UN rows j0..nb-1, TT rows 0..j0+bw-1, TS rows 0..nb-1
template <int KIND>
__device__ __forceinline__ void su_range(int j0, int bw, int ntile, int &lo, int &hi) {
  lo = KIND == SU_UN ? (j0 >> 3) : 0;
  hi = KIND == SU_TT ? ((j0 + bw + 7) >> 3) : ntile;
}
// V element (row r, reflector l) of block j0 from its raw tile value
template <int KIND>
__device__ __forceinline__ double vmask(double v, int r, int l, int j0) {
  if (KIND == SU_UN) {
    const int rr = r - j0;
    return rr > l ? v : (rr == l ? 1.0 : 0.0);
  }
  return r <= j0 + l ? v : 0.0;
}

// copies of block b into buffer `buf`, issued by ONE warp (32 mbarrier
// arrivals); vt = false: V and T are already there (panel chain), only the C1
// window moves
template <int KIND>
__device__ __forceinline__ void su_issue(const StripJob &J, const SmemLayout &L, double *smem, int buf, int b,
                                         bool vt = true) {
  const int lane = threadIdx.x & 31;
  const int j0 = b * J.ib, bw = min(J.ib, J.nb - j0);
  int lo, hi;
  su_range<KIND>(j0, bw, L.ntile, lo, hi);
  if (J.mV) {
    // one copy per lane: V as boxes of kBoxTiles row tiles ending at row tile
    // hi (lanes 0..; a box never leaves [0, ntile): ntile >= 4 on this path),
    // T as one bulk copy (lane 30), the C1 window as one 4-tile box at row
    // tile j0/8 (lane 31; j0 % 8 == 0 on this path)
    const int nv = vt ? (hi - lo + kBoxTiles - 1) / kBoxTiles : 0;
    const unsigned tbytes = vt ? (unsigned)(bw * J.ib) * 8u : 0u;
    if (lane == 0)
      mbar_expect_tx(buf, (unsigned)nv * (2048u * kBoxTiles) + tbytes + (KIND != SU_UN ? 8192u : 0u));
    // generic -> async proxy ordering: global data acquired from other SMs,
    // this CTA's shared-memory writes (masked band tiles of earlier blocks)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane < nv) {
      const int e = hi - kBoxTiles * lane, st = e - kBoxTiles > 0 ? e - kBoxTiles : 0;
      tma_box(smem + L.offV[buf] + st * 256, J.mV, J.vcol + j0, st, buf);
    } else if (lane == 30 && vt) {
      tma_bulk(smem + L.offT[buf], J.Tslot + (size_t)j0 * J.ib, tbytes, buf);
    } else if (lane == 31 && KIND != SU_UN) {
      tma_box(smem + L.offC1[buf], J.mC1, J.c1col + J.cs, j0 >> 3, buf);
    }
  } else {
    if (vt) {
      load_tiles8(smem + L.offV[buf] + lo * 256, J.Vt, J.nb, 8 * lo, hi - lo, j0, bw);
      load_tblock(smem + L.offT[buf], J.Tslot, J.ib, j0, bw);
    }
    if (KIND != SU_UN) load_tiles8(smem + L.offC1[buf], J.C1, J.nb, j0, (bw + 7) >> 3, J.cs, J.wsz);
  }
  mbar_arrive_cp(buf);
}

// Row tile of slot s of row group rg. Slots are dealt so that the tiles a
// block touches are always a PREFIX of every warp's slots (UN: bottom-up, since
// block b touches rows j0..nb-1; TT/TS: top-down, rows 0..): the math then runs
// as fully unrolled instances for n = 0..kSlots active slots without a
// per-slot guard around the DMMAs (a DMMA under a runtime branch serialises).
template <int KIND>
__device__ __forceinline__ int su_tile(int rg, int s, int ntile) {
  return KIND == SU_UN ? ntile - 1 - rg - 4 * s : rg + 4 * s;
}
// active slots of row group rg when the touched row tiles are [lo, hi)
template <int KIND>
__device__ __forceinline__ int su_nact(int rg, int lo, int hi, int ntile) {
  const int R = KIND == SU_UN ? ntile - lo : hi;
  return R > rg ? (R - rg + 3) >> 2 : 0;
}

// phase 1 on N slots: partial W^T (16 columns x 32 reflectors) += C^T V
template <int KIND, int N>
__device__ __forceinline__ void su_p1(const double (&acc)[kSlots][4], double (&w)[4][4], double *Vb, int rg,
                                      int ntile, int j0, int band_lo, int band_hi, bool wb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int s = 0; s < N; ++s) {
    const int j = su_tile<KIND>(rg, s, ntile);
    double *vt = Vb + j * 256 + g * 8 + 2 * t;
    double2 bv[4];
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) bv[nn] = *reinterpret_cast<const double2 *>(vt + 64 * ((TQR_EXP & 128) ? 0 : nn));
    // the band tiles (<= 5, crossing the block's diagonal) are always among
    // the last two active slots: mask them here and store the masked tile back
    // (both column groups store the same values) so phase 3 reads a clean V
    if (KIND != SU_TS && s + 2 >= N && j < band_hi && j >= band_lo) {
      const int r = 8 * j + 2 * t;
#pragma unroll
      for (int nn = 0; nn < 4; ++nn) {
        bv[nn].x = vmask<KIND>(bv[nn].x, r, 8 * nn + g, j0);
        bv[nn].y = vmask<KIND>(bv[nn].y, r + 1, 8 * nn + g, j0);
      }
      if (wb) {
#pragma unroll
        for (int nn = 0; nn < 4; ++nn) *reinterpret_cast<double2 *>(vt + 64 * nn) = bv[nn];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // before a later TMA refill of this buffer
      }
    }
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) dmma(w[nn], acc[s][0], acc[s][2], bv[nn].x);
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) dmma(w[nn], acc[s][1], acc[s][3], bv[nn].y);
  }
}
// phase 3 on N slots: C^T += W2^T V^T (W2^T fragments wa0/wa1 per k-step; V already masked)
template <int KIND, int N>
__device__ __forceinline__ void su_p3(double (&acc)[kSlots][4], const double *W2c, const double *Vb, int rg,
                                      int ntile) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const double wa0 = W2c[(4 * kk) * kLdw], wa1 = W2c[8 + (4 * kk) * kLdw];   // W2^T fragment of this k-step
    double bb[N > 0 ? N : 1];
#pragma unroll
    for (int s = 0; s < N; ++s) {
      const int j = su_tile<KIND>(rg, s, ntile);
      bb[s] = Vb[j * 256 + (4 * ((TQR_EXP & 256) ? 0 : kk) + t) * 8 + g];
    }
#pragma unroll
    for (int s = 0; s < N; ++s) dmma(acc[s], wa0, wa1, bb[s]);
  }
}

#define TQR_SLOT_SWITCH(n, CALL)                                                            \
  switch (n) {                                                                              \
    case 1: CALL(1); break; case 2: CALL(2); break; case 3: CALL(3); break;                 \
    case 4: CALL(4); break; case 5: CALL(5); break; case 6: CALL(6); break;                 \
    case 7: CALL(7); break; case 8: CALL(8); break; default: break;                         \
  }

__device__ __forceinline__ void group_sync(int id) {   // named barrier of one 4-warp column group
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}

// C strip <-> registers: acc[s] = C^T fragment of row tile su_tile(rg, s)
// (columns cg, cg+8; rows 8j+2t, 8j+2t+1); only the first `ntask` slots hold
// rows of this task
template <int KIND>
__device__ __forceinline__ void su_load_c(const StripJob &J, double (&acc)[kSlots][4], int rg, int ntask, int ntile) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int cg = 16 * (warp >> 2) + g, nb = J.nb, wsz = J.wsz;
  const bool even = (nb & 1) == 0;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    const int j = su_tile<KIND>(rg, s, ntile), r = 8 * j + 2 * t;
    const bool act = s < ntask && r < nb;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = cg + 8 * h;
      double x0 = 0.0, x1 = 0.0;
      if (act && col < wsz) {
        const double *src = J.C2 + r + (size_t)(J.cs + col) * nb;
        if (even) {
          const double2 v = __ldcg(reinterpret_cast<const double2 *>(src));
          x0 = v.x; x1 = v.y;
        } else {
          x0 = __ldcg(src);
          if (r + 1 < nb) x1 = __ldcg(src + 1);
        }
      }
      acc[s][2 * h] = x0;
      acc[s][2 * h + 1] = x1;
    }
  }
}
template <int KIND>
__device__ __forceinline__ void su_store_c(const StripJob &J, const double (&acc)[kSlots][4], int rg, int ntask,
                                           int ntile) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int cg = 16 * (warp >> 2) + g, nb = J.nb, wsz = J.wsz;
  const bool even = (nb & 1) == 0;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    const int j = su_tile<KIND>(rg, s, ntile), r = 8 * j + 2 * t;
    const bool act = s < ntask && r < nb;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = cg + 8 * h;
      if (act && col < wsz) {
        double *dst = J.C2 + r + (size_t)(J.cs + col) * nb;
        if (even) {
          *reinterpret_cast<double2 *>(dst) = make_double2(acc[s][2 * h], acc[s][2 * h + 1]);
        } else {
          dst[0] = acc[s][2 * h];
          if (r + 1 < nb) dst[1] = acc[s][2 * h + 1];
        }
      }
    }
  }
}

// The block loop of one strip job. Block idx uses buffer (base + idx) & 1; the
// copies of the first two blocks were issued by the caller. The 8th warp done
// with a buffer refills it with block idx + 2, or, past the job's last block,
// with the blocks of the next job JN (a TT job: fused UNMQR + TTMQR tasks).
template <int KIND>
__device__ __forceinline__ void su_loop(const StripJob &J, const StripJob *JN, double *smem, const SmemLayout &L,
                                        unsigned &ph, double (&acc)[kSlots][4], int rg, int base, bool wait0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int mh = warp >> 2, cg = 16 * mh + g, gbar = 1 + mh;
  const int nb = J.nb, ib = J.ib, ntile = L.ntile, wsz = J.wsz;
  const int nblk = J.b_hi - J.b_lo;
  const bool active = 16 * mh < wsz;                  // a column group beyond a narrow strip idles
  auto blk = [&](int idx) { return J.trans ? J.b_lo + idx : J.b_hi - 1 - idx; };

  for (int idx = 0; idx < nblk; ++idx) {
    const int cur = (base + idx) & 1;
    const int b = blk(idx);
    const int j0 = b * ib, bw = min(ib, nb - j0);
    int blo, bhi;
    su_range<KIND>(j0, bw, ntile, blo, bhi);
    const int nact = active ? su_nact<KIND>(rg, blo, bhi, ntile) : 0;
    const int band_lo = j0 >> 3, band_hi = (j0 + bw + 7) >> 3;   // tiles crossing the block's diagonal
    if (idx > 0 || wait0) mbar_wait(cur, ph);
    prof_mark(idx == 0 ? PH_LOAD : PH_PANEL);   // (tracer: first copy wait vs later ones)
    double *Vb = smem + L.offV[cur];
    const double *Tb = smem + L.offT[cur], *C1w = smem + L.offC1[cur];

    // ---- phase 1: partial W^T (16 columns x 32 reflectors) over this warp's row tiles
    double wacc[4][4];
#pragma unroll
    for (int nn = 0; nn < 4; ++nn)
#pragma unroll
      for (int e = 0; e < 4; ++e) wacc[nn][e] = 0.0;
#define TQR_P1(N) su_p1<KIND, N>(acc, wacc, Vb, rg, ntile, j0, band_lo, band_hi, true)
    for (int rep = 0; rep < ((TQR_EXP & 32) ? 4 : 1); ++rep) {
      TQR_SLOT_SWITCH(nact, TQR_P1)
    }
#undef TQR_P1
    {
      double *Wp = smem + L.offWp + rg * 32 * kLdwP;
#pragma unroll
      for (int nn = 0; nn < 4; ++nn) {
        const int rf = 8 * nn + 2 * t;
        Wp[cg + rf * kLdwP] = wacc[nn][0];
        Wp[cg + (rf + 1) * kLdwP] = wacc[nn][1];
        Wp[cg + 8 + rf * kLdwP] = wacc[nn][2];
        Wp[cg + 8 + (rf + 1) * kLdwP] = wacc[nn][3];
      }
    }
    // phase-2 B operand (loaded here, not at block start: 16 registers less across phase 1): op(T)^T fragments of this warp's n-tile (T upper triangular, zero-padded)
    double tb[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int r = J.trans ? 4 * kk + t : 8 * rg + g, c = J.trans ? 8 * rg + g : 4 * kk + t;
      tb[kk] = (r <= c && c < bw) ? Tb[r + c * ib] : 0.0;
    }
    group_sync(gbar);
    prof_mark(PH_MMA1);

    // ---- reduction: W^T = the group's 4 partials (+ the C1 window: identity part of V);
    // every warp reduces the accumulator positions of its own n-tile rg (a quarter of
    // the group's W^T) instead of all four warps summing all of it while loading
    double2 c1w[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    {
      const double *Wp0 = smem + L.offWp;
      double *W = smem + L.offW;
      const int rf = 8 * rg + 2 * t;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int o = cg + 8 * h + rf * kLdwP, ow = cg + 8 * h + rf * kLdw;
        double r0 = (Wp0[o] + Wp0[o + 32 * kLdwP]) + (Wp0[o + 64 * kLdwP] + Wp0[o + 96 * kLdwP]);
        double r1 = (Wp0[o + kLdwP] + Wp0[o + kLdwP + 32 * kLdwP]) + (Wp0[o + kLdwP + 64 * kLdwP] + Wp0[o + kLdwP + 96 * kLdwP]);
        if (KIND != SU_UN) {
          c1w[h] = *reinterpret_cast<const double2 *>(C1w + rg * 256 + (cg + 8 * h) * 8 + 2 * t);
          r0 += c1w[h].x;
          r1 += c1w[h].y;
        }
        W[ow] = r0;
        W[ow + kLdw] = r1;
      }
    }
    group_sync(gbar);
    // ---- phase 2: W2^T fragment (columns 16 mh.., reflectors 8 rg..) = -W^T op(T)^T
    {
      const double *Wr = smem + L.offW;
      double *W2 = smem + L.offW2;
      double a2[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int o0 = (16 * mh + g) + (4 * kk + t) * kLdw;
        dmma(a2[kk & 1], Wr[o0], Wr[o0 + 8], tb[kk]);
      }
      prof_mark(PH_FIX);
      double w2[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) w2[e] = -(a2[0][e] + a2[1][e]);
      const int rf = 8 * rg + 2 * t;
      W2[(16 * mh + g) + rf * kLdw] = w2[0];
      W2[(16 * mh + g) + (rf + 1) * kLdw] = w2[1];
      W2[(16 * mh + g + 8) + rf * kLdw] = w2[2];
      W2[(16 * mh + g + 8) + (rf + 1) * kLdw] = w2[3];
      if (KIND != SU_UN) {   // C1_b rows j0 + rf, rf + 1 += W2 (straight to global)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 16 * mh + g + 8 * h;
          if (col < wsz && rf < bw) {
            const double2 c1 = c1w[h];
            double *dst = J.C1 + (j0 + rf) + (size_t)(J.cs + col) * nb;
            const double v0 = c1.x + w2[2 * h], v1 = c1.y + w2[2 * h + 1];
            if (rf + 1 < bw && ((nb | j0) & 1) == 0) {
              *reinterpret_cast<double2 *>(dst) = make_double2(v0, v1);
            } else {
              dst[0] = v0;
              if (rf + 1 < bw) dst[1] = v1;
            }
          }
        }
      }
    }
    group_sync(gbar);
    prof_mark(PH_TRI);

    // ---- phase 3: C^T += W2^T V^T on this warp's row tiles
    {
      const double *W2c = smem + L.offW2 + cg + t * kLdw;
#define TQR_P3(N) su_p3<KIND, N>(acc, W2c, Vb, rg, ntile)
      for (int rep = 0; rep < ((TQR_EXP & 64) ? 4 : 1); ++rep) {
        TQR_SLOT_SWITCH(nact, TQR_P3)
      }
#undef TQR_P3
    }
    prof_mark(PH_MMA3);
    // this warp is done with buffer `cur`; the 8th warp to finish refills it with block idx + 2
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      __threadfence_block();
      last = atomicAdd(&s_done[cur], 1) == kWarps - 1;
      if (last) s_done[cur] = 0;
      __threadfence_block();
    }
    if (__shfl_sync(0xffffffffu, last, 0)) {
      if (idx + 2 < nblk) {
        su_issue<KIND>(J, L, smem, cur, blk(idx + 2));
      } else if (KIND == SU_UN && JN != nullptr) {
        const int n = idx + 2 - nblk;
        if (n < JN->b_hi - JN->b_lo) su_issue<SU_TT>(*JN, L, smem, cur, JN->trans ? JN->b_lo + n : JN->b_hi - 1 - n);
      }
    }
  }
}

template <int KIND>
__device__ void strip_update(const StripJob &J, double *smem, const SmemLayout &L, unsigned &ph) {
  const int warp = threadIdx.x >> 5;
  // two independent column groups (warps 0-3: columns 0-15, warps 4-7:
  // columns 16-31), one warp per SM sub-partition each, synchronised only by
  // their own named barriers: one group's latency-bound steps (reduction,
  // phase 2, copy issue) overlap the other group's DMMA phases
  // the row groups of column group 1 are rotated by one against group 0's, so
  // the row group with an extra row tile (n_tiles % 4 != 0) lands on two
  // different sub-partitions (warp w runs on sub-partition w % 4)
  const int mh = warp >> 2, rg = (warp + mh) & 3;
  const int ib = J.ib, nb = J.nb, ntile = L.ntile;
  const int nblk = J.b_hi - J.b_lo;
  int ct_lo = 0, ct_hi = ntile;                       // row tiles of C this task touches
  if (KIND == SU_UN) ct_lo = (J.b_lo * ib) >> 3;
  if (KIND == SU_TT) ct_hi = (min(J.b_hi * ib, nb) + 7) >> 3;
  const int ntask = su_nact<KIND>(rg, ct_lo, ct_hi, ntile);   // slots holding C rows of this task
  const bool wait0 = !J.resident || KIND != SU_UN;     // resident TT/TS blocks still load their C1 window
  auto blk = [&](int idx) { return J.trans ? J.b_lo + idx : J.b_hi - 1 - idx; };
  if (warp == 0) {                                    // both buffers are free: blocks 0 and 1
    if (wait0) su_issue<KIND>(J, L, smem, 0, blk(0), !J.resident);
    if (nblk > 1) su_issue<KIND>(J, L, smem, 1, blk(1));
  }
  double acc[kSlots][4];
  su_load_c<KIND>(J, acc, rg, ntask, ntile);
  su_loop<KIND>(J, nullptr, smem, L, ph, acc, rg, 0, wait0);
  su_store_c<KIND>(J, acc, rg, ntask, ntile);
}

// Fused UNMQR + TTMQR of one strip of tile (i, j) (K_UNTTMQR): the UNMQR by
// GEQRT(i, k)'s reflectors (JU) and then the TTMQR by TTQRT(i, piv, k)'s (JT)
// with the strip of tile (i, j) kept in registers between the two, and the
// TT job's first blocks streamed in behind the UN job's last ones. Both jobs
// cover all blocks, so every row tile is live. The UN loop deals row tiles
// bottom-up (tile ntile-1-rg-4s), the TT loop top-down (tile rg'+4s'): with
// rg' = (ntile-1-rg) & 3 a warp keeps the same row tiles, in reversed slot
// order, so the hand-over is a register permutation. Same arithmetic, in the
// same order, as the two separate tasks (bit-identical results).
__device__ void strip_update_untt(const StripJob &JU, const StripJob &JT, double *smem, const SmemLayout &L,
                                  unsigned &ph) {
  const int warp = threadIdx.x >> 5;
  const int mh = warp >> 2, rg = (warp + mh) & 3;
  const int ntile = L.ntile;
  const int rg2 = (ntile - 1 - rg) & 3;
  const int nu = JU.b_hi - JU.b_lo, nt = JT.b_hi - JT.b_lo;
  const int ntask = su_nact<SU_UN>(rg, 0, ntile, ntile);
  if (warp == 0) {   // sequence blocks 0 and 1 (UN blocks, then TT blocks)
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      if (x < nu) su_issue<SU_UN>(JU, L, smem, x, JU.trans ? JU.b_lo + x : JU.b_hi - 1 - x);
      else if (x - nu < nt) su_issue<SU_TT>(JT, L, smem, x, JT.trans ? JT.b_lo + x - nu : JT.b_hi - 1 - (x - nu));
    }
  }
  double acc[kSlots][4];
  su_load_c<SU_UN>(JU, acc, rg, ntask, ntile);
  su_loop<SU_UN>(JU, &JT, smem, L, ph, acc, rg, 0, true);
  // slot s (tile ntile-1-rg-4s) -> slot ntask-1-s (tile rg2 + 4(ntask-1-s))
#define TQR_REV(M)                                                  \
  {                                                                 \
    double tmp[kSlots][4];                                          \
    _Pragma("unroll") for (int s = 0; s < kSlots; ++s)              \
    _Pragma("unroll") for (int e = 0; e < 4; ++e)                   \
      tmp[s][e] = s < (M) ? acc[(M) - 1 - s][e] : 0.0;              \
    _Pragma("unroll") for (int s = 0; s < kSlots; ++s)              \
    _Pragma("unroll") for (int e = 0; e < 4; ++e) acc[s][e] = tmp[s][e]; \
  }
  TQR_SLOT_SWITCH(ntask, TQR_REV)
#undef TQR_REV
  su_loop<SU_TT>(JT, nullptr, smem, L, ph, acc, rg2, nu & 1, true);
  su_store_c<SU_TT>(JT, acc, rg2, ntask, ntile);
}

// ---- panel kernels: GEQRT / TTQRT / TSQRT on whole tiles ------------------
// (monolithic form, TQR_SPLIT=0: every block's trailing update runs here)
template <int MODE>
__device__ void panel_task(double *X, double *A1, double *Tslot, int nb, int ib, int ws, double *smem,
                           const SmemLayout &L, unsigned &ph, const CUtensorMap *mA, int a1col) {
  for (int j0 = 0; j0 < nb; j0 += ib) {
    const int bw = min(ib, nb - j0);
    panel_block<MODE>(X, A1, Tslot, nb, ib, j0, bw, smem + L.offV[0], smem + L.offT[0], smem + L.offWp);
    __syncthreads();
    for (int cs = j0 + bw; cs < nb; cs += ws) {
      const StripJob J{X, Tslot, A1, X, nb, ib, cs, min(ws, nb - cs), j0 / ib, j0 / ib + 1, true, true, mA, mA, 0,
                       a1col};
      if (MODE == 0) strip_update<SU_UN>(J, smem, L, ph);
      else if (MODE == 1) strip_update<SU_TT>(J, smem, L, ph);
      else strip_update<SU_TS>(J, smem, L, ph);
      __syncthreads();
    }
  }
}

__device__ void run_task(const RunArgs &a, const DevTask &t, double *smem, const SmemLayout &L, bool resident,
                         unsigned &ph) {
  const int p = a.p, nb = a.nb, ib = a.ib, ws = a.ws;
  const int nblk = (nb + ib - 1) / ib;
  double *Vb = smem + L.offV[0], *Tb = smem + L.offT[0], *scr = smem + L.offWp;
  const CUtensorMap *mA = a.tma ? &a.mapA : nullptr, *mC = a.tma ? &a.mapC : nullptr;
  auto col = [&](int i, int k) { return (k * p + i) * nb; };   // global column of tile (i, k)
  switch (t.kind) {
    case K_GEQRT:
      panel_task<0>(tile_ptr(a.A, p, nb, t.i, t.k), nullptr, tslot_ptr(a.T, p, nb, ib, t.i, t.k, 0), nb, ib, ws,
                    smem, L, ph, mA, 0);
      break;
    case K_TTQRT:
      panel_task<1>(tile_ptr(a.A, p, nb, t.i, t.k), tile_ptr(a.A, p, nb, t.piv, t.k),
                    tslot_ptr(a.T, p, nb, ib, t.i, t.k, 1), nb, ib, ws, smem, L, ph, mA, col(t.piv, t.k));
      break;
    case K_TSQRT:
      panel_task<2>(tile_ptr(a.A, p, nb, t.i, t.k), tile_ptr(a.A, p, nb, t.piv, t.k),
                    tslot_ptr(a.T, p, nb, ib, t.i, t.k, 1), nb, ib, ws, smem, L, ph, mA, col(t.piv, t.k));
      break;
    // ---- split panels: inner block s of the panel, or update of strip s by block j
    case K_GEQRT_B: {
      const int j0 = t.s * ib;
      panel_block<0>(tile_ptr(a.A, p, nb, t.i, t.k), nullptr, tslot_ptr(a.T, p, nb, ib, t.i, t.k, 0), nb, ib, j0,
                     min(ib, nb - j0), Vb, Tb, scr);
      break;
    }
    case K_TTQRT_B:
    case K_TSQRT_B: {
      const int j0 = t.s * ib;
      double *X = tile_ptr(a.A, p, nb, t.i, t.k), *A1 = tile_ptr(a.A, p, nb, t.piv, t.k);
      double *Tsl = tslot_ptr(a.T, p, nb, ib, t.i, t.k, 1);
      if (t.kind == K_TTQRT_B) panel_block<1>(X, A1, Tsl, nb, ib, j0, min(ib, nb - j0), Vb, Tb, scr);
      else panel_block<2>(X, A1, Tsl, nb, ib, j0, min(ib, nb - j0), Vb, Tb, scr);
      break;
    }
    case K_GEQRT_U: {
      const int cs = t.s * ws;
      double *X = tile_ptr(a.A, p, nb, t.i, t.k);
      const StripJob J{X, tslot_ptr(a.T, p, nb, ib, t.i, t.k, 0), nullptr, X, nb, ib, cs, min(ws, nb - cs),
                       t.j, t.j + 1, true, resident, mA, mA, col(t.i, t.k), 0};
      strip_update<SU_UN>(J, smem, L, ph);
      break;
    }
    case K_TTQRT_U:
    case K_TSQRT_U: {
      const int cs = t.s * ws;
      double *X = tile_ptr(a.A, p, nb, t.i, t.k);
      const StripJob J{X, tslot_ptr(a.T, p, nb, ib, t.i, t.k, 1), tile_ptr(a.A, p, nb, t.piv, t.k), X, nb, ib, cs,
                       min(ws, nb - cs), t.j, t.j + 1, true, resident, mA, mA, col(t.i, t.k), col(t.piv, t.k)};
      if (t.kind == K_TTQRT_U) strip_update<SU_TT>(J, smem, L, ph);
      else strip_update<SU_TS>(J, smem, L, ph);
      break;
    }
    // ---- updates of other tiles (factorization) and of C (apply)
    case K_UNMQR:
    case K_AP_UNMQR: {
      double *Cbase = t.kind == K_UNMQR ? a.A : a.C;
      for (int u = 0; u < max(t.pad, 1); ++u) {   // (multi-strip task: its strips in turn)
        if (u > 0) __syncthreads();
        const int cs = (t.s + u) * ws;
        const StripJob J{tile_ptr(a.A, p, nb, t.i, t.k), tslot_ptr(a.T, p, nb, ib, t.i, t.k, 0), nullptr,
                         tile_ptr(Cbase, p, nb, t.i, t.j), nb, ib, cs, min(ws, nb - cs), 0, nblk, a.trans != 0, false,
                         mA, t.kind == K_UNMQR ? mA : mC, col(t.i, t.k), 0};
        strip_update<SU_UN>(J, smem, L, ph);
      }
      break;
    }
    case K_UNTTMQR: {   // fused UNMQR by GEQRT(i, k) + TTMQR by TTQRT(i, piv, k) of tile (i, j)
      for (int u = 0; u < max(t.pad, 1); ++u) {
        if (u > 0) __syncthreads();
        const int cs = (t.s + u) * ws;
        double *Ci = tile_ptr(a.A, p, nb, t.i, t.j);
        const StripJob JU{tile_ptr(a.A, p, nb, t.i, t.k), tslot_ptr(a.T, p, nb, ib, t.i, t.k, 0), nullptr, Ci, nb, ib,
                          cs, min(ws, nb - cs), 0, nblk, true, false, mA, mA, col(t.i, t.k), 0};
        const StripJob JT{tile_ptr(a.A, p, nb, t.i, t.k), tslot_ptr(a.T, p, nb, ib, t.i, t.k, 1),
                          tile_ptr(a.A, p, nb, t.piv, t.j), Ci, nb, ib, cs, min(ws, nb - cs), 0, nblk, true, false,
                          mA, mA, col(t.i, t.k), col(t.piv, t.j)};
        strip_update_untt(JU, JT, smem, L, ph);
      }
      break;
    }
    case K_TTMQR:
    case K_TSMQR:
    case K_AP_TTMQR:
    case K_AP_TSMQR: {
      const bool ap = t.kind == K_AP_TTMQR || t.kind == K_AP_TSMQR;
      const bool tri = t.kind == K_TTMQR || t.kind == K_AP_TTMQR;
      double *Cbase = ap ? a.C : a.A;
      for (int u = 0; u < max(t.pad, 1); ++u) {
        if (u > 0) __syncthreads();
        const int cs = (t.s + u) * ws;
        const StripJob J{tile_ptr(a.A, p, nb, t.i, t.k), tslot_ptr(a.T, p, nb, ib, t.i, t.k, 1),
                         tile_ptr(Cbase, p, nb, t.piv, t.j), tile_ptr(Cbase, p, nb, t.i, t.j), nb, ib, cs,
                         min(ws, nb - cs), 0, nblk, a.trans != 0, false, mA, ap ? mC : mA, col(t.i, t.k),
                         col(t.piv, t.j)};
        if (tri) strip_update<SU_TT>(J, smem, L, ph);
        else strip_update<SU_TS>(J, smem, L, ph);
      }
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

__global__ void __launch_bounds__(kThreads, 1) tqr_persistent(const __grid_constant__ RunArgs a) {
  extern __shared__ __align__(128) double smem[];   // (TMA tensor copies need 128-byte-aligned destinations)
  __shared__ int s_task, s_chain, s_resident;
  const SmemLayout L = smem_layout(a.nb, a.ib, a.ws);
  if (threadIdx.x == 0) {
    s_prof_on = 0; s_chain = -1; s_resident = 0; mbar_init_all();
    s_epoch = (unsigned)ld_acquire(&a.ctrl[kCtrlEpoch]);
  }
  unsigned ph = 0u;     // parity bits of the two buffer mbarriers (identical in every thread)
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
    run_task(a, tk, smem, L, s_resident != 0, ph);
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
