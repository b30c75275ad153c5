/*
 * tiledqr.h — C ABI of the B200-native tiled QR hot path of arXiv:1104.4475
 * ("Tiled QR factorization algorithms", Bouwmeester, Jacquelin, Langou, Robert).
 *
 * Citations are PAPER.md line numbers with the section they fall in.
 *
 * CONVENTIONS (all entry points)
 *   - Plain C types only; no torch / CUDA types in the signatures. A `stream`
 *     argument is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Tile indices in elimination lists are 1-based, as in the paper
 *     (Algorithm 1: elim(i, piv(i,k), k) zeroes tile (i,k) with
 *     row piv(i,k)).
 *   - Tiled matrix layout in memory: an m x n fp64 matrix,
 *     m = p*nb, n = q*nb, is stored as p*q contiguous nb x nb tiles; tile
 *     (i,k) (0-based) starts at element (k*p + i)*nb*nb and is column-major
 *     inside (leading dimension nb). Column strips of a tile are therefore
 *     contiguous in memory.
 *   - After tiled_qr, tile (i,k) holds R and Householder vectors exactly as
 *     LAPACK GEQRT / TPQRT store them (Table 1):
 *       GEQRT(r,k):    upper triangle incl. diagonal = R, strict lower = V
 *       TTQRT(i,p,k):  upper triangle incl. diagonal of tile (i,k) = V2
 *       TSQRT(i,p,k):  whole tile (i,k) = V2
 *     R (n x n) is the upper triangle of the top q x q tiles.
 *   - T buffer (compact-WY factors, lines 62-66, inner blocking i_b line 1031):
 *     p*q*2 slots of ib x nb doubles, column-major (ld = ib); slot 0 of tile
 *     (i,k) = T of GEQRT(i,k), slot 1 = T of TTQRT/TSQRT that zeroed (i,k);
 *     slot s of tile (i,k) starts at element (((k*p + i)*2 + s) * ib*nb).
 *     Inner block b (columns b*ib .. b*ib+ib-1) stores its ib x ib upper
 *     triangular T (zeros below the diagonal and in unused rows).
 *   - Ownership: the caller owns every buffer. The library caches execution
 *     plans (task graphs uploaded to device memory) keyed by shape, tree and
 *     device; tqr_release_plans() frees them. Calls that share a plan key
 *     must not run concurrently on different streams.
 *   - Errors: int-returning calls return 0 (or a non-negative count) on
 *     success and a negative TQR_E* code on failure; tqr_last_error() then
 *     returns a thread-local message. Device faults are reported by the next
 *     call that synchronises (CUDA semantics). Nothing falls back to the CPU.
 */
#ifndef TILEDQR_H
#define TILEDQR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Trees (elimination schemes), §3.1-§3.2 */
enum tqr_tree {
  TQR_FLAT = 0,       /* Sameh-Kuck / FlatTree, line 488 */
  TQR_FIBONACCI = 1,  /* Fibonacci scheme of order 1, lines 490-505 */
  TQR_GREEDY = 2,     /* Greedy, lines 507-512 and Algorithm 4 (lines 563-619) */
  TQR_BINARY = 3,     /* BinaryTree, lines 914-918 */
  TQR_PLASMA = 4,     /* PlasmaTree(BS): flat inside domains of BS rows + binary
                         merge of the domain heads, lines 936-953 */
  TQR_MERGE = 5,      /* merge of two stacked tile-upper-triangular R factors
                         [R1; R2] (p = 2q): column k zeroes tiles (q+t, k),
                         t = 1..k, against pivot row k. Used by the cross-GPU
                         reduction of tall-skinny matrices: the
                         input's diagonal tiles count as triangles, tiles below
                         them as structural zeros (they must hold zeros). */
  TQR_ASAP = 6,       /* ASAP, lines 666-682: eliminations decided while the
                         tiled algorithm runs: one starts as soon as two rows
                         are ready */
  TQR_GRASAP = 7      /* Grasap(k), lines 685-692: Greedy on columns 1..q-k,
                         ASAP on the last k columns; k is passed as `bs` */
};

/* Kernel families, §2.1 (lines 231-352) */
enum tqr_family {
  TQR_TT = 0,  /* triangle on top of triangle: GEQRT+UNMQR both rows, TTQRT+TTMQR (Algorithm 3) */
  TQR_TS = 1   /* triangle on top of square: GEQRT+UNMQR pivot row, TSQRT+TSMQR (Algorithm 2) */
};

enum tqr_status {
  TQR_OK = 0,
  TQR_EINVAL = -1,    /* bad argument (shape, tree, sizes, null pointer) */
  TQR_ECAP = -2,      /* output capacity too small */
  TQR_ECUDA = -3,     /* CUDA runtime error (message in tqr_last_error) */
  TQR_ENOMEM = -4,    /* host or device allocation failed */
  TQR_EUNSUP = -5     /* configuration outside the supported envelope (nb > 256, ib > 32, ...) */
};

/* ------------------------------------------------------------------------
 * Host-side elimination lists and schedules (no GPU needed)
 * ---------------------------------------------------------------------- */

/* elim_list — the elimination list of `tree` for a p x q tile matrix
 * (p >= q >= 1; §2.2 lines 354-373 for the validity conditions).
 *   bs     PlasmaTree domain size (1 <= bs <= p; ignored by other trees)
 *   i, piv, k   out: 1-based elim(i, piv, k) triplets, in list order
 *   step   out (may be NULL): coarse-grain time-step of each elimination
 *          (Table 2: Sameh-Kuck i+k-2, Fibonacci's closed
 *          form, Greedy's simulation; BinaryTree/PlasmaTree: coarse ASAP of
 *          their list, reading R5)
 *   cap    capacity of each output array
 * List order is DESIGN.md reading R2: flat by (k,i); fibonacci and greedy by
 * (coarse step, k, i); binary by (k, round, i); plasma by (k, phase, round, i).
 * Returns the number of eliminations (= sum_k (p-k) over k <= min(p,q)) or a
 * negative TQR_E* code (TQR_ECAP if cap is too small). */
int elim_list(int p, int q, int tree, int bs,
              int32_t *i, int32_t *piv, int32_t *k, int32_t *step, int64_t cap);

/* critical_path — length of the critical path of the tiled algorithm driven
 * by the list of `tree` with kernel `family`, unbounded processors, in units
 * of nb^3/3 flops (kernel weights of Table 1; execution
 * semantics §2.3). Reproduces Table 6 (lines 1317-1368),
 * Table 5(b) and the closed forms of Theorem 1(1) and Propositions 1-2.
 * Returns the length (>0) or a negative TQR_E* code. */
int64_t critical_path(int p, int q, int tree, int bs, int family);

/* tiled_times — per-tile zeroing time of the same simulation (Table 3,
 * lines 622-649: "the time-steps at which tiles are actually zeroed out").
 *   zero_time   out: p*q int32, column-major over tiles (entry (i,k) 0-based
 *               at k*p + i); tiles on/above the diagonal get 0.
 * Returns the critical path length or a negative TQR_E* code. */
int64_t tiled_times(int p, int q, int tree, int bs, int family, int32_t *zero_time);

/* ------------------------------------------------------------------------
 * Device computation (B200, sm_100a). Pointers are DEVICE pointers.
 * ---------------------------------------------------------------------- */

/* tiled_qr — factor A = QR in place (§2, Algorithm 1 with the list of `tree`,
 * each elimination executed by the TT or TS kernels of Algorithms 2-3).
 *   m, n   matrix size, m = p*nb >= n = q*nb (nb must divide both)
 *   nb     tile size, 1 <= nb <= 256;  ib  inner blocking, 1 <= ib <= 32
 *   A      device, p*q*nb*nb doubles in the tiled layout; overwritten by R/V
 *   T      device, p*q*2*ib*nb doubles; overwritten by the compact-WY factors
 * The whole factorization is ONE persistent kernel launch on `stream`: a
 * dataflow scheduler with per-task dependency counters and priority ready
 * queues; every CTA only takes tasks whose inputs are complete.
 * Returns 0 or a negative TQR_E* code; asynchronous w.r.t. the host. */
int tiled_qr(int m, int n, int nb, int ib, int tree, int bs, int family,
             double *A, double *T, void *stream);

/* apply_qt / apply_q — C <- Q^T C  /  C <- Q C with the Q of a previous
 * tiled_qr(m, n, nb, ib, tree, bs, family, A, T) (same arguments).
 *   C      device, m x nrhs in the tiled layout with p tile rows and
 *          nrhs/nb tile columns (nrhs must be a multiple of nb)
 * Q^T replays the panel kernels (GEQRT -> UNMQR, TxQRT -> TxMQR) in list
 * emission order on the rows of C; Q replays them transposed in reverse.
 * Returns 0 or a negative TQR_E* code. */
int apply_qt(int m, int n, int nb, int ib, int tree, int bs, int family,
             const double *A, const double *T, double *C, int nrhs, void *stream);
int apply_q(int m, int n, int nb, int ib, int tree, int bs, int family,
            const double *A, const double *T, double *C, int nrhs, void *stream);

/* tiled_qr_host — end-to-end variant on HOST buffers (pinned or pageable):
 * copies A to the device, factors, copies A (R and V) and T back, all on
 * `stream`, and synchronises it. Device scratch is cached per shape. */
int tiled_qr_host(int m, int n, int nb, int ib, int tree, int bs, int family,
                  double *A_host, double *T_host, void *stream);

/* Diagnostics: per-task tracing of the persistent kernel. While enabled, every
 * launch records, per task, globaltimer stamps (taken, dependencies ready,
 * done) and the SM id. tqr_trace_fetch copies the last traced launch to
 * `out` as 16 uint64 per task in execution-priority order: taken, ready, done,
 * smid, kind (Table 1 kernel: 0 GEQRT, 1 UNMQR, 2 TTQRT, 3 TTMQR, 4 TSQRT,
 * 5 TSMQR, 6-8 apply kinds), i | piv<<16, k | j<<16 (0-based), strip, then
 * 8 SM-cycle counters of the task's phases (load wait, V fix-up, V^T C
 * contraction, T multiply, V W contraction, panel columns, T recurrence,
 * stores/other). Returns the task count or a negative TQR_E* code
 * (TQR_ECAP if cap < 16*n). */
int tqr_trace_enable(int on);
int64_t tqr_trace_fetch(uint64_t *out, int64_t cap);
/* Successor lists (CSR, task ids in trace order) of the last traced plan:
 * succ_ptr[ntask+1], succ[...]. Returns the number of edges or TQR_E*. */
int64_t tqr_trace_graph(int32_t *succ_ptr, int32_t *succ, int64_t cap);

/* Diagnostics, host only (no GPU): the device task graph tiled_qr would run
 * (strip width ws, 0 = default; split bit 0 = per-inner-block panel tasks,
 * bit 1 / bit 2 = UNMQR+TTMQR fusion on / off (neither: TQR_FUSE, default off),
 * bits 8.. = strips per update task, 0 = default). Fills
 * out_tasks with 8 int32 per task (kind, i, piv, k, j, s, chain, meta) in
 * priority order and the successor CSR (succ_ptr[ntask+1], succ). With null
 * outputs it only returns the task count. Returns ntask or a TQR_E* code. */
int64_t tqr_plan_graph(int m, int n, int nb, int ib, int tree, int bs, int family, int ws, int split,
                       int32_t *out_tasks, int64_t task_cap, int32_t *succ_ptr, int32_t *succ, int64_t succ_cap);

/* tiled_qr_host_async — pipelined end-to-end variant: enqueues the upload of
 * A_host (pinned host memory for real overlap), the factorization on
 * `stream`, and the download of the factored A (R and V) into R_host and of T
 * into T_host, and returns. Consecutive calls alternate between two device
 * slots and two internal copy streams, so copies overlap the neighbouring
 * calls' compute. A_host must stay valid and R_host/T_host must not be read
 * until tqr_host_wait() returns. Returns 0 or a negative TQR_E* code. */
int tiled_qr_host_async(int m, int n, int nb, int ib, int tree, int bs, int family,
                        const double *A_host, double *R_host, double *T_host, void *stream);
int tqr_host_wait(void);

/* Number of kernel launches the last device call issued (for bench accounting). */
int tqr_last_launch_count(void);

/* 1 if the last device call moved its V blocks and C1 windows with TMA tensor
 * copies (cp.async.bulk.tensor, needs nb % 8 == 0, ib % 8 == 0, nb >= 32 and
 * TQR_TMA unset or non-zero in the environment), 0 if it used cp.async. */
int tqr_last_launch_tma(void);

/* Free every cached plan and scratch buffer (all devices). */
void tqr_release_plans(void);

/* Thread-local message of the last failing call ("" if none). */
const char *tqr_last_error(void);

/* ABI version (major*100 + minor). */
int tqr_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TILEDQR_H */
