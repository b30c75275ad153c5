// B200 (sm_100a) tiled QR: one persistent dataflow kernel executes the whole
// task graph of an elimination list (§2.3 execution scheme, lines
// 385-411), with the six tile kernels of Table 1 (lines 239-251) as device
// routines. See DESIGN.md §5 for the design and include/tiledqr.h for the ABI.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "plan.h"
#include "tqr_device.cuh"
#include "../../include/tiledqr.h"

using namespace tqr;

// ============================================================================
// Host side: errors, plans, launches
// ============================================================================
static thread_local std::string g_err;
static thread_local int g_launches = 0;
struct DevPlan;
static int g_trace_on = 0;
static DevPlan *g_trace_plan = nullptr;

static int fail(int code, const std::string &msg) { g_err = msg; return code; }
static int cuda_fail(cudaError_t e, const char *where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return TQR_ECUDA;
}
#define CUDA_TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return cuda_fail(_e, #x); } while (0)

extern "C" const char *tqr_last_error(void) { return g_err.c_str(); }
extern "C" int tqr_version(void) { return 100; }
extern "C" int tqr_last_launch_count(void) { return g_launches; }

extern "C" int elim_list(int p, int q, int tree, int bs, int32_t *i, int32_t *piv, int32_t *k,
                         int32_t *step, int64_t cap) {
  std::vector<Elim> lst;
  std::string err;
  if (!build_elim_list(p, q, tree, bs, lst, err)) return fail(TQR_EINVAL, err);
  if ((int64_t)lst.size() > cap) return fail(TQR_ECAP, "elim_list: capacity too small");
  if (!lst.empty() && (!i || !piv || !k)) return fail(TQR_EINVAL, "elim_list: null output");
  for (size_t x = 0; x < lst.size(); ++x) {
    i[x] = lst[x].i; piv[x] = lst[x].piv; k[x] = lst[x].k;
    if (step) step[x] = lst[x].step;
  }
  return (int)lst.size();
}

static int tile_sim(int p, int q, int tree, int bs, int family, std::vector<TileTask> &tt,
                    std::vector<int64_t> &st, std::vector<int64_t> &fin, int64_t &mk) {
  std::vector<Elim> lst;
  std::string err;
  if (family != TQR_TT && family != TQR_TS) return fail(TQR_EINVAL, "unknown kernel family");
  if (!build_elim_list(p, q, tree, bs, lst, err)) return fail(TQR_EINVAL, err);
  expand(lst, p, q, family, tt, tree == TQR_MERGE);
  mk = simulate(tt, st, fin);
  return 0;
}

extern "C" int64_t critical_path(int p, int q, int tree, int bs, int family) {
  std::vector<TileTask> tt;
  std::vector<int64_t> st, fin;
  int64_t mk;
  int rc = tile_sim(p, q, tree, bs, family, tt, st, fin, mk);
  return rc < 0 ? rc : mk;
}

extern "C" int64_t tiled_times(int p, int q, int tree, int bs, int family, int32_t *zt) {
  std::vector<TileTask> tt;
  std::vector<int64_t> st, fin;
  int64_t mk;
  int rc = tile_sim(p, q, tree, bs, family, tt, st, fin, mk);
  if (rc < 0) return rc;
  if (!zt) return fail(TQR_EINVAL, "tiled_times: null output");
  for (int x = 0; x < p * q; ++x) zt[x] = 0;
  for (size_t x = 0; x < tt.size(); ++x)
    if (tt[x].kind == K_TTQRT || tt[x].kind == K_TSQRT)
      zt[(tt[x].k - 1) * p + (tt[x].i - 1)] = (int32_t)fin[x];
  return mk;
}

// ---- strip width and shared-memory footprint --------------------------------
static int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// Column-strip width of the update tasks: 32 columns = 4 n8 DMMA tiles, so the
// W = V^T C contraction of a 32-wide block is exactly one 16x8 fragment per warp
// (DESIGN.md §5); the last strip of a tile may be narrower.
static int pick_ws(int nb, int ib) {
  int forced = env_int("TQR_WS", 0);
  if (forced > 0) return forced < nb ? forced : nb;   // > 32 is rejected by get_plan
  if (nb <= 32) return nb;
  for (int w : {32, 24, 16, 8})
    if (smem_bytes(nb, ib, w) <= kMaxSmem) return w;
  return 8;
}

static int check_shape(int m, int n, int nb, int ib, int &p, int &q);

// strips per update task of the factorization (TQR_MSTRIP; default 3 when q >= 20,
// where parallelism is ample, else 2: profiles/r02_experiments_session3.txt item 10)
static int mstrip_default(int q) {
  const int m = env_int("TQR_MSTRIP", q >= 20 ? 3 : 2);
  return m < 1 ? 1 : (m > 8 ? 8 : m);
}

// UNMQR + TTMQR fusion of the factorization graph (TQR_FUSE=1; off by default:
// delaying each UNMQR until its row's TTQRT is done costs more than the saved
// strip load/store and claim, profiles/r02_experiments_session4.txt item 2)
static bool fuse_default() { return env_int("TQR_FUSE", 0) != 0; }

// ---- plan cache -------------------------------------------------------------
struct DevPlan {
  DevTask *tasks = nullptr;
  int32_t *succ = nullptr;
  int32_t *roots = nullptr;
  unsigned *cnt = nullptr;                // per-task arrivals (accumulate epoch x indegree)
  unsigned long long *queue = nullptr;    // ntask ready-queue slots, split by level (epoch-tagged)
  int *ctrl = nullptr;                    // scheduler counters (kCtrlWords ints)
  unsigned long long *trace = nullptr;    // diagnostic per-task timestamps
  std::vector<DevTask> host_tasks;        // kept for tqr_trace_fetch
  int ntask = 0, nroots = 0;
  int ws = 0;
  int qoff[kLevels + 1] = {0};            // per-level queue offsets
  ~DevPlan() {
    cudaFree(tasks); cudaFree(succ); cudaFree(roots); cudaFree(cnt); cudaFree(queue); cudaFree(ctrl);
    cudaFree(trace);
  }
};

using PlanKey = std::tuple<int, int, int, int, int, int, int, int, int, int, int>;
static std::mutex g_mu;
static std::map<PlanKey, std::unique_ptr<DevPlan>> g_plans;

static int upload(const DevGraph &g, int ws, DevPlan &pl) {
  pl.ntask = (int)g.tasks.size();
  pl.nroots = (int)g.roots.size();
  pl.host_tasks = g.tasks;
  pl.ws = ws;
  const size_t n1 = pl.ntask ? pl.ntask : 1;
  CUDA_TRY(cudaMalloc(&pl.tasks, sizeof(DevTask) * n1));
  // successor edges as (task, that task's meta) pairs: releasing a successor
  // needs its indegree, and one 8-byte load beats two dependent ones
  CUDA_TRY(cudaMalloc(&pl.succ, sizeof(int32_t) * 2 * (g.succ.empty() ? 1 : g.succ.size())));
  CUDA_TRY(cudaMalloc(&pl.roots, sizeof(int32_t) * (g.roots.empty() ? 1 : g.roots.size())));
  CUDA_TRY(cudaMalloc(&pl.cnt, sizeof(unsigned) * n1));
  for (int l = 0; l <= kLevels; ++l) pl.qoff[l] = 0;
  for (const DevTask &t : g.tasks) pl.qoff[((t.meta >> 16) & 15) + 1]++;
  for (int l = 0; l < kLevels; ++l) pl.qoff[l + 1] += pl.qoff[l];
  CUDA_TRY(cudaMalloc(&pl.queue, sizeof(unsigned long long) * n1));
  CUDA_TRY(cudaMalloc(&pl.ctrl, sizeof(int) * kCtrlWords));
  if (!g.tasks.empty()) CUDA_TRY(cudaMemcpy(pl.tasks, g.tasks.data(), sizeof(DevTask) * g.tasks.size(), cudaMemcpyHostToDevice));
  if (!g.succ.empty()) {
    std::vector<int32_t> edges(2 * g.succ.size());
    for (size_t x = 0; x < g.succ.size(); ++x) {
      edges[2 * x] = g.succ[x];
      edges[2 * x + 1] = g.tasks[g.succ[x]].meta;
    }
    CUDA_TRY(cudaMemcpy(pl.succ, edges.data(), sizeof(int32_t) * edges.size(), cudaMemcpyHostToDevice));
  }
  if (!g.roots.empty()) CUDA_TRY(cudaMemcpy(pl.roots, g.roots.data(), sizeof(int32_t) * g.roots.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemset(pl.cnt, 0, sizeof(unsigned) * n1));
  CUDA_TRY(cudaMemset(pl.queue, 0, sizeof(unsigned long long) * n1));
  CUDA_TRY(cudaMemset(pl.ctrl, 0, sizeof(int) * kCtrlWords));
  const int epoch1 = 1;   // launch epochs start at 1 (counters accumulate epoch x indegree)
  CUDA_TRY(cudaMemcpy(pl.ctrl + kCtrlEpoch, &epoch1, sizeof(int), cudaMemcpyHostToDevice));
  return 0;
}

// mode: 0 factor, 1 apply Q^T, 2 apply Q
static int get_plan(int mode, int p, int q, int qc, int nb, int ib, int tree, int bs, int family,
                    DevPlan **out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  int ws = pick_ws(nb, ib);
  if (ws > 32)   // the strip kernels deal 4 n8 column tiles (32 columns) over the warps
    return fail(TQR_EUNSUP, "strip width " + std::to_string(ws) + " (TQR_WS) > 32 is not supported");
  if (smem_bytes(nb, ib, ws) > kMaxSmem)
    return fail(TQR_EUNSUP, "strip width " + std::to_string(ws) + " (TQR_WS) needs " +
                                std::to_string(smem_bytes(nb, ib, ws)) + " bytes of shared memory for nb = " +
                                std::to_string(nb) + "; at most " + std::to_string(kMaxSmem) + " fit");
  PlanKey key{dev, mode, p, q, qc, nb, ib, tree, bs, family,
              (1 << 24) * (int)fuse_default() + 65536 * mstrip_default(q) + (ws * 4 + (env_int("TQR_SPLIT", 1) != 0) * 2 + (env_int("TQR_LOOKAHEAD", 1) != 0)) * 64 +
                  env_int("TQR_LEVELS", kLevels) + 4096 * env_int("TQR_PRIO", 0)};
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) { *out = it->second.get(); return 0; }
  std::vector<TileTask> tt;
  std::vector<int64_t> st, fin;
  int64_t mk;
  int rc = tile_sim(p, q, tree, bs, family, tt, st, fin, mk);
  if (rc < 0) return rc;
  DevGraph g;
  const bool split = env_int("TQR_SPLIT", 1) != 0 && ws == ib && nb > ib;
  if (mode == 0) build_factor_graph(tt, st, p, q, nb, ws, split, g, mstrip_default(q), fuse_default());
  else build_apply_graph(tt, p, qc, nb, ws, mode == 1, g);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  finalize_dataflow(g, env_int("TQR_LOOKAHEAD", 1) != 0, env_int("TQR_LEVELS", kLevels), env_int("TQR_PRIO", 0),
                    sms);
  auto pl = std::make_unique<DevPlan>();
  rc = upload(g, ws, *pl);
  if (rc < 0) return rc;
  *out = pl.get();
  g_plans[key] = std::move(pl);
  return 0;
}

// Host-only view of the device task graph (no GPU needed): the same builder
// get_plan uses. out_tasks: 8 int32 per task (kind, i, piv, k, j, s, chain,
// meta); succ_ptr[ntask+1], succ[...]. Returns ntask or TQR_E*.
extern "C" int64_t tqr_plan_graph(int m, int n, int nb, int ib, int tree, int bs, int family, int ws, int split,
                                  int32_t *out_tasks, int64_t task_cap, int32_t *succ_ptr, int32_t *succ,
                                  int64_t succ_cap) {
  int p, q;
  int rc = check_shape(m, n, nb, ib, p, q);
  if (rc < 0) return rc;
  if (ws <= 0) ws = pick_ws(nb, ib);
  std::vector<TileTask> tt;
  std::vector<int64_t> st, fin;
  int64_t mk;
  rc = tile_sim(p, q, tree, bs, family, tt, st, fin, mk);
  if (rc < 0) return rc;
  DevGraph g;
  const int ms = (split >> 8) > 0 ? (split >> 8) : mstrip_default(q);
  // split bit 1: fusion on, bit 2: fusion off, neither: the default (TQR_FUSE)
  const bool fuse = (split & 2) ? true : ((split & 4) ? false : fuse_default());
  build_factor_graph(tt, st, p, q, nb, ws, (split & 1) != 0 && ws == ib && nb > ib, g, ms, fuse);
  finalize_dataflow(g, true, kLevels, 0, 148);
  const int64_t nt = (int64_t)g.tasks.size();
  if (!out_tasks || !succ_ptr || !succ) return nt;          // size query
  if (task_cap < 8 * nt || succ_cap < (int64_t)g.succ.size()) return fail(TQR_ECAP, "tqr_plan_graph: capacity");
  for (int64_t t = 0; t < nt; ++t) {
    const DevTask &d = g.tasks[t];
    int32_t *o = out_tasks + 8 * t;
    o[0] = d.kind; o[1] = d.i; o[2] = d.piv; o[3] = d.k; o[4] = d.j; o[6] = d.chain; o[7] = d.meta;
    o[5] = d.s | ((d.pad > 1 ? d.pad : 1) << 16);   // strip | strip count << 16
    succ_ptr[t] = d.dep_begin;
  }
  succ_ptr[nt] = (int32_t)g.succ.size();
  std::copy(g.succ.begin(), g.succ.end(), succ);
  return nt;
}

extern "C" void tqr_release_plans(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_plans.clear();
  g_trace_plan = nullptr;
}

extern "C" int64_t tqr_trace_graph(int32_t *succ_ptr, int32_t *succ, int64_t cap) {
  DevPlan *pl = g_trace_plan;
  if (!pl) return fail(TQR_EINVAL, "tqr_trace_graph: no traced launch");
  int64_t ns = pl->host_tasks.empty() ? 0 : pl->host_tasks.back().dep_end;
  if (cap < ns || cap < (int64_t)pl->ntask + 1) return fail(TQR_ECAP, "tqr_trace_graph: capacity too small");
  for (int t = 0; t < pl->ntask; ++t) succ_ptr[t] = pl->host_tasks[t].dep_begin;
  succ_ptr[pl->ntask] = (int32_t)ns;
  if (ns) {
    std::vector<int32_t> edges(2 * ns);
    CUDA_TRY(cudaMemcpy(edges.data(), pl->succ, sizeof(int32_t) * 2 * ns, cudaMemcpyDeviceToHost));
    for (int64_t x = 0; x < ns; ++x) succ[x] = edges[2 * x];
  }
  return ns;
}

extern "C" int tqr_trace_enable(int on) {
  g_trace_on = on ? 1 : 0;
  return 0;
}

extern "C" int64_t tqr_trace_fetch(uint64_t *out, int64_t cap) {
  DevPlan *pl = g_trace_plan;
  if (!pl || !pl->trace) return fail(TQR_EINVAL, "tqr_trace_fetch: no traced launch");
  if (cap < (int64_t)pl->ntask * 16) return fail(TQR_ECAP, "tqr_trace_fetch: capacity < 16 * ntask");
  std::vector<uint64_t> raw((size_t)pl->ntask * kTraceWords);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(raw.data(), pl->trace, raw.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  for (int t = 0; t < pl->ntask; ++t) {
    const DevTask &d = pl->host_tasks[t];
    const uint64_t *r = raw.data() + (size_t)kTraceWords * t;
    uint64_t *o = out + 16 * (size_t)t;
    o[0] = r[0]; o[1] = r[1]; o[2] = r[2]; o[3] = r[3] >> 32;
    o[4] = (uint64_t)d.kind; o[5] = (uint64_t)d.i | ((uint64_t)(uint16_t)d.piv << 16);
    o[6] = (uint64_t)d.k | ((uint64_t)(uint16_t)d.j << 16); o[7] = (uint64_t)d.s;
    for (int x = 0; x < 8; ++x) o[8 + x] = r[4 + x];
  }
  return pl->ntask;
}

static int check_shape(int m, int n, int nb, int ib, int &p, int &q) {
  if (nb < 1 || ib < 1 || m < 1 || n < 1) return fail(TQR_EINVAL, "need m, n, nb, ib >= 1");
  if (nb > kMaxNb) return fail(TQR_EUNSUP, "nb > 256 is not supported");
  if (ib > kMaxIb) return fail(TQR_EUNSUP, "ib > 32 is not supported");
  if (m % nb || n % nb) return fail(TQR_EINVAL, "nb must divide m and n");
  p = m / nb; q = n / nb;
  if (q > p) return fail(TQR_EINVAL, "need m >= n");
  if (p > 32767 || q > 32767) return fail(TQR_EUNSUP, "too many tiles");
  return 0;
}

// ---- TMA tensor maps -----------------------------------------------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda
// link). A matrix of p x qc tiles of nb x nb (column-major tiles, tile (i, k)
// at column (k p + i) nb of the stacked columns) is viewed as the 3-D tensor
// (row within a tile of 8, stacked column, row tile), strides (8 B, 8 nb B,
// 64 B): a box of 8 x 32 x 4 is 4 row tiles of 32 columns in the row-tile
// shared-memory layout of the strip update (tqr_device.cuh).
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}
static bool encode_tiles8(CUtensorMap *m, const double *base, int nb, long long ncols) {
  PFN_cuTensorMapEncodeTiled_v12000 fn = tensor_map_encoder();
  if (!fn || !base) return false;
  const cuuint64_t dims[3] = {8, (cuuint64_t)ncols, (cuuint64_t)(nb / 8)};
  const cuuint64_t strides[2] = {(cuuint64_t)nb * 8, 64};
  const cuuint32_t box[3] = {8, 32, 4};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int g_tma_used = 0;
extern "C" int tqr_last_launch_tma(void) { return g_tma_used; }

static int launch(DevPlan *pl, int p, int q, int qc, int nb, int ib, double *A, double *T, double *C,
                  int trans, cudaStream_t stream) {
  if (pl->ntask == 0) { g_launches = 0; return 0; }
  int dev = 0, sms = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  size_t smem = smem_bytes(nb, ib, pl->ws);
  static thread_local int attr_set_dev = -1;
  if (attr_set_dev != dev) {
    int optin = 0;
    cudaFuncAttributes fa;
    CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    CUDA_TRY(cudaFuncGetAttributes(&fa, tqr_persistent));
    CUDA_TRY(cudaFuncSetAttribute(tqr_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - (int)fa.sharedSizeBytes));
    attr_set_dev = dev;
  }
  RunArgs a;
  memset(&a, 0, sizeof a);
  a.tasks = pl->tasks; a.succ = reinterpret_cast<const int2 *>(pl->succ); a.roots = pl->roots; a.nroots = pl->nroots; a.ntask = pl->ntask;
  a.cnt = pl->cnt; a.queue = pl->queue; a.ctrl = pl->ctrl;
  for (int l = 0; l <= kLevels; ++l) a.qoff[l] = pl->qoff[l];
  a.A = A; a.T = T; a.C = C;
  a.p = p; a.q = q; a.nb = nb; a.ib = ib; a.ws = pl->ws; a.trans = trans;
  // TMA tensor copies of V blocks and C1 windows when the shapes allow (row
  // tiles of 8 align with inner blocks, >= 4 row tiles); else cp.async
  a.tma = 0;
  if (env_int("TQR_TMA", 1) && nb % 8 == 0 && ib % 8 == 0 && nb >= 32 &&
      encode_tiles8(&a.mapA, A, nb, (long long)p * q * nb) &&
      (!C || encode_tiles8(&a.mapC, C, nb, (long long)p * qc * nb)))
    a.tma = 1;
  g_tma_used = a.tma;
  a.work_first = env_int("TQR_WORK_FIRST", 1) != 0;
  a.chain_spin = env_int("TQR_CHAIN_SPIN", 0);   // measured best: no spin (profiles/r01_chain_spin_sweep.txt)
  a.trace = nullptr;
  if (g_trace_on) {
    if (!pl->trace) CUDA_TRY(cudaMalloc(&pl->trace, sizeof(unsigned long long) * kTraceWords * pl->ntask));
    a.trace = pl->trace;
    g_trace_plan = pl;
  }
  int grid = sms;
  int forced = env_int("TQR_GRID", 0);
  if (forced > 0) grid = forced;
  // never more CTAs than can be co-resident (1 per SM at this footprint)
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tqr_persistent, kThreads, smem));
  if (per_sm < 1) return fail(TQR_EUNSUP, "tqr_persistent does not fit on an SM with " + std::to_string(smem) +
                                              " bytes of shared memory");
  if (grid > per_sm * sms) grid = per_sm * sms;
  if (grid > pl->ntask) grid = pl->ntask;
  a.nctas = grid;
  tqr_persistent<<<grid, kThreads, smem, stream>>>(a);
  CUDA_TRY(cudaGetLastError());
  g_launches = 1;
  return 0;
}

extern "C" int tiled_qr(int m, int n, int nb, int ib, int tree, int bs, int family, double *A,
                        double *T, void *stream) {
  int p, q;
  int rc = check_shape(m, n, nb, ib, p, q);
  if (rc < 0) return rc;
  if (!A || !T) return fail(TQR_EINVAL, "tiled_qr: null pointer");
  if (((uintptr_t)A | (uintptr_t)T) & 15) return fail(TQR_EINVAL, "tiled_qr: A and T must be 16-byte aligned");
  DevPlan *pl;
  rc = get_plan(0, p, q, 0, nb, ib, tree, bs, family, &pl);
  if (rc < 0) return rc;
  return launch(pl, p, q, 0, nb, ib, A, T, nullptr, 1, (cudaStream_t)stream);
}

static int apply_common(int trans, int m, int n, int nb, int ib, int tree, int bs, int family,
                        const double *A, const double *T, double *C, int nrhs, void *stream) {
  int p, q;
  int rc = check_shape(m, n, nb, ib, p, q);
  if (rc < 0) return rc;
  if (!A || !T || !C) return fail(TQR_EINVAL, "apply: null pointer");
  if (((uintptr_t)A | (uintptr_t)T | (uintptr_t)C) & 15)
    return fail(TQR_EINVAL, "apply: A, T and C must be 16-byte aligned");
  if (nrhs < 0 || nrhs % nb) return fail(TQR_EINVAL, "apply: nrhs must be a multiple of nb");
  int qc = nrhs / nb;
  if (qc == 0) { g_launches = 0; return 0; }
  DevPlan *pl;
  rc = get_plan(trans ? 1 : 2, p, q, qc, nb, ib, tree, bs, family, &pl);
  if (rc < 0) return rc;
  return launch(pl, p, q, qc, nb, ib, const_cast<double *>(A), const_cast<double *>(T), C, trans,
                (cudaStream_t)stream);
}

extern "C" int apply_qt(int m, int n, int nb, int ib, int tree, int bs, int family,
                        const double *A, const double *T, double *C, int nrhs, void *stream) {
  return apply_common(1, m, n, nb, ib, tree, bs, family, A, T, C, nrhs, stream);
}

extern "C" int apply_q(int m, int n, int nb, int ib, int tree, int bs, int family,
                       const double *A, const double *T, double *C, int nrhs, void *stream) {
  return apply_common(0, m, n, nb, ib, tree, bs, family, A, T, C, nrhs, stream);
}

// ---- end-to-end on host buffers ----------------------------------------------
struct Scratch { double *A = nullptr, *T = nullptr; size_t na = 0, nt = 0; int dev = -1; };
static std::mutex g_smu;
static Scratch g_scratch;

extern "C" int tiled_qr_host(int m, int n, int nb, int ib, int tree, int bs, int family,
                             double *A_host, double *T_host, void *stream) {
  int p, q;
  int rc = check_shape(m, n, nb, ib, p, q);
  if (rc < 0) return rc;
  if (!A_host || !T_host) return fail(TQR_EINVAL, "tiled_qr_host: null pointer");
  std::lock_guard<std::mutex> lk(g_smu);
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  size_t na = (size_t)m * n, nt = (size_t)p * q * 2 * ib * nb;
  if (g_scratch.dev != dev || g_scratch.na < na || g_scratch.nt < nt) {
    cudaFree(g_scratch.A); cudaFree(g_scratch.T);
    g_scratch = Scratch();
    CUDA_TRY(cudaMalloc(&g_scratch.A, na * sizeof(double)));
    CUDA_TRY(cudaMalloc(&g_scratch.T, nt * sizeof(double)));
    g_scratch.na = na; g_scratch.nt = nt; g_scratch.dev = dev;
  }
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(g_scratch.A, A_host, na * sizeof(double), cudaMemcpyHostToDevice, s));
  rc = tiled_qr(m, n, nb, ib, tree, bs, family, g_scratch.A, g_scratch.T, stream);
  if (rc < 0) return rc;
  CUDA_TRY(cudaMemcpyAsync(A_host, g_scratch.A, na * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(T_host, g_scratch.T, nt * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return 0;
}

// ---- pipelined end-to-end calls (two device slots, dedicated copy streams) ----
// Call k uses slot k % 2: H2D on the upload stream (after the slot's previous
// download finished), the factorization on the caller's stream (after the
// upload), the download of A and T on the download stream (after the
// factorization). Consecutive calls therefore overlap their copies with the
// neighbours' compute. tqr_host_wait() waits for everything issued.
struct AsyncPipe {
  int dev = -1;
  size_t na = 0, nt = 0;
  double *A[2] = {nullptr, nullptr}, *T[2] = {nullptr, nullptr};
  cudaStream_t up = nullptr, down = nullptr;
  cudaEvent_t uploaded[2], computed[2], downloaded[2];
  unsigned long long calls = 0;
};
static std::mutex g_pmu;
static AsyncPipe g_pipe;

static int pipe_init(AsyncPipe &P, int dev, size_t na, size_t nt) {
  if (P.dev == dev && P.na >= na && P.nt >= nt) return 0;
  if (P.dev >= 0) {
    cudaStreamSynchronize(P.down);
    for (int k = 0; k < 2; ++k) { cudaFree(P.A[k]); cudaFree(P.T[k]); }
  } else {
    CUDA_TRY(cudaStreamCreateWithFlags(&P.up, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&P.down, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      CUDA_TRY(cudaEventCreateWithFlags(&P.uploaded[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&P.computed[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&P.downloaded[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(P.downloaded[k], P.down));
    }
  }
  for (int k = 0; k < 2; ++k) {
    CUDA_TRY(cudaMalloc(&P.A[k], na * sizeof(double)));
    CUDA_TRY(cudaMalloc(&P.T[k], nt * sizeof(double)));
  }
  P.dev = dev; P.na = na; P.nt = nt;
  return 0;
}

extern "C" int tiled_qr_host_async(int m, int n, int nb, int ib, int tree, int bs, int family,
                                   const double *A_host, double *R_host, double *T_host, void *stream) {
  int p, q;
  int rc = check_shape(m, n, nb, ib, p, q);
  if (rc < 0) return rc;
  if (!A_host || !R_host || !T_host) return fail(TQR_EINVAL, "tiled_qr_host_async: null pointer");
  std::lock_guard<std::mutex> lk(g_pmu);
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  const size_t na = (size_t)m * n, nt = (size_t)p * q * 2 * ib * nb;
  rc = pipe_init(g_pipe, dev, na, nt);
  if (rc < 0) return rc;
  AsyncPipe &P = g_pipe;
  const int k = (int)(P.calls++ & 1);
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaStreamWaitEvent(P.up, P.downloaded[k], 0));
  CUDA_TRY(cudaMemcpyAsync(P.A[k], A_host, na * sizeof(double), cudaMemcpyHostToDevice, P.up));
  CUDA_TRY(cudaEventRecord(P.uploaded[k], P.up));
  CUDA_TRY(cudaStreamWaitEvent(s, P.uploaded[k], 0));
  rc = tiled_qr(m, n, nb, ib, tree, bs, family, P.A[k], P.T[k], stream);
  if (rc < 0) return rc;
  CUDA_TRY(cudaEventRecord(P.computed[k], s));
  CUDA_TRY(cudaStreamWaitEvent(P.down, P.computed[k], 0));
  CUDA_TRY(cudaMemcpyAsync(R_host, P.A[k], na * sizeof(double), cudaMemcpyDeviceToHost, P.down));
  CUDA_TRY(cudaMemcpyAsync(T_host, P.T[k], nt * sizeof(double), cudaMemcpyDeviceToHost, P.down));
  CUDA_TRY(cudaEventRecord(P.downloaded[k], P.down));
  return 0;
}

extern "C" int tqr_host_wait(void) {
  std::lock_guard<std::mutex> lk(g_pmu);
  if (g_pipe.dev >= 0) {
    CUDA_TRY(cudaStreamSynchronize(g_pipe.up));
    CUDA_TRY(cudaStreamSynchronize(g_pipe.down));
  }
  return 0;
}
