// Internal host-side structures of the tiled QR plan (not part of the C ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace tqr {

struct Elim {            // elim(i, piv, k), 1-based (Algorithm 1)
  int i, piv, k, step;   // step = coarse-grain time-step (Table 2)
};

// Kernel kinds (Table 1). Values are shared with the device code.
enum Kind : int {
  K_GEQRT = 0, K_UNMQR = 1, K_TTQRT = 2, K_TTMQR = 3, K_TSQRT = 4, K_TSMQR = 5,
  // apply-only kinds (apply_qt / apply_q on a right-hand side C)
  K_AP_UNMQR = 6, K_AP_TTMQR = 7, K_AP_TSMQR = 8,
  // split panel kinds: one inner block b of a panel kernel (s = b), and the
  // update of strip s of the same tile(s) by block b (j = b)
  K_GEQRT_B = 9, K_GEQRT_U = 10, K_TTQRT_B = 11, K_TTQRT_U = 12, K_TSQRT_B = 13, K_TSQRT_U = 14,
  // factorization only: UNMQR(i, k, j) fused with the TTMQR(i, piv, k, j) that
  // follows it on tile (i, j) (TT family; one task, the strip stays in registers)
  K_UNTTMQR = 15
};

int kind_weight(int kind);   // Table 1 weights in units of nb^3/3

// Elimination lists of every tree (trees.cpp). Returns false on bad args.
bool build_elim_list(int p, int q, int tree, int bs, std::vector<Elim> &out, std::string &err);

// ASAP (k_asap = q) / Grasap(k_asap) eliminations, decided by the tiled
// discrete-event execution (dag.cpp).
void grasap_elims(int p, int q, int k_asap, std::vector<Elim> &out);

// Tile-level task of the expanded DAG (Algorithms 2-3); 1-based indices.
struct TileTask {
  int kind, i, piv, k, j;          // j = updated column (updates only), else 0
  std::vector<int> deps;           // indices of predecessor TileTasks
};

// Expansion of an elimination list into kernel tasks (dag.cpp), in emission order.
// merge_input: the matrix is [R1; R2] (p = 2q) whose diagonal tiles are
// already triangles and whose lower tiles are structurally zero.
void expand(const std::vector<Elim> &lst, int p, int q, int family, std::vector<TileTask> &tasks,
            bool merge_input = false);

// Discrete-event simulation with unbounded processors; returns makespan.
int64_t simulate(const std::vector<TileTask> &tasks, std::vector<int64_t> &start,
                 std::vector<int64_t> &finish);

// Device task record. Shared layout with tiledqr.cu / tqr_device.cuh.
// Before finalize_dataflow: [dep_begin, dep_end) indexes DevGraph::deps.
// After: [dep_begin, dep_end) indexes DevGraph::succ (successors) and
// meta = indegree | (priority class << 16).
// chain = a successor the same CTA runs next when it is ready (panel chain of
// split panels: P(b) -> U(b,b+1) -> P(b+1)), -1 if none.
struct DevTask {
  int16_t kind, i, piv, k, j, s;   // 0-based tile indices; s = column strip
  int32_t dep_begin, dep_end;
  int32_t meta;
  int32_t chain;
  int32_t pad;                     // update tasks of other tiles: number of strips (>= 1), else 0
};
static_assert(sizeof(DevTask) == 32, "DevTask layout");

struct DevGraph {
  std::vector<DevTask> tasks;      // in priority order (topological)
  std::vector<int32_t> deps;       // predecessor task ids (positions in `tasks`)
  std::vector<int32_t> succ;       // successor task ids (after finalize_dataflow)
  std::vector<int32_t> roots;      // tasks without predecessors, in priority order
};

// Convert the predecessor lists into successor lists, indegrees and the
// priority level of every task (meta bits 16-19, up to kLevels levels from the
// task's estimated bottom level: longest path to the end of the graph);
// chain targets get meta bit 20 (one virtual extra dependency held by the
// chain owner). prioritize = false puts every task on level 0 (FIFO).
constexpr int kLevels = 16;
void finalize_dataflow(DevGraph &g, bool prioritize = true, int levels = kLevels, int prio_rule = 0,
                       int nproc = 148);

// Strip-refined factorization graph: every update task is split into
// ceil(nb/ws) column strips of width ws; with split_panels (requires ws == ib)
// every panel kernel becomes per-inner-block panel tasks plus trailing strip
// tasks.
// Update tasks of other tiles (UNMQR / TTMQR / TSMQR) cover mstrip consecutive
// strips each (DevTask::pad = their count), run one after another by one CTA.
// fuse: UNMQR + TTMQR pairs on the same tile become K_UNTTMQR tasks.
void build_factor_graph(const std::vector<TileTask> &tt, const std::vector<int64_t> &start,
                        int p, int q, int nb, int ws, bool split_panels, DevGraph &g, int mstrip = 1,
                        bool fuse = false);

// Apply graph for C (p x qc tiles): Q^T (trans=1) or Q (trans=0).
void build_apply_graph(const std::vector<TileTask> &tt, int p, int qc, int nb, int ws,
                       bool trans, DevGraph &g);

}  // namespace tqr
