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
  K_AP_UNMQR = 6, K_AP_TTMQR = 7, K_AP_TSMQR = 8
};

int kind_weight(int kind);   // Table 1 weights in units of nb^3/3

// Elimination lists of every tree (trees.cpp). Returns false on bad args.
bool build_elim_list(int p, int q, int tree, int bs, std::vector<Elim> &out, std::string &err);

// Tile-level task of the expanded DAG (Algorithms 2-3); 1-based indices.
struct TileTask {
  int kind, i, piv, k, j;          // j = updated column (updates only), else 0
  std::vector<int> deps;           // indices of predecessor TileTasks
};

// Expansion of an elimination list into kernel tasks (dag.cpp), in emission order.
void expand(const std::vector<Elim> &lst, int p, int q, int family, std::vector<TileTask> &tasks);

// Discrete-event simulation with unbounded processors; returns makespan.
int64_t simulate(const std::vector<TileTask> &tasks, std::vector<int64_t> &start,
                 std::vector<int64_t> &finish);

// Device task (16 bytes + dependency range). Shared layout with tiledqr.cu.
struct DevTask {
  int16_t kind, i, piv, k, j, s;   // 0-based tile indices; s = column strip
  int32_t dep_begin, dep_end;      // range in the dependency array
  int32_t pad;
};
static_assert(sizeof(DevTask) == 24, "DevTask layout");

struct DevGraph {
  std::vector<DevTask> tasks;      // in execution priority order (topological)
  std::vector<int32_t> deps;       // predecessor task ids (positions in `tasks`)
};

// Strip-refined factorization graph: every update task is split into
// ceil(nb/ws) column strips of width ws.
void build_factor_graph(const std::vector<TileTask> &tt, const std::vector<int64_t> &start,
                        int p, int q, int nb, int ws, DevGraph &g);

// Apply graph for C (p x qc tiles): Q^T (trans=1) or Q (trans=0).
void build_apply_graph(const std::vector<TileTask> &tt, int p, int qc, int nb, int ws,
                       bool trans, DevGraph &g);

}  // namespace tqr
