// Elimination lists of the tiled QR trees (product code; independent of oracle/).
//
// PAPER.md §3.1 "Coarse-grain algorithms" (lines 478-512) and §3.2 "Tiled
// algorithms" (lines 652-956). Indices are 1-based as in the paper.
#include <algorithm>
#include <cstdio>
#include <tuple>
#include "plan.h"

namespace tqr {

namespace {

// ---- Sameh-Kuck / FlatTree (line 488): elim(i,k,k), i = k+1..p; coarse(i,k) = i+k-2.
void flat(int p, int q, std::vector<Elim> &out) {
  int kmax = std::min(p, q);
  for (int k = 1; k <= kmax; ++k)
    for (int i = k + 1; i <= p; ++i) out.push_back({i, k, k, i + k - 2});
}

// ---- Fibonacci scheme of order 1 (lines 490-505).
// Column 1: x = least integer with x(x+1)/2 >= p-1; the rows are cut, from the
// top, into groups of sizes 1, 2, 3, ... (y-th group: rows y(y-1)/2+2 ..
// y(y+1)/2+1); group y is zeroed at step x-y+1. Column k repeats column 1's
// pattern shifted down k-1 rows and 2(k-1) steps later. A group of z
// consecutive rows a..a+z-1 zeroed at one step uses the z rows right above it.
void fibonacci(int p, int q, std::vector<Elim> &out) {
  int x = 0;
  while ((int64_t)x * (x + 1) / 2 < p - 1) ++x;
  int kmax = std::min(p, q);
  for (int k = 1; k <= kmax; ++k) {
    // rows k+1..p; relative row u = i-k+1 in 2..p-k+1
    for (int y = 1;; ++y) {
      int lo = y * (y - 1) / 2 + 2 + (k - 1);      // first row of group y in column k
      if (lo > p) break;
      int hi = std::min(y * (y + 1) / 2 + 1 + (k - 1), p);
      int z = hi - lo + 1;
      int step = x - y + 1 + 2 * (k - 1);
      for (int r = lo; r <= hi; ++r) out.push_back({r, r - z, k, step});
    }
  }
}

// ---- Greedy (lines 507-512): at every step, in every column, zero as many
// tiles as possible, bottom rows first, pairing as Fibonacci. Counters as in
// Algorithm 4 (lines 563-619): nZ[k] = tiles zeroed in column k so far; they
// are always the bottom nZ[k] rows. A row is ready for column k once its tile
// in column k-1 is zeroed (validity condition, lines 362-366), so the rows
// available in column k are p-nZ[k-1]+1 .. p-nZ[k] (k >= 2) or 1 .. p-nZ[1].
void greedy(int p, int q, std::vector<Elim> &out) {
  int kmax = std::min(p, q);
  std::vector<int> nz(kmax + 1, 0), nznew(kmax + 1, 0);
  int left = 0;
  for (int k = 1; k <= kmax; ++k) left += p - k;
  for (int s = 1; left > 0; ++s) {
    for (int k = 1; k <= kmax; ++k) {
      int top = (k == 1) ? 1 : p - nz[k - 1] + 1;     // first available row
      int bot = p - nz[k];                             // last available row
      int avail = bot - top + 1;
      int z = avail > 0 ? avail / 2 : 0;
      nznew[k] = nz[k] + z;
      for (int r = bot - z + 1; r <= bot; ++r) out.push_back({r, r - z, k, s});
      left -= z;
    }
    nz = nznew;
  }
}

int lowbit(int d) { return d & (-d); }
int bitlen(int v) { int b = 0; while (v) { ++b; v >>= 1; } return b; }

// ---- BinaryTree (lines 914-918): in column k, round r pairs the survivors at
// distance 2^(r-1); the upper row survives. Relative index d = i-k.
void binary(int p, int q, std::vector<Elim> &out) {
  int kmax = std::min(p, q);
  for (int k = 1; k <= kmax; ++k) {
    std::vector<std::tuple<int, int, int>> col;   // (round, i, piv)
    for (int i = k + 1; i <= p; ++i) {
      int lb = lowbit(i - k);
      col.emplace_back(bitlen(lb), i, i - lb);
    }
    std::sort(col.begin(), col.end());
    for (auto &t : col) out.push_back({std::get<1>(t), std::get<2>(t), k, 0});
  }
}

// ---- PlasmaTree(BS) (lines 936-953): domains of BS consecutive rows starting
// at the diagonal row k (so the bottom domain shrinks as k grows); FlatTree
// inside each domain with its first row as local panel; then the domain heads
// are merged by a binary tree (reading R4).
void plasma(int p, int q, int bs, std::vector<Elim> &out) {
  int kmax = std::min(p, q);
  for (int k = 1; k <= kmax; ++k) {
    std::vector<int> heads;
    for (int h = k; h <= p; h += bs) heads.push_back(h);
    // phase 0: flat eliminations inside the domains, by row
    for (int i = k + 1; i <= p; ++i) {
      int h = k + ((i - k) / bs) * bs;
      if (h != i) out.push_back({i, h, k, 0});
    }
    // phase 1: binary merge of the heads
    std::vector<std::tuple<int, int, int>> merge;
    for (int d = 1; d < (int)heads.size(); ++d) {
      int lb = lowbit(d);
      merge.emplace_back(bitlen(lb), heads[d], heads[d - lb]);
    }
    std::sort(merge.begin(), merge.end());
    for (auto &t : merge) out.push_back({std::get<1>(t), std::get<2>(t), k, 0});
  }
}

// Coarse ASAP time-steps of a list (one elimination = one step; an
// elimination waits for the previous eliminations of both its rows; lines
// 466-471). Used for BinaryTree / PlasmaTree (reading R5).
void coarse_asap(int p, std::vector<Elim> &lst) {
  std::vector<int> last(p + 1, 0);
  for (auto &e : lst) {
    int s = 1 + std::max(last[e.i], last[e.piv]);
    e.step = s;
    last[e.i] = last[e.piv] = s;
  }
}

// ---- Merge of two stacked tile-upper-triangular R factors [R1; R2] (2q x q
// tiles): column k zeroes the bottom tiles (q+t, k), t = 1..k,
// against the top pivot row k (flat within the merge). Bottom row q+t has
// structural zeros left of column t, so it is ready for column k once it was
// eliminated in columns t..k-1 (validity conditions, lines 362-369).
void merge(int q, std::vector<Elim> &out) {
  for (int k = 1; k <= q; ++k)
    for (int t = 1; t <= k; ++t) out.push_back({q + t, k, k, 0});
}

}  // namespace

bool build_elim_list(int p, int q, int tree, int bs, std::vector<Elim> &out, std::string &err) {
  out.clear();
  if (p < 1 || q < 1 || q > p) { err = "elim_list: need p >= q >= 1"; return false; }
  switch (tree) {
    case 0: flat(p, q, out); break;
    case 1: fibonacci(p, q, out); break;
    case 2: greedy(p, q, out); break;
    case 3: binary(p, q, out); coarse_asap(p, out); break;
    case 4:
      if (bs < 1 || bs > p) { err = "elim_list: PlasmaTree needs 1 <= bs <= p"; return false; }
      plasma(p, q, bs, out); coarse_asap(p, out); break;
    case 5:
      if (p != 2 * q) { err = "elim_list: the merge scheme needs p = 2q"; return false; }
      merge(q, out); coarse_asap(p, out); break;
    case 6:
      grasap_elims(p, q, q, out); coarse_asap(p, out); break;
    case 7:
      if (bs < 0 || bs > q) { err = "elim_list: Grasap(k) needs 0 <= k <= q (passed as bs)"; return false; }
      grasap_elims(p, q, bs, out); coarse_asap(p, out); break;
    default: err = "elim_list: unknown tree"; return false;
  }
  if (tree == 1 || tree == 2) {
    // list order (R2): (coarse step, k, i)
    std::stable_sort(out.begin(), out.end(), [](const Elim &a, const Elim &b) {
      return std::tie(a.step, a.k, a.i) < std::tie(b.step, b.k, b.i);
    });
  }
  return true;
}

int kind_weight(int kind) {
  switch (kind) {
    case K_GEQRT: return 4;
    case K_UNMQR: return 6;
    case K_TSQRT: return 6;
    case K_TSMQR: return 12;
    case K_TTQRT: return 2;
    case K_TTMQR: return 6;
    default: return 0;
  }
}

}  // namespace tqr
