// Kernel-task DAG of a tiled QR elimination list, its discrete-event critical
// path, and the strip-refined device task graphs (product code; independent of
// oracle/).
//
// Expansion (§2.1): TT family = Algorithm 3 (lines 289-307), TS
// family = Algorithm 2 (lines 254-268); "if a tile is already in triangle form,
// then the associated GEQRT and update kernels are not applied" (lines 333-335);
// a TS elimination of a tile that already is a triangle (it was a pivot earlier
// in the column) uses TTQRT/TTMQR (reading R6); finally every
// diagonal tile not yet a triangle is factored by GEQRT (the square case of
// Theorem 1(1)).
// Dependencies (execution scheme §2.3, with the NODEP relaxation
// of §4): successive writers of a tile are chained; an update
// waits for the panel kernel whose reflectors it applies; reading reflectors
// does not block a later writer (the reflectors and the rewritten part of the
// tile are disjoint).
#include <algorithm>
#include <map>
#include <numeric>
#include <queue>
#include "plan.h"

namespace tqr {

// ---- ASAP / Grasap(k) (§3.2) -----------------------
// ASAP decides its eliminations during the tiled execution: at every instant,
// in every column, with r rows ready (tile a triangle, not inside a running
// TTQRT), s = r/2 eliminations start, the bottom s ready rows zeroed by the s
// ready rows right above them. Grasap(k) runs Greedy's list on the first q-k
// columns, then ASAP. The execution model is the TT expansion + unbounded
// processors of expand/simulate, tracked incrementally here through the finish
// time of every tile's last writer (reading R11).
void grasap_elims(int p, int q, int k_asap, std::vector<Elim> &out) {
  out.clear();
  const int kmax = std::min(p, q);
  std::vector<int64_t> lastfin((size_t)(p + 1) * (q + 1), 0);
  std::vector<char> tri((size_t)(p + 1) * (q + 1), 0);
  auto at = [q](int r, int c) { return (size_t)r * (q + 1) + c; };
  auto emit = [&](int weight, int64_t readfin, int r1, int c1, int r2, int c2) {
    int64_t st = std::max(readfin, lastfin[at(r1, c1)]);
    if (r2 >= 0) st = std::max(st, lastfin[at(r2, c2)]);
    const int64_t fin = st + weight;
    lastfin[at(r1, c1)] = fin;
    if (r2 >= 0) lastfin[at(r2, c2)] = fin;
    return fin;
  };
  auto factor = [&](int r, int k) {
    const int64_t g = emit(kind_weight(K_GEQRT), 0, r, k, -1, 0);
    for (int j = k + 1; j <= q; ++j) emit(kind_weight(K_UNMQR), g, r, j, -1, 0);
    tri[at(r, k)] = 1;
    return g;
  };
  auto eliminate = [&](int i, int piv, int k) {
    if (!tri[at(piv, k)]) factor(piv, k);
    if (!tri[at(i, k)]) factor(i, k);
    const int64_t x = emit(kind_weight(K_TTQRT), 0, piv, k, i, k);
    for (int j = k + 1; j <= q; ++j) emit(kind_weight(K_TTMQR), x, piv, j, i, j);
    out.push_back({i, piv, k, 0});
    return x;
  };
  const int first = q - k_asap + 1;        // first ASAP column
  if (first > 1) {
    std::vector<Elim> gl;
    std::string err;
    build_elim_list(p, q, 2, 1, gl, err);
    for (const Elim &e : gl)
      if (e.k < first) eliminate(e.i, e.piv, e.k);
  }
  if (first > kmax) return;
  // ready[k][r] = time row r is ready in column k (-1 = not ready / done)
  std::vector<std::vector<int64_t>> ready(kmax + 2, std::vector<int64_t>(p + 1, -1));
  std::vector<int> left(kmax + 2, 0);      // rows still to zero in each ASAP column
  for (int k = first; k <= kmax; ++k) left[k] = p - k;
  std::vector<char> zeroed_prev((size_t)p + 1, 0);
  for (const Elim &e : out)
    if (e.k == first - 1) zeroed_prev[e.i] = 1;
  for (int r = first; r <= p; ++r)
    if (first == 1 || zeroed_prev[r]) ready[first][r] = factor(r, first);
  int64_t t = 0;
  for (;;) {
    // next instant with a ready row
    int64_t tn = -1;
    for (int k = first; k <= kmax; ++k)
      for (int r = k; r <= p; ++r)
        if (ready[k][r] >= t && (tn < 0 || ready[k][r] < tn)) tn = ready[k][r];
    if (tn < 0) break;
    t = tn;
    for (int k = first; k <= kmax; ++k) {
      if (left[k] == 0) continue;
      std::vector<int> rows;
      for (int r = k; r <= p; ++r)
        if (ready[k][r] >= 0 && ready[k][r] <= t) rows.push_back(r);
      const int nrow = (int)rows.size(), s = nrow / 2;
      for (int x = 0; x < s; ++x) {
        const int i = rows[nrow - s + x], pv = rows[nrow - 2 * s + x];
        const int64_t done = eliminate(i, pv, k);
        ready[k][i] = -1;
        ready[k][pv] = done;
        --left[k];
        if (k + 1 <= kmax) ready[k + 1][i] = factor(i, k + 1);
      }
      if (left[k] == 0) std::fill(ready[k].begin(), ready[k].end(), -1);
    }
    ++t;      // every later event is at a strictly larger integer time
  }
}

void expand(const std::vector<Elim> &lst, int p, int q, int family, std::vector<TileTask> &tasks,
            bool merge_input) {
  tasks.clear();
  const int kmax = std::min(p, q);
  std::vector<int> last((size_t)(p + 1) * (q + 1), -1);   // last writer per tile (1-based)
  std::vector<char> tri((size_t)(p + 1) * (q + 1), 0);
  std::vector<int> geqrt_of((size_t)(p + 1) * (q + 1), -1);
  auto at = [q](int r, int c) { return (size_t)r * (q + 1) + c; };
  if (merge_input)    // [R1; R2]: both diagonals of tiles are already triangles
    for (int k = 1; k <= q; ++k) tri[at(k, k)] = tri[at(q + k, k)] = 1;

  auto emit = [&](int kind, int i, int piv, int k, int j, int reads, std::initializer_list<std::pair<int, int>> writes) {
    TileTask t{kind, i, piv, k, j, {}};
    if (reads >= 0) t.deps.push_back(reads);
    for (auto &w : writes) {
      int lw = last[at(w.first, w.second)];
      if (lw >= 0) t.deps.push_back(lw);
    }
    std::sort(t.deps.begin(), t.deps.end());
    t.deps.erase(std::unique(t.deps.begin(), t.deps.end()), t.deps.end());
    int id = (int)tasks.size();
    for (auto &w : writes) last[at(w.first, w.second)] = id;
    tasks.push_back(std::move(t));
    return id;
  };
  auto factor = [&](int r, int k) {
    int g = emit(K_GEQRT, r, 0, k, 0, -1, {{r, k}});
    geqrt_of[at(r, k)] = g;
    for (int j = k + 1; j <= q; ++j) emit(K_UNMQR, r, 0, k, j, g, {{r, j}});
    tri[at(r, k)] = 1;
  };
  for (const Elim &e : lst) {
    const int i = e.i, pv = e.piv, k = e.k;
    if (!tri[at(pv, k)]) factor(pv, k);
    int qrt, mqr;
    if (family == 0 || tri[at(i, k)]) {
      if (!tri[at(i, k)]) factor(i, k);
      qrt = K_TTQRT; mqr = K_TTMQR;
    } else {
      qrt = K_TSQRT; mqr = K_TSMQR;
    }
    int x = emit(qrt, i, pv, k, 0, -1, {{pv, k}, {i, k}});
    for (int j = k + 1; j <= q; ++j) emit(mqr, i, pv, k, j, x, {{pv, j}, {i, j}});
  }
  for (int k = 1; k <= kmax; ++k)
    if (!tri[at(k, k)]) factor(k, k);
}

int64_t simulate(const std::vector<TileTask> &tasks, std::vector<int64_t> &start,
                 std::vector<int64_t> &finish) {
  start.assign(tasks.size(), 0);
  finish.assign(tasks.size(), 0);
  int64_t mk = 0;
  for (size_t t = 0; t < tasks.size(); ++t) {
    int64_t s = 0;
    for (int d : tasks[t].deps) s = std::max(s, finish[d]);
    start[t] = s;
    finish[t] = s + kind_weight(tasks[t].kind);
    mk = std::max(mk, finish[t]);
  }
  return mk;
}

namespace {

// Reorder a graph built in a topological emission order by a priority key
// that is itself topological (key(dep) < key(task)), then remap dependencies.
void reorder(DevGraph &g, const std::vector<std::pair<int64_t, int64_t>> &key,
             const std::vector<std::vector<int>> &deps) {
  const int n = (int)g.tasks.size();
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return key[a] < key[b]; });
  std::vector<int> pos(n);
  for (int r = 0; r < n; ++r) pos[ord[r]] = r;
  std::vector<DevTask> out(n);
  g.deps.clear();
  for (int r = 0; r < n; ++r) {
    DevTask t = g.tasks[ord[r]];
    if (t.chain >= 0) t.chain = pos[t.chain];
    t.dep_begin = (int32_t)g.deps.size();
    for (int d : deps[ord[r]]) g.deps.push_back(pos[d]);
    t.dep_end = (int32_t)g.deps.size();
    out[r] = t;
  }
  g.tasks.swap(out);
}

DevTask mk(int kind, int i, int piv, int k, int j, int s) {
  DevTask t;
  t.kind = (int16_t)kind; t.i = (int16_t)i; t.piv = (int16_t)piv; t.k = (int16_t)k;
  t.j = (int16_t)j; t.s = (int16_t)s; t.dep_begin = t.dep_end = 0; t.meta = 0; t.chain = -1; t.pad = 0;
  return t;
}

}  // namespace

void build_factor_graph(const std::vector<TileTask> &tt, const std::vector<int64_t> &start,
                        int p, int q, int nb, int ws, bool split_panels, DevGraph &g, int mstrip, bool fuse) {
  if (mstrip < 1) mstrip = 1;
  // Fusion (TT family): an UNMQR(i, k, j) whose next task on tile (i, j) (in
  // emission order, i.e. its only successor on that tile) is the
  // TTMQR(i, piv, k, j) eliminating the same row is not emitted; the TTMQR's
  // device tasks become K_UNTTMQR tasks that run both on each strip. Nothing
  // else touches tile (i, j) in between, so the strip's history is unchanged.
  std::vector<int> fused_from(tt.size(), -1);
  if (fuse) {
    std::map<std::pair<int, int>, int> last;   // tile -> last tile task touching it
    auto touch = [&](int r, int c, int x) {
      auto it = last.find({r, c});
      if (it != last.end()) {
        const TileTask &u = tt[it->second], &y = tt[x];
        if (u.kind == K_UNMQR && y.kind == K_TTMQR && y.i == u.i && y.k == u.k && y.j == u.j && r == y.i)
          fused_from[x] = it->second;
      }
      last[{r, c}] = x;
    };
    for (size_t x = 0; x < tt.size(); ++x) {
      const TileTask &t = tt[x];
      switch (t.kind) {
        case K_GEQRT: touch(t.i, t.k, (int)x); break;
        case K_UNMQR: touch(t.i, t.j, (int)x); break;
        case K_TTQRT: case K_TSQRT: touch(t.i, t.k, (int)x); touch(t.piv, t.k, (int)x); break;
        case K_TTMQR: case K_TSMQR: touch(t.i, t.j, (int)x); touch(t.piv, t.j, (int)x); break;
        default: break;
      }
    }
  }
  std::vector<char> skip(tt.size(), 0);
  for (size_t x = 0; x < tt.size(); ++x)
    if (fused_from[x] >= 0) skip[fused_from[x]] = 1;
  const int S = (nb + ws - 1) / ws;
  g.tasks.clear();
  std::vector<std::vector<int>> deps;
  std::vector<std::pair<int64_t, int64_t>> key;
  // last device writer of every (tile, strip); tiles 0-based
  std::vector<int> lw((size_t)p * q * S, -1);
  auto slot = [p, S](int r, int c, int s) { return ((size_t)c * p + r) * S + s; };
  // device tasks holding the reflectors (V, T) of each panel tile task
  std::vector<std::vector<int>> panel_dev(tt.size());
  std::vector<int> dl;
  auto add = [&](DevTask t, std::vector<int> &d, int64_t prio) {
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    g.tasks.push_back(t);
    deps.push_back(d);
    key.emplace_back(prio, (int64_t)g.tasks.size());
    return (int)g.tasks.size() - 1;
  };
  auto push_lw = [&](int r, int c, int s) { if (lw[slot(r, c, s)] >= 0) dl.push_back(lw[slot(r, c, s)]); };
  for (size_t x = 0; x < tt.size(); ++x) {
    const TileTask &t = tt[x];
    const int i = t.i - 1, pv = t.piv - 1, k = t.k - 1, j = t.j - 1;
    switch (t.kind) {
      case K_GEQRT: {
        if (!split_panels) {
          dl.clear();
          for (int s = 0; s < S; ++s) push_lw(i, k, s);
          int id = add(mk(K_GEQRT, i, 0, k, 0, 0), dl, start[x]);
          for (int s = 0; s < S; ++s) lw[slot(i, k, s)] = id;
          panel_dev[x].push_back(id);
          break;
        }
        // left-looking emission: for each strip s, the updates by blocks < s, then its panel
        std::vector<int> P(S, -1);
        for (int s = 0; s < S; ++s) {
          for (int b = 0; b < s; ++b) {
            dl.clear();
            dl.push_back(P[b]);
            push_lw(i, k, s);
            const int u = add(mk(K_GEQRT_U, i, 0, k, b, s), dl, start[x]);
            lw[slot(i, k, s)] = u;
            if (b == s - 1) g.tasks[P[b]].chain = u;          // P(b) -> U(b, b+1)
          }
          dl.clear();
          push_lw(i, k, s);
          P[s] = add(mk(K_GEQRT_B, i, 0, k, 0, s), dl, start[x]);
          if (s > 0) g.tasks[lw[slot(i, k, s)]].chain = P[s];  // U(s-1, s) -> P(s)
          lw[slot(i, k, s)] = P[s];
        }
        panel_dev[x] = P;
        break;
      }
      case K_TTQRT: case K_TSQRT: {
        if (!split_panels) {
          dl.clear();
          for (int s = 0; s < S; ++s) { push_lw(pv, k, s); push_lw(i, k, s); }
          int id = add(mk(t.kind, i, pv, k, 0, 0), dl, start[x]);
          for (int s = 0; s < S; ++s) lw[slot(pv, k, s)] = lw[slot(i, k, s)] = id;
          panel_dev[x].push_back(id);
          break;
        }
        const int kb = t.kind == K_TTQRT ? K_TTQRT_B : K_TSQRT_B;
        const int ku = t.kind == K_TTQRT ? K_TTQRT_U : K_TSQRT_U;
        std::vector<int> P(S, -1);
        for (int s = 0; s < S; ++s) {
          for (int b = 0; b < s; ++b) {
            dl.clear();
            dl.push_back(P[b]);
            push_lw(pv, k, s);
            push_lw(i, k, s);
            int id = add(mk(ku, i, pv, k, b, s), dl, start[x]);
            lw[slot(pv, k, s)] = lw[slot(i, k, s)] = id;
            if (b == s - 1) g.tasks[P[b]].chain = id;         // P(b) -> U(b, b+1)
          }
          dl.clear();
          push_lw(pv, k, s);
          push_lw(i, k, s);
          P[s] = add(mk(kb, i, pv, k, 0, s), dl, start[x]);
          if (s > 0) g.tasks[lw[slot(i, k, s)]].chain = P[s];  // U(s-1, s) -> P(s)
          lw[slot(pv, k, s)] = lw[slot(i, k, s)] = P[s];
        }
        panel_dev[x] = P;
        break;
      }
      case K_UNMQR: {
        if (skip[x]) break;   // runs inside the fused task of its TTMQR
        // the reflector source is the GEQRT of tile (i,k): the unique dep with kind GEQRT on (i,k)
        const std::vector<int> *src = nullptr;
        for (int d : t.deps)
          if (tt[d].kind == K_GEQRT && tt[d].i == t.i && tt[d].k == t.k) src = &panel_dev[d];
        for (int s = 0; s < S; s += mstrip) {   // one task per mstrip consecutive strips
          const int ns = std::min(mstrip, S - s);
          dl.assign(src->begin(), src->end());
          for (int u = 0; u < ns; ++u) push_lw(i, j, s + u);
          DevTask m = mk(K_UNMQR, i, 0, k, j, s);
          m.pad = ns;
          int id = add(m, dl, start[x]);
          for (int u = 0; u < ns; ++u) lw[slot(i, j, s + u)] = id;
        }
        break;
      }
      case K_TTMQR: case K_TSMQR: {
        const std::vector<int> *src = nullptr;
        const int qk = t.kind == K_TTMQR ? K_TTQRT : K_TSQRT;
        for (int d : t.deps)
          if (tt[d].kind == qk && tt[d].i == t.i && tt[d].k == t.k) src = &panel_dev[d];
        const std::vector<int> *usrc = nullptr;   // fused: the UNMQR's reflector source, GEQRT(i, k)
        if (fused_from[x] >= 0)
          for (int d : tt[fused_from[x]].deps)
            if (tt[d].kind == K_GEQRT && tt[d].i == t.i && tt[d].k == t.k) usrc = &panel_dev[d];
        for (int s = 0; s < S; s += mstrip) {
          const int ns = std::min(mstrip, S - s);
          dl.assign(src->begin(), src->end());
          if (usrc) dl.insert(dl.end(), usrc->begin(), usrc->end());
          for (int u = 0; u < ns; ++u) { push_lw(pv, j, s + u); push_lw(i, j, s + u); }
          DevTask m = mk(usrc ? K_UNTTMQR : t.kind, i, pv, k, j, s);
          m.pad = ns;
          int id = add(m, dl, start[x]);
          for (int u = 0; u < ns; ++u) lw[slot(pv, j, s + u)] = lw[slot(i, j, s + u)] = id;
        }
        break;
      }
      default: break;
    }
  }
  reorder(g, key, deps);
}

void build_apply_graph(const std::vector<TileTask> &tt, int p, int qc, int nb, int ws,
                       bool trans, DevGraph &g) {
  const int S = (nb + ws - 1) / ws;
  g.tasks.clear();
  std::vector<std::vector<int>> deps;
  std::vector<std::pair<int64_t, int64_t>> key;
  std::vector<int> lw((size_t)p * qc * S, -1);
  std::vector<int64_t> fin;   // ASAP finish of each device task (priority)
  auto slot = [p, S](int r, int c, int s) { return ((size_t)c * p + r) * S + s; };
  std::vector<size_t> order;
  for (size_t x = 0; x < tt.size(); ++x)
    if (tt[x].kind == K_GEQRT || tt[x].kind == K_TTQRT || tt[x].kind == K_TSQRT) order.push_back(x);
  if (!trans) std::reverse(order.begin(), order.end());
  for (size_t x : order) {
    const TileTask &t = tt[x];
    const int i = t.i - 1, pv = t.piv - 1, k = t.k - 1;
    for (int c = 0; c < qc; ++c)
      for (int s = 0; s < S; ++s) {
        std::vector<int> d;
        int64_t st = 0;
        int kind, w;
        if (t.kind == K_GEQRT) {
          kind = K_AP_UNMQR; w = 6;
          if (lw[slot(i, c, s)] >= 0) d.push_back(lw[slot(i, c, s)]);
        } else {
          kind = t.kind == K_TTQRT ? K_AP_TTMQR : K_AP_TSMQR; w = t.kind == K_TTQRT ? 6 : 12;
          if (lw[slot(pv, c, s)] >= 0) d.push_back(lw[slot(pv, c, s)]);
          if (lw[slot(i, c, s)] >= 0) d.push_back(lw[slot(i, c, s)]);
        }
        for (int y : d) st = std::max(st, fin[y]);
        g.tasks.push_back(mk(kind, i, t.kind == K_GEQRT ? 0 : pv, k, c, s));
        deps.push_back(d);
        fin.push_back(st + w);
        key.emplace_back(st, (int64_t)g.tasks.size());
        int id = (int)g.tasks.size() - 1;
        lw[slot(i, c, s)] = id;
        if (t.kind != K_GEQRT) lw[slot(pv, c, s)] = id;
      }
  }
  reorder(g, key, deps);
}

// Relative task durations for the bottom-level priorities (microseconds of the
// B200 kernels on nb = 200 tiles, from the per-task tracer; only the ratios matter).
static double est_kind_duration(int kind) {
  switch (kind) {
    case K_GEQRT_B: case K_TTQRT_B: return 71;
    case K_TSQRT_B: return 80;
    case K_GEQRT_U: case K_TTQRT_U: case K_TSQRT_U: return 10;
    case K_UNMQR: case K_AP_UNMQR: return 40;
    case K_TTMQR: case K_AP_TTMQR: return 52;
    case K_UNTTMQR: return 84;
    case K_TSMQR: case K_AP_TSMQR: return 64;
    case K_GEQRT: return 450;
    case K_TTQRT: return 430;
    case K_TSQRT: return 500;
    default: return 40;
  }
}

static double est_duration(const DevTask &t) {   // multi-strip update tasks run their strips in turn
  return est_kind_duration(t.kind) * (t.pad > 1 ? t.pad : 1);
}

// Non-preemptive list scheduling on nproc identical processors: whenever a
// processor is free, start the ready task with the highest key. Returns the
// makespan; start[t] receives each task's start time.
static double list_schedule(const DevGraph &g, const std::vector<int32_t> &cnt, const std::vector<double> &key,
                            int nproc, std::vector<double> &start) {
  const int n = (int)g.tasks.size();
  std::vector<int> indeg(n, 0);
  for (int t = 0; t < n; ++t)
    for (int x = cnt[t]; x < cnt[t + 1]; ++x) ++indeg[g.succ[x]];
  using RT = std::pair<double, int>;                         // (key, task): max-heap of ready tasks
  std::priority_queue<RT> ready;
  using EV = std::pair<double, int>;                         // (finish time, task): min-heap of running
  std::priority_queue<EV, std::vector<EV>, std::greater<EV>> running;
  for (int t = 0; t < n; ++t)
    if (indeg[t] == 0) ready.emplace(key[t], t);
  double now = 0.0, mk = 0.0;
  int free = nproc;
  while (!ready.empty() || !running.empty()) {
    while (free > 0 && !ready.empty()) {
      const int t = ready.top().second;
      ready.pop();
      start[t] = now;
      running.emplace(now + est_duration(g.tasks[t]), t);
      --free;
    }
    if (running.empty()) break;
    const double tf = running.top().first;
    now = tf;
    while (!running.empty() && running.top().first <= tf) {
      const int t = running.top().second;
      running.pop();
      ++free;
      mk = std::max(mk, tf);
      for (int x = cnt[t]; x < cnt[t + 1]; ++x)
        if (--indeg[g.succ[x]] == 0) ready.emplace(key[g.succ[x]], g.succ[x]);
    }
  }
  return mk;
}

void finalize_dataflow(DevGraph &g, bool lookahead, int levels, int prio_rule, int nproc) {
  const int n = (int)g.tasks.size();
  std::vector<int32_t> cnt(n + 1, 0);
  for (int t = 0; t < n; ++t)
    for (int d = g.tasks[t].dep_begin; d < g.tasks[t].dep_end; ++d) ++cnt[g.deps[d] + 1];
  for (int t = 0; t < n; ++t) cnt[t + 1] += cnt[t];
  g.succ.assign(cnt[n], 0);
  std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1);
  g.roots.clear();
  for (int t = 0; t < n; ++t) {
    const DevTask &x = g.tasks[t];
    for (int d = x.dep_begin; d < x.dep_end; ++d) g.succ[fill[g.deps[d]]++] = t;
  }
  std::vector<char> chained(n, 0);
  for (int t = 0; t < n; ++t)
    if (g.tasks[t].chain >= 0) chained[g.tasks[t].chain] = 1;
  // bottom level = longest estimated path from the task to the end (tasks are
  // in a topological order); priority level = its quantised fraction of the max
  std::vector<double> bl(n, 0.0);
  double blmax = 1.0;
  for (int t = n - 1; t >= 0; --t) {
    double m = 0.0;
    for (int x = cnt[t]; x < cnt[t + 1]; ++x) m = std::max(m, bl[g.succ[x]]);
    bl[t] = est_duration(g.tasks[t]) + m;
    blmax = std::max(blmax, bl[t]);
  }
  // ASAP start of every task with the same estimates (tasks are in topological order)
  std::vector<double> asap(n, 0.0);
  for (int t = 0; t < n; ++t) {
    const double f = asap[t] + est_duration(g.tasks[t]);
    for (int x = cnt[t]; x < cnt[t + 1]; ++x) asap[g.succ[x]] = std::max(asap[g.succ[x]], f);
  }
  // priority key: 0 = bottom level; 1 = earliest ASAP start first; 2 = bottom level
  // plus (CP - ASAP start): also lifts early tasks whose long chains have slack in the
  // unbounded model but become critical once resources are limited
  std::vector<double> key(n);
  double kmax = 1e-9;
  auto make_key = [&](int rule, double alpha, std::vector<double> &k) {
    for (int t = 0; t < n; ++t)
      k[t] = rule == 1 ? blmax - asap[t] : (rule == 2 ? bl[t] + alpha * (blmax - asap[t]) : bl[t]);
  };
  if (prio_rule == 3) {
    // list-schedule the graph on `nproc` SMs with each candidate key (host DES with the
    // duration estimates); keep the best and use its simulated start order as priority
    std::vector<double> cand(n), best_start, start(n);
    double best = 1e300;
    for (double alpha : {0.0, 0.25, 0.5, 1.0, 2.0}) {
      make_key(alpha == 0.0 ? 0 : 2, alpha, cand);
      const double mk = list_schedule(g, cnt, cand, nproc, start);
      if (mk < best) { best = mk; best_start = start; }
    }
    double smax = 1e-9;
    for (int t = 0; t < n; ++t) smax = std::max(smax, best_start[t]);
    for (int t = 0; t < n; ++t) key[t] = smax - best_start[t];       // earlier simulated start = higher
  } else {
    make_key(prio_rule, 1.0, key);
  }
  for (int t = 0; t < n; ++t) kmax = std::max(kmax, key[t]);
  for (int t = 0; t < n; ++t) {
    DevTask &x = g.tasks[t];
    const int indeg = x.dep_end - x.dep_begin;
    const int nlev = std::min(kLevels, std::max(1, levels));
    int level = lookahead ? std::min(nlev - 1, std::max(0, (int)(nlev * key[t] / kmax))) : 0;
    x.meta = indeg | (level << 16) | (chained[t] ? 1 << 20 : 0);
    x.dep_begin = cnt[t];
    x.dep_end = cnt[t + 1];
    if (indeg == 0) g.roots.push_back(t);
  }
}

}  // namespace tqr
