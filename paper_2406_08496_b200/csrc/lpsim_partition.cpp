// lpsim_partition.cpp — node partition for the multi-partition step (§8(e)).
//
// Weighted recursive coordinate bisection: the paper partitions a graph whose
// node weights are the route visit counts over the studied window
// and assigns never-visited nodes to the nearest subgraph.  RCB on
// node coordinates does both at once: the split points balance the visit
// weight, and a zero-weight node lands in the part whose region contains it.
// Balanced multilevel k-way partition (§8(f) item 1): the graph is
// coarsened by heavy-edge matching, the coarsest graph is split by recursive
// greedy graph growing, and the partition is projected back level by level
// with greedy boundary refinement under a balance bound — the METIS scheme
// the paper uses, written from its description.  Unbalanced Leiden + k-means
// (P:L423-429): modularity communities (local moving, then each community
// split into its connected components — Leiden's connectivity guarantee —
// then aggregation, repeated), grouped into k parts by weighted k-means on
// the community centroids.  The partition affects speed only, never results.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

#include "../../include/lpsim.h"

namespace {

void rcb(std::vector<int32_t>& idx, size_t lo, size_t hi, int32_t k0, int32_t K, const float* xy,
         const double* w, int32_t* part) {
  if (K <= 1 || hi - lo <= 1) {
    for (size_t i = lo; i < hi; ++i) part[idx[i]] = k0;
    return;
  }
  // axis of the larger extent (node id order when no coordinates)
  int axis = 2;
  if (xy) {
    float mnx = xy[2 * idx[lo]], mxx = mnx, mny = xy[2 * idx[lo] + 1], mxy = mny;
    for (size_t i = lo; i < hi; ++i) {
      const float x = xy[2 * idx[i]], y = xy[2 * idx[i] + 1];
      mnx = std::min(mnx, x); mxx = std::max(mxx, x);
      mny = std::min(mny, y); mxy = std::max(mxy, y);
    }
    axis = (mxx - mnx) >= (mxy - mny) ? 0 : 1;
  }
  auto key = [&](int32_t n) -> double { return axis == 2 ? (double)n : (double)xy[2 * n + axis]; };
  std::sort(idx.begin() + lo, idx.begin() + hi, [&](int32_t a, int32_t b) {
    const double ka = key(a), kb = key(b);
    return ka < kb || (ka == kb && a < b);
  });
  const int32_t K1 = K / 2, K2 = K - K1;
  double tot = 0.0;
  for (size_t i = lo; i < hi; ++i) tot += w[idx[i]];
  size_t cut = lo;
  if (tot > 0.0) {
    const double target = tot * (double)K1 / (double)K;
    double acc = 0.0;
    while (cut < hi && acc + w[idx[cut]] <= target) acc += w[idx[cut++]];
    if (cut < hi && (target - acc) > 0.5 * w[idx[cut]]) acc += w[idx[cut++]];
  } else {
    cut = lo + (hi - lo) * (size_t)K1 / (size_t)K;
  }
  cut = std::max(cut, lo + 1);
  cut = std::min(cut, hi - 1);
  rcb(idx, lo, cut, k0, K1, xy, w, part);
  rcb(idx, cut, hi, k0 + K1, K2, xy, w, part);
}

// ---- balanced multilevel k-way ----
struct Level {
  std::vector<int64_t> xadj;    // undirected CSR
  std::vector<int32_t> adj;
  std::vector<double> ew;       // edge weights (both directions)
  std::vector<double> vw;       // vertex weights
  std::vector<int32_t> cmap;    // vertex -> coarse vertex of the next level
  int32_t n() const { return (int32_t)vw.size(); }
};

// heavy-edge matching; returns the coarse level (cmap of `f` filled)
Level coarsen(Level& f, double max_vw, std::mt19937_64& rng) {
  const int32_t n = f.n();
  std::vector<int32_t> order((size_t)n), match((size_t)n, -1);
  std::iota(order.begin(), order.end(), 0);
  std::shuffle(order.begin(), order.end(), rng);
  for (int32_t u : order) {
    if (match[u] >= 0) continue;
    int32_t best = u;
    double bw = -1.0;
    for (int64_t e = f.xadj[u]; e < f.xadj[u + 1]; ++e) {
      const int32_t v = f.adj[e];
      if (match[v] >= 0 || v == u || f.vw[u] + f.vw[v] > max_vw) continue;
      if (f.ew[e] > bw || (f.ew[e] == bw && v < best)) { bw = f.ew[e]; best = v; }
    }
    match[u] = best;
    match[best] = u;
  }
  f.cmap.assign((size_t)n, -1);
  int32_t nc = 0;
  for (int32_t u = 0; u < n; ++u)
    if (f.cmap[u] < 0) { f.cmap[u] = nc; f.cmap[match[u]] = nc; ++nc; }
  Level c;
  c.vw.assign((size_t)nc, 0.0);
  std::vector<std::vector<int32_t>> members((size_t)nc);
  for (int32_t u = 0; u < n; ++u) { c.vw[f.cmap[u]] += f.vw[u]; members[f.cmap[u]].push_back(u); }
  c.xadj.assign((size_t)nc + 1, 0);
  std::vector<int64_t> slot((size_t)nc, -1);  // position of coarse neighbour in the row being built
  for (int32_t cu = 0; cu < nc; ++cu) {
    const int64_t row0 = (int64_t)c.adj.size();
    for (int32_t u : members[cu])
      for (int64_t e = f.xadj[u]; e < f.xadj[u + 1]; ++e) {
        const int32_t cv = f.cmap[f.adj[e]];
        if (cv == cu) continue;
        if (slot[cv] < row0) { slot[cv] = (int64_t)c.adj.size(); c.adj.push_back(cv); c.ew.push_back(0.0); }
        c.ew[slot[cv]] += f.ew[e];
      }
    c.xadj[cu + 1] = (int64_t)c.adj.size();
  }
  return c;
}

// greedy graph growing bisection of the vertices in `set` (part ids a / b), target weight share
// `frac` for side a; a few seeds, the lowest cut kept
void grow_bisect(const Level& L, const std::vector<int32_t>& set, int32_t a, int32_t b, double frac,
                 std::vector<int32_t>& part, std::mt19937_64& rng) {
  double tot = 0.0;
  for (int32_t u : set) tot += L.vw[u];
  const double target = tot * frac;
  std::vector<char> in((size_t)L.n(), 0);
  for (int32_t u : set) in[u] = 1;
  double best_cut = -1.0;
  std::vector<int32_t> best;
  std::vector<double> gain((size_t)L.n(), 0.0);
  std::vector<char> side((size_t)L.n(), 0);
  for (int trial = 0; trial < 4 && !set.empty(); ++trial) {
    for (int32_t u : set) { side[u] = 0; gain[u] = 0.0; }
    const int32_t seed = set[rng() % set.size()];
    double acc = 0.0;
    std::vector<int32_t> frontier{seed};
    std::vector<char> inf((size_t)L.n(), 0);
    inf[seed] = 1;
    size_t taken = 0;
    while (acc < target && taken < set.size()) {
      int32_t pick = -1;
      double pg = -1e300;
      size_t pi = 0;
      for (size_t i = 0; i < frontier.size(); ++i) {
        const int32_t u = frontier[i];
        if (gain[u] > pg || (gain[u] == pg && u < pick)) { pg = gain[u]; pick = u; pi = i; }
      }
      if (pick < 0) {  // disconnected remainder: any vertex not taken
        for (int32_t u : set) if (!side[u]) { pick = u; break; }
        frontier.push_back(pick);
        pi = frontier.size() - 1;
        inf[pick] = 1;
      }
      frontier[pi] = frontier.back();
      frontier.pop_back();
      side[pick] = 1;
      acc += L.vw[pick];
      ++taken;
      for (int64_t e = L.xadj[pick]; e < L.xadj[pick + 1]; ++e) {
        const int32_t v = L.adj[e];
        if (!in[v] || side[v]) continue;
        gain[v] += 2.0 * L.ew[e];
        if (!inf[v]) { inf[v] = 1; frontier.push_back(v); }
      }
    }
    double cut = 0.0;
    for (int32_t u : set)
      if (side[u])
        for (int64_t e = L.xadj[u]; e < L.xadj[u + 1]; ++e)
          if (in[L.adj[e]] && !side[L.adj[e]]) cut += L.ew[e];
    if (best_cut < 0.0 || cut < best_cut) {
      best_cut = cut;
      best.clear();
      for (int32_t u : set) if (side[u]) best.push_back(u);
    }
  }
  for (int32_t u : set) part[u] = b;
  for (int32_t u : best) part[u] = a;
}

void recursive_grow(const Level& L, const std::vector<int32_t>& set, int32_t k0, int32_t K, std::vector<int32_t>& part,
                    std::mt19937_64& rng) {
  if (K <= 1 || set.size() <= 1) {
    for (int32_t u : set) part[u] = k0;
    return;
  }
  const int32_t K1 = K / 2;
  grow_bisect(L, set, k0, k0 + K1, (double)K1 / (double)K, part, rng);
  std::vector<int32_t> s1, s2;
  for (int32_t u : set) (part[u] == k0 ? s1 : s2).push_back(u);
  recursive_grow(L, s1, k0, K1, part, rng);
  recursive_grow(L, s2, k0 + K1, K - K1, part, rng);
}

// greedy k-way boundary refinement: move a vertex to the adjacent part with the largest cut gain
// if the target stays under max_pw; overweight parts shed their least-loss boundary vertices
void refine(const Level& L, int32_t K, double max_pw, std::vector<int32_t>& part, std::mt19937_64& rng) {
  const int32_t n = L.n();
  std::vector<double> pw((size_t)K, 0.0), conn((size_t)K, 0.0);
  for (int32_t u = 0; u < n; ++u) pw[part[u]] += L.vw[u];
  std::vector<int32_t> order((size_t)n), touched;
  std::iota(order.begin(), order.end(), 0);
  for (int pass = 0; pass < 8; ++pass) {
    std::shuffle(order.begin(), order.end(), rng);
    int moves = 0;
    for (int32_t u : order) {
      const int32_t own = part[u];
      touched.clear();
      bool boundary = false;
      for (int64_t e = L.xadj[u]; e < L.xadj[u + 1]; ++e) {
        const int32_t p = part[L.adj[e]];
        if (conn[p] == 0.0) touched.push_back(p);
        conn[p] += L.ew[e];
        boundary |= p != own;
      }
      if (boundary) {
        const bool over = pw[own] > max_pw;
        int32_t bp = -1;
        double bg = 0.0;
        for (int32_t p : touched) {
          if (p == own || pw[p] + L.vw[u] > max_pw) continue;
          const double g = conn[p] - conn[own];
          const bool better = bp < 0 ? (g > 0.0 || (g == 0.0 && pw[p] + L.vw[u] < pw[own]) || over)
                                     : (g > bg || (g == bg && pw[p] < pw[bp]));
          if (better) { bp = p; bg = g; }
        }
        if (bp >= 0) {
          pw[own] -= L.vw[u];
          pw[bp] += L.vw[u];
          part[u] = bp;
          ++moves;
        }
      }
      for (int32_t p : touched) conn[p] = 0.0;
      conn[own] = 0.0;
    }
    if (moves == 0) break;
  }
}

// ---- unbalanced Leiden communities + k-means ----
// one level of modularity local moving (resolution gamma) on L; comm[] in/out
void local_moving(const Level& L, const std::vector<double>& self, double gamma, std::vector<int32_t>& comm,
                  std::mt19937_64& rng) {
  const int32_t n = L.n();
  std::vector<double> kdeg((size_t)n, 0.0), tot((size_t)n, 0.0), link((size_t)n, 0.0);
  double m2 = 0.0;
  for (int32_t u = 0; u < n; ++u) {
    for (int64_t e = L.xadj[u]; e < L.xadj[u + 1]; ++e) kdeg[u] += L.ew[e];
    kdeg[u] += self[u];
    m2 += kdeg[u];
  }
  if (m2 <= 0.0) return;
  for (int32_t u = 0; u < n; ++u) tot[comm[u]] += kdeg[u];
  std::vector<int32_t> order((size_t)n), seen;
  std::iota(order.begin(), order.end(), 0);
  for (int pass = 0; pass < 16; ++pass) {
    std::shuffle(order.begin(), order.end(), rng);
    int moves = 0;
    for (int32_t u : order) {
      const int32_t cu = comm[u];
      seen.clear();
      for (int64_t e = L.xadj[u]; e < L.xadj[u + 1]; ++e) {
        const int32_t c = comm[L.adj[e]];
        if (link[c] == 0.0) seen.push_back(c);
        link[c] += L.ew[e];
      }
      tot[cu] -= kdeg[u];
      int32_t best = cu;
      double bg = link[cu] - gamma * tot[cu] * kdeg[u] / m2;
      for (int32_t c : seen) {
        const double gn = link[c] - gamma * tot[c] * kdeg[u] / m2;
        if (gn > bg + 1e-12) { bg = gn; best = c; }  // strict gain: ties stay (no oscillation)
      }
      tot[best] += kdeg[u];
      if (best != cu) { comm[u] = best; ++moves; }
      for (int32_t c : seen) link[c] = 0.0;
      link[cu] = 0.0;
    }
    if (moves == 0) break;
  }
}

// split every community into its connected components (Leiden's refinement guarantee: no
// community is internally disconnected); returns the number of refined communities
int32_t split_components(const Level& L, std::vector<int32_t>& comm) {
  const int32_t n = L.n();
  std::vector<int32_t> out((size_t)n, -1), stack;
  int32_t nc = 0;
  for (int32_t s0 = 0; s0 < n; ++s0) {
    if (out[s0] >= 0) continue;
    out[s0] = nc;
    stack.assign(1, s0);
    while (!stack.empty()) {
      const int32_t u = stack.back();
      stack.pop_back();
      for (int64_t e = L.xadj[u]; e < L.xadj[u + 1]; ++e) {
        const int32_t v = L.adj[e];
        if (out[v] < 0 && comm[v] == comm[s0]) { out[v] = nc; stack.push_back(v); }
      }
    }
    ++nc;
  }
  comm.swap(out);
  return nc;
}

}  // namespace

extern "C" lpsim_status lpsim_partition_rcb(int32_t num_nodes, const float* node_xy, const double* weight, int32_t k,
                                           int32_t* part_out) {
  if (num_nodes <= 0 || k < 1 || !part_out) return LPSIM_E_INVALID_ARG;
  std::vector<double> w((size_t)num_nodes, 0.0);
  if (weight)
    for (int32_t i = 0; i < num_nodes; ++i) w[i] = weight[i] > 0.0 ? weight[i] : 0.0;
  std::vector<int32_t> idx((size_t)num_nodes);
  std::iota(idx.begin(), idx.end(), 0);
  rcb(idx, 0, idx.size(), 0, k, node_xy, w.data(), part_out);
  return LPSIM_OK;
}

extern "C" lpsim_status lpsim_plan_cut_lanes(const lpsim_graph* g, const int32_t* node_part, int32_t k, int64_t* out) {
  if (!g || !node_part || k < 1 || !out || g->num_nodes <= 0 || g->num_edges < 0 || !g->row_ptr ||
      (g->num_edges > 0 && (!g->dst || !g->lanes)))
    return LPSIM_E_INVALID_ARG;
  for (int64_t i = 0; i < (int64_t)k * k; ++i) out[i] = 0;
  for (int32_t u = 0; u < g->num_nodes; ++u) {
    const int32_t p = node_part[u];
    if (p < 0 || p >= k) return LPSIM_E_INVALID_ARG;
    for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e) {
      const int32_t w = g->dst[e];
      if (w < 0 || w >= g->num_nodes) return LPSIM_E_INVALID_GRAPH;
      const int32_t q = node_part[w];
      if (q < 0 || q >= k) return LPSIM_E_INVALID_ARG;
      if (p != q) out[(int64_t)p * k + q] += g->lanes[e];
    }
  }
  return LPSIM_OK;
}

extern "C" lpsim_status lpsim_partition_multilevel(const lpsim_graph* g, const double* node_weight,
                                                  const double* edge_weight, int32_t k, double imbalance,
                                                  uint64_t seed, int32_t* part_out) {
  if (!g || k < 1 || !part_out || g->num_nodes <= 0 || g->num_edges < 0 || !g->row_ptr ||
      (g->num_edges > 0 && !g->dst) || !(imbalance >= 0.0) || (!edge_weight && g->num_edges > 0 && !g->lanes))
    return LPSIM_E_INVALID_ARG;
  const int32_t N = g->num_nodes;
  if (k == 1) {
    std::fill(part_out, part_out + N, 0);
    return LPSIM_OK;
  }
  // symmetrised, merged adjacency; vertex weights = visits (zero-visit nodes get a small weight so
  // that they still follow their neighbours: "nearest subgraph")
  Level L0;
  L0.vw.assign((size_t)N, 1.0);
  if (node_weight) {
    double tot = 0.0;
    for (int32_t u = 0; u < N; ++u) tot += node_weight[u] > 0.0 ? node_weight[u] : 0.0;
    const double eps = tot > 0.0 ? 1e-6 * tot / N : 1.0;
    for (int32_t u = 0; u < N; ++u) L0.vw[u] = (node_weight[u] > 0.0 ? node_weight[u] : 0.0) + eps;
  }
  std::vector<int64_t> deg((size_t)N + 1, 0);
  for (int32_t u = 0; u < N; ++u)
    for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e) {
      const int32_t v = g->dst[e];
      if (v < 0 || v >= N) return LPSIM_E_INVALID_GRAPH;
      if (v != u) { ++deg[u + 1]; ++deg[v + 1]; }
    }
  for (int32_t u = 0; u < N; ++u) deg[u + 1] += deg[u];
  std::vector<int32_t> tadj((size_t)deg[N]);
  std::vector<double> tw((size_t)deg[N]);
  {
    std::vector<int64_t> pos(deg.begin(), deg.end() - 1);
    for (int32_t u = 0; u < N; ++u)
      for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e) {
        const int32_t v = g->dst[e];
        if (v == u) continue;
        const double w = edge_weight ? std::max(edge_weight[e], 0.0) : (double)g->lanes[e];
        tadj[pos[u]] = v; tw[pos[u]++] = w;
        tadj[pos[v]] = u; tw[pos[v]++] = w;
      }
  }
  L0.xadj.assign((size_t)N + 1, 0);
  {
    std::vector<int64_t> slot((size_t)N, -1);
    for (int32_t u = 0; u < N; ++u) {
      const int64_t row0 = (int64_t)L0.adj.size();
      for (int64_t e = deg[u]; e < deg[u + 1]; ++e) {
        const int32_t v = tadj[e];
        if (slot[v] < row0) { slot[v] = (int64_t)L0.adj.size(); L0.adj.push_back(v); L0.ew.push_back(0.0); }
        L0.ew[slot[v]] += tw[e];
      }
      L0.xadj[u + 1] = (int64_t)L0.adj.size();
    }
  }
  std::mt19937_64 rng(seed);
  double total = 0.0;
  for (double w : L0.vw) total += w;
  const double max_pw = (1.0 + imbalance) * total / k;
  // coarsen until ~30 vertices per part (or no more progress)
  std::vector<Level> levels;
  levels.push_back(std::move(L0));
  const double max_vw = 1.5 * total / std::max<double>(30.0 * k, 1.0);
  while (levels.back().n() > 30 * k) {
    Level c = coarsen(levels.back(), max_vw, rng);
    if (c.n() > 0.95 * levels.back().n()) { levels.back().cmap.clear(); break; }
    levels.push_back(std::move(c));
  }
  // initial partition of the coarsest graph, then project + refine level by level
  std::vector<int32_t> part((size_t)levels.back().n(), 0);
  {
    std::vector<int32_t> all((size_t)levels.back().n());
    std::iota(all.begin(), all.end(), 0);
    recursive_grow(levels.back(), all, 0, k, part, rng);
    refine(levels.back(), k, max_pw, part, rng);
  }
  for (int li = (int)levels.size() - 2; li >= 0; --li) {
    const Level& f = levels[li];
    std::vector<int32_t> fp((size_t)f.n());
    for (int32_t u = 0; u < f.n(); ++u) fp[u] = part[f.cmap[u]];
    part.swap(fp);
    refine(f, k, max_pw, part, rng);
  }
  std::copy(part.begin(), part.end(), part_out);
  return LPSIM_OK;
}

extern "C" lpsim_status lpsim_partition_leiden_kmeans(const lpsim_graph* g, const double* node_weight,
                                                     const double* edge_weight, int32_t k, double resolution,
                                                     uint64_t seed, int32_t* part_out) {
  if (!g || k < 1 || !part_out || g->num_nodes <= 0 || g->num_edges < 0 || !g->row_ptr || !g->node_xy ||
      (g->num_edges > 0 && !g->dst) || !(resolution > 0.0) || (!edge_weight && g->num_edges > 0 && !g->lanes))
    return LPSIM_E_INVALID_ARG;
  const int32_t N = g->num_nodes;
  // symmetrised merged adjacency (as the multilevel partition)
  Level L;
  L.vw.assign((size_t)N, 1.0);
  std::vector<std::vector<std::pair<int32_t, double>>> nb((size_t)N);
  for (int32_t u = 0; u < N; ++u)
    for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e) {
      const int32_t v = g->dst[e];
      if (v < 0 || v >= N) return LPSIM_E_INVALID_GRAPH;
      if (v == u) continue;
      const double w = edge_weight ? std::max(edge_weight[e], 0.0) : (double)g->lanes[e];
      nb[u].push_back({v, w});
      nb[v].push_back({u, w});
    }
  L.xadj.assign((size_t)N + 1, 0);
  for (int32_t u = 0; u < N; ++u) {
    std::sort(nb[u].begin(), nb[u].end());
    for (size_t j = 0; j < nb[u].size(); ++j) {
      if (j > 0 && nb[u][j].first == nb[u][j - 1].first) { L.ew.back() += nb[u][j].second; continue; }
      L.adj.push_back(nb[u][j].first);
      L.ew.push_back(nb[u][j].second);
    }
    L.xadj[u + 1] = (int64_t)L.adj.size();
    std::vector<std::pair<int32_t, double>>().swap(nb[u]);
  }
  std::mt19937_64 rng(seed);
  // Leiden-style levels: local moving, connected-component refinement, aggregation
  std::vector<int32_t> node_comm((size_t)N);
  std::iota(node_comm.begin(), node_comm.end(), 0);
  Level cur = L;
  std::vector<double> self((size_t)N, 0.0);
  for (int level = 0; level < 20; ++level) {
    const int32_t n = cur.n();
    std::vector<int32_t> comm((size_t)n);
    std::iota(comm.begin(), comm.end(), 0);
    local_moving(cur, self, resolution, comm, rng);
    const int32_t nc = split_components(cur, comm);
    if (nc == n) break;
    for (int32_t u = 0; u < N; ++u) node_comm[u] = comm[node_comm[u]];
    // aggregate: coarse vertex = refined community; internal weight kept as a self loop
    Level nxt;
    nxt.vw.assign((size_t)nc, 0.0);
    std::vector<double> nself((size_t)nc, 0.0);
    std::vector<std::vector<int32_t>> members((size_t)nc);
    for (int32_t u = 0; u < n; ++u) { members[comm[u]].push_back(u); nxt.vw[comm[u]] += cur.vw[u]; nself[comm[u]] += self[u]; }
    nxt.xadj.assign((size_t)nc + 1, 0);
    std::vector<int64_t> slot((size_t)nc, -1);
    for (int32_t c = 0; c < nc; ++c) {
      const int64_t row0 = (int64_t)nxt.adj.size();
      for (int32_t u : members[c])
        for (int64_t e = cur.xadj[u]; e < cur.xadj[u + 1]; ++e) {
          const int32_t cv = comm[cur.adj[e]];
          if (cv == c) { nself[c] += cur.ew[e]; continue; }
          if (slot[cv] < row0) { slot[cv] = (int64_t)nxt.adj.size(); nxt.adj.push_back(cv); nxt.ew.push_back(0.0); }
          nxt.ew[slot[cv]] += cur.ew[e];
        }
      nxt.xadj[c + 1] = (int64_t)nxt.adj.size();
    }
    cur = std::move(nxt);
    self.swap(nself);
  }
  // k-means (Lloyd, k-means++ seeding from `seed`) on the community centroids, weighted by visits
  int32_t C = 0;
  for (int32_t u = 0; u < N; ++u) C = std::max(C, node_comm[u] + 1);
  std::vector<double> cw((size_t)C, 0.0), cx((size_t)C, 0.0), cy((size_t)C, 0.0);
  for (int32_t u = 0; u < N; ++u) {
    const double w = (node_weight && node_weight[u] > 0.0 ? node_weight[u] : 0.0) + 1e-9;
    const int32_t c = node_comm[u];
    cw[c] += w; cx[c] += w * g->node_xy[2 * u]; cy[c] += w * g->node_xy[2 * u + 1];
  }
  for (int32_t c = 0; c < C; ++c) { cx[c] /= cw[c]; cy[c] /= cw[c]; }
  const int32_t K = std::min(k, C);
  std::vector<double> mx((size_t)K), my((size_t)K), d2((size_t)C, 1e300);
  std::vector<int32_t> asg((size_t)C, 0);
  {
    const int32_t c0 = (int32_t)(rng() % (uint64_t)C);
    mx[0] = cx[c0]; my[0] = cy[c0];
    for (int32_t j = 1; j < K; ++j) {
      double sum = 0.0;
      for (int32_t c = 0; c < C; ++c) {
        const double dx = cx[c] - mx[j - 1], dy = cy[c] - my[j - 1];
        d2[c] = std::min(d2[c], dx * dx + dy * dy);
        sum += cw[c] * d2[c];
      }
      double r = std::uniform_real_distribution<double>(0.0, sum)(rng);
      int32_t pick = C - 1;
      for (int32_t c = 0; c < C; ++c) { r -= cw[c] * d2[c]; if (r <= 0.0) { pick = c; break; } }
      mx[j] = cx[pick]; my[j] = cy[pick];
    }
  }
  for (int it = 0; it < 100; ++it) {
    bool changed = false;
    for (int32_t c = 0; c < C; ++c) {
      int32_t best = 0;
      double bd = 1e300;
      for (int32_t j = 0; j < K; ++j) {
        const double dx = cx[c] - mx[j], dy = cy[c] - my[j], dd = dx * dx + dy * dy;
        if (dd < bd) { bd = dd; best = j; }
      }
      if (asg[c] != best || it == 0) { changed |= asg[c] != best; asg[c] = best; }
    }
    std::vector<double> sw((size_t)K, 0.0), sx((size_t)K, 0.0), sy((size_t)K, 0.0);
    for (int32_t c = 0; c < C; ++c) { sw[asg[c]] += cw[c]; sx[asg[c]] += cw[c] * cx[c]; sy[asg[c]] += cw[c] * cy[c]; }
    for (int32_t j = 0; j < K; ++j)
      if (sw[j] > 0.0) { mx[j] = sx[j] / sw[j]; my[j] = sy[j] / sw[j]; }
    if (!changed && it > 0) break;
  }
  // parts renumbered densely in first-appearance order (empty clusters dropped)
  std::vector<int32_t> remap((size_t)K, -1);
  int32_t np = 0;
  for (int32_t u = 0; u < N; ++u) {
    const int32_t j = asg[node_comm[u]];
    if (remap[j] < 0) remap[j] = np++;
    part_out[u] = remap[j];
  }
  return LPSIM_OK;
}
