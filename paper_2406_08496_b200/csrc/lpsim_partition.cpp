// lpsim_partition.cpp — node partition for the multi-partition step (§8(e)).
//
// Weighted recursive coordinate bisection: the paper partitions a graph whose
// node weights are the route visit counts over the studied window
// and assigns never-visited nodes to the nearest subgraph.  RCB on
// node coordinates does both at once: the split points balance the visit
// weight, and a zero-weight node lands in the part whose region contains it.
// (The paper's balanced multilevel and Leiden+k-means variants, P:L413-429,
// are NEXT — the partition affects speed only, never results.)
#include <algorithm>
#include <cstdint>
#include <numeric>
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
