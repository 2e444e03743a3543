// lpsim_capi.cu — host runtime behind the C ABI of include/lpsim.h.
//
// Validation, the spatial tiling (parts -> tiles, neighbour tables, channels),
// device allocation, the departure structures (A7), the launch of the
// persistent step kernel and the result / state queries.  Every step of the
// simulated method runs in the kernels of lpsim_step.cu; this file only
// prepares integer metadata (CSR ranks, ownership, slots, release order) and
// moves data.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lpsim.h"
#include "lpsim_dev.h"
#include "lpsim_kernels.h"

using namespace lpsim;

struct lpsim_ctx {
  std::string err;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  lpsim_config cfg{};
  Params P{};
  // graph (host)
  int32_t n_nodes = 0, n_edges = 0;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> dst, src;
  std::vector<float> length, v0;
  std::vector<uint8_t> lanes;
  std::vector<uint32_t> ncells;
  std::vector<uint64_t> gbase;  // global lane-map layout (a0), from the device builder
  uint64_t total_cells = 0;
  std::vector<uint32_t> meta;   // rank | out-degree << 10 | SIG | PHASE per edge
  std::vector<float> node_xy;
  std::vector<int32_t> node_part;  // user partition (optional)
  // device graph
  float* d_length = nullptr;
  uint8_t* d_lanes = nullptr;
  uint32_t* d_ncells = nullptr;
  float* d_v0 = nullptr;
  uint64_t* d_gbase = nullptr;
  // demand
  bool loaded = false, restored = false, failed = false;
  int64_t n_trips = 0, r_total = 0;
  std::vector<uint32_t> trip_first_edge;
  uint32_t* d_route = nullptr;
  uint32_t* d_trip_rstart = nullptr;
  int32_t* d_arrival = nullptr;
  int32_t* d_edge_entry = nullptr;
  // tiling
  int32_t K = 1;            // parts (GPUs): num_parts in one process, or world
  int32_t rank = 0, world = 1;
  int max_tiles = 0;        // tiles one GPU runs at once (resident CTAs)
  int32_t n_tiles = 0;
  std::vector<int32_t> part_of;       // node -> part
  std::vector<int32_t> tile_of_node;  // node -> tile
  std::vector<uint8_t> tile_part;     // tile -> part
  std::vector<int32_t> part_tile0;    // first tile of each part (K + 1)
  std::vector<uint8_t> edge_opart;    // part owning each edge
  std::vector<TileInfo> tinfo;
  std::vector<uint4> rel_h;           // releases (for restore's cursor search)
  // device tiling
  EdgeRec* d_edges = nullptr;
  uint8_t *d_edge_mpart = nullptr, *d_edge_opart = nullptr, *d_tile_part = nullptr;
  uint32_t* d_tile_of_edge = nullptr;
  TileInfo* d_tinfo = nullptr;
  TileCtl* d_tctl = nullptr;
  std::vector<PartPtrs> parts;
  PartPtrs* d_parts = nullptr;
  ErrCtl* d_err = nullptr;
  Global G{};
  // instrumentation
  unsigned long long* d_digest_log = nullptr;
  uint32_t digest_cap = 4096;
  std::vector<uint64_t> last_digests;
  int64_t step = 0;
  int64_t on_road_base = 0;  // on-road trips a restore started with (counters start at its values)
  double last_step_ms = 0.0;
  int64_t device_bytes = 0;
  std::vector<void*> allocs;
  int64_t launches = 0;
  std::vector<void*> ipc_opened;
  bool attached = false;
  bool is_local(int32_t p) const { return world == 1 || p == rank; }
  int32_t t0() const { return world == 1 ? 0 : part_tile0[rank]; }
  int32_t t1() const { return world == 1 ? n_tiles : part_tile0[rank + 1]; }
};

namespace {

lpsim_status fail(lpsim_ctx* c, lpsim_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

#define CU(call)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(c, LPSIM_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                      \
  } while (0)

#define TRY(x)                     \
  do {                             \
    lpsim_status s_ = (x);         \
    if (s_ != LPSIM_OK) return s_; \
  } while (0)

template <class T>
lpsim_status dalloc(lpsim_ctx* c, T** p, size_t count) {
  size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  cudaError_t e = cudaMalloc((void**)p, bytes);
  if (e != cudaSuccess) return fail(c, LPSIM_E_NOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
  c->allocs.push_back((void*)*p);
  c->device_bytes += (int64_t)bytes;
  return LPSIM_OK;
}

// every copy and memset that feeds a kernel goes through the context's stream (ordered with it)
template <class T>
lpsim_status upload(lpsim_ctx* c, T** p, const T* h, size_t count) {
  TRY(dalloc(c, p, count));
  if (count) CU(cudaMemcpyAsync(*p, h, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  return LPSIM_OK;
}

int grid_for(size_t n, int bs = 256) {
  size_t g = (n + bs - 1) / bs;
  return (int)std::max<size_t>(1, std::min<size_t>(g, 148 * 16));
}

// depart step = smallest k with k·Δt >= depart_s (Q22), in double
int64_t depart_step_of(double t, float dt) {
  const double h = (double)dt;
  int64_t k = (int64_t)std::ceil(t / h);
  if (k < 0) k = 0;
  while (k > 0 && (double)(k - 1) * h >= t) --k;
  while ((double)k * h < t) ++k;
  return k;
}

int bm_depth_host(uint32_t n) {
  int d = 1;
  uint64_t cap = 32;
  while (cap < n) { cap *= 32; ++d; }
  return d;
}
uint64_t bm_total_words(uint32_t n) {
  const int d = bm_depth_host(n);
  uint64_t t = 0;
  for (int i = 0; i < d; ++i) {
    const uint32_t shift = 5u * (uint32_t)(d - i);
    t += ((uint64_t)n + (1ull << shift) - 1) >> shift;
  }
  return t;
}

// host-side preparation of the demand runs on all host cores: [0, n) split into contiguous ranges
int64_t par_threads(int64_t n, int64_t grain = 65536) {
  const int64_t hw = std::max<int64_t>(1, (int64_t)std::thread::hardware_concurrency());
  return std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(hw, 64), n / grain));
}
template <class F>
void parallel_for(int64_t n, F fn, int64_t grain = 65536) {
  const int64_t nt = par_threads(n, grain);
  if (nt <= 1) {
    fn(0, n, 0);
    return;
  }
  std::vector<std::thread> th;
  for (int64_t t = 0; t < nt; ++t) th.emplace_back([&, t] { fn(n * t / nt, n * (t + 1) / nt, (int)t); });
  for (auto& x : th) x.join();
}

// LPSIM_LOAD_TIMES=1: wall time of the host / setup stages of create and load_demand on stderr
struct StageTimer {
  bool on = std::getenv("LPSIM_LOAD_TIMES") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto u = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[lpsim] %-28s %8.3f s\n", what, std::chrono::duration<double>(u - t).count());
    t = u;
  }
};

lpsim_status upload_parts(lpsim_ctx* c) {
  CU(cudaMemcpyAsync(c->d_parts, c->parts.data(), c->parts.size() * sizeof(PartPtrs), cudaMemcpyHostToDevice,
                     c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return LPSIM_OK;
}

// tiles of a part: the nodes of part p split into `nt` tiles (balanced multilevel partition of the
// induced subgraph on the route-visit weights, P:L413-421 / P:L457; RCB for tiny parts)
void tile_part_nodes(const lpsim_ctx* c, const std::vector<int32_t>& nodes, int32_t nt, const std::vector<double>& w,
                     std::vector<int32_t>& local_tile) {
  const int32_t n = (int32_t)nodes.size();
  local_tile.assign((size_t)n, 0);
  if (nt <= 1 || n == 0) return;
  std::vector<int32_t> idx((size_t)c->n_nodes, -1);
  for (int32_t i = 0; i < n; ++i) idx[nodes[i]] = i;
  std::vector<double> wl((size_t)n);
  for (int32_t i = 0; i < n; ++i) wl[i] = w[nodes[i]];
  if (n >= 8 * nt) {
    std::vector<int64_t> rp((size_t)n + 1, 0);
    std::vector<int32_t> ds;
    std::vector<uint8_t> ln;
    for (int32_t i = 0; i < n; ++i) {
      const int32_t u = nodes[i];
      for (int64_t e = c->row_ptr[u]; e < c->row_ptr[u + 1]; ++e) {
        const int32_t j = idx[c->dst[e]];
        if (j < 0) continue;
        ds.push_back(j);
        ln.push_back(c->lanes[e]);
      }
      rp[i + 1] = (int64_t)ds.size();
    }
    lpsim_graph gg;
    std::memset(&gg, 0, sizeof(gg));
    gg.struct_size = sizeof(gg);
    gg.num_nodes = n;
    gg.num_edges = (int32_t)ds.size();
    gg.row_ptr = rp.data();
    gg.dst = ds.data();
    gg.lanes = ln.data();
    if (lpsim_partition_multilevel(&gg, wl.data(), nullptr, nt, 0.05, 1, local_tile.data()) == LPSIM_OK) return;
  }
  std::vector<float> xy;
  if (!c->node_xy.empty()) {
    xy.resize(2 * (size_t)n);
    for (int32_t i = 0; i < n; ++i) {
      xy[2 * i] = c->node_xy[2 * (size_t)nodes[i]];
      xy[2 * i + 1] = c->node_xy[2 * (size_t)nodes[i] + 1];
    }
  }
  lpsim_partition_rcb(n, xy.empty() ? nullptr : xy.data(), wl.data(), nt, local_tile.data());
}

}  // namespace

// ===========================================================================
extern "C" {

lpsim_status lpsim_config_default(lpsim_config* cfg) {
  if (!cfg) return LPSIM_E_INVALID_ARG;
  if (cfg->struct_size != sizeof(lpsim_config)) return LPSIM_E_INVALID_ARG;
  lpsim_config d;
  std::memset(&d, 0, sizeof(d));
  d.struct_size = sizeof(lpsim_config);
  d.dt_s = 0.5f;
  d.a = 1.5f; d.b = 2.0f; d.s0 = 2.0f; d.T_headway = 1.5f; d.delta = 4;
  d.x0 = 100.0f;
  d.g_a = 2.0f; d.g_b = 2.0f;
  d.alpha_i = 0.5f; d.alpha_a = 0.5f; d.alpha_b = 0.5f;
  d.sigma_a = 0.5f; d.sigma_b = 0.5f;
  d.h_min = 2; d.h_max = 0; d.lc_window = 0; d.sort_every = 0;
  d.seed = 1;
  d.device = 0;
  d.num_parts = 1;
  d.rank = 0;
  d.world = 1;
  *cfg = d;
  return LPSIM_OK;
}

static thread_local std::string g_create_error;

const char* lpsim_last_error(const lpsim_ctx* c) { return c ? c->err.c_str() : g_create_error.c_str(); }

lpsim_status lpsim_create(const lpsim_graph* g, const lpsim_config* cfg, lpsim_ctx** out) {
  StageTimer tm;
  if (!out) return LPSIM_E_INVALID_ARG;
  *out = nullptr;
  if (!g || !cfg || g->struct_size != sizeof(lpsim_graph) || cfg->struct_size != sizeof(lpsim_config))
    return LPSIM_E_INVALID_ARG;
  lpsim_ctx* c = new lpsim_ctx();
  g_create_error.clear();
  auto bail = [&](lpsim_status s) {
    g_create_error = c->err;  // readable through lpsim_last_error(NULL)
    lpsim_destroy(c);
    return s;
  };
  const int32_t N = g->num_nodes, E = g->num_edges;
  // ---- validation ----
  if (N <= 0 || E < 0 || !g->row_ptr || (E > 0 && (!g->dst || !g->length_m || !g->lanes || !g->speed_limit_mps)))
    return bail(fail(c, LPSIM_E_INVALID_ARG, "null array or negative size"));
  if (g->row_ptr[0] != 0) return bail(fail(c, LPSIM_E_INVALID_GRAPH, "row_ptr[0] != 0 (index 0)"));
  for (int32_t u = 0; u < N; ++u) {
    if (g->row_ptr[u + 1] < g->row_ptr[u]) return bail(fail(c, LPSIM_E_INVALID_GRAPH, "row_ptr not monotone (index %d)", u));
    if (g->row_ptr[u + 1] - g->row_ptr[u] > 1023)
      return bail(fail(c, LPSIM_E_CAPACITY, "out-degree > 1023 (node %d)", u));
  }
  if (g->row_ptr[N] != E) return bail(fail(c, LPSIM_E_INVALID_GRAPH, "row_ptr[num_nodes] != num_edges"));
  if ((uint64_t)E > EDGE_MASK) return bail(fail(c, LPSIM_E_CAPACITY, "num_edges >= 2^25"));
  for (int32_t e = 0; e < E; ++e) {
    if (g->dst[e] < 0 || g->dst[e] >= N) return bail(fail(c, LPSIM_E_INVALID_GRAPH, "dst out of range (index %d)", e));
    const float L = g->length_m[e];
    if (!(L >= 1.0f) || !std::isfinite(L)) return bail(fail(c, LPSIM_E_INVALID_GRAPH, "length_m < 1 (index %d)", e));
    if (L > (float)LC_MASK) return bail(fail(c, LPSIM_E_CAPACITY, "length_m >= 2^20 m (index %d)", e));
    if (g->lanes[e] < 1 || g->lanes[e] > 63) return bail(fail(c, LPSIM_E_INVALID_GRAPH, "lanes not in 1..63 (index %d)", e));
    const float v = g->speed_limit_mps[e];
    if (!(v > 0.0f && v <= 254.0f)) return bail(fail(c, LPSIM_E_INVALID_GRAPH, "speed limit not in (0,254] (index %d)", e));
  }
  const lpsim_config& C = *cfg;
  if (!(C.dt_s > 0) || !(C.a > 0) || !(C.b > 0) || C.delta < 1 || C.h_min < 1 || !(C.x0 > 0) || C.num_parts < 1)
    return bail(fail(c, LPSIM_E_INVALID_ARG, "invalid parameter"));
  if (C.num_parts > 15) return bail(fail(c, LPSIM_E_INVALID_ARG, "num_parts > 15"));
  if (C.world < 1 || C.rank < 0 || C.rank >= C.world || C.world > 15)
    return bail(fail(c, LPSIM_E_INVALID_ARG, "rank / world out of range"));
  if (C.world > 1 && C.num_parts != 1 && C.num_parts != C.world)
    return bail(fail(c, LPSIM_E_INVALID_ARG, "multi-process mode: num_parts must be 1 or world"));
  c->cfg = C;
  c->rank = C.rank;
  c->world = C.world;
  c->K = C.world > 1 ? C.world : C.num_parts;  // one part per process in multi-process mode
  c->cfg.num_parts = c->K;
  c->n_nodes = N;
  c->n_edges = E;
  c->row_ptr.assign(g->row_ptr, g->row_ptr + N + 1);
  c->dst.assign(g->dst, g->dst + E);
  c->length.assign(g->length_m, g->length_m + E);
  c->lanes.assign(g->lanes, g->lanes + E);
  c->v0.assign(g->speed_limit_mps, g->speed_limit_mps + E);
  c->src.resize(E);
  for (int32_t u = 0; u < N; ++u)
    for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e) c->src[e] = u;

  // ---- parameters (fp32 constants computed once) ----
  float vmax = 0.0f;
  for (float v : c->v0) vmax = std::max(vmax, v);
  Params& P = c->P;
  P.dt = C.dt_s; P.a = C.a; P.b = C.b; P.s0 = C.s0; P.T = C.T_headway; P.delta = C.delta;
  P.x0 = C.x0; P.g_a = C.g_a; P.g_b = C.g_b; P.alpha_i = C.alpha_i; P.alpha_a = C.alpha_a; P.alpha_b = C.alpha_b;
  volatile float s3 = std::sqrt(3.0f);
  P.sigma_a_s3 = C.sigma_a * s3;
  P.sigma_b_s3 = C.sigma_b * s3;
  volatile float ab = C.a * C.b;
  P.c_ab = 2.0f * std::sqrt((float)ab);
  volatile float dt2 = C.dt_s * C.dt_s;
  P.dt2 = dt2;
  volatile float ha = 0.5f * C.a;
  P.half_a_dt2 = ha * P.dt2;
  P.h_min = C.h_min;
  volatile float twodt = 2.0f * C.dt_s;
  P.h_max = C.h_max > 0 ? C.h_max : (int)std::ceil((float)(twodt * vmax)) + 2;
  P.lc_n = C.lc_window > 0 ? C.lc_window : P.h_max;
  if (!(C.signal_cycle_s >= 0.0f) || !std::isfinite(C.signal_cycle_s))
    return bail(fail(c, LPSIM_E_INVALID_ARG, "signal_cycle_s must be >= 0"));
  P.sig_cycle = C.signal_cycle_s > 0.0f ? (int)std::floor(C.signal_cycle_s / C.dt_s + 0.5f) : 0;
  if (C.signal_cycle_s > 0.0f && P.sig_cycle < 2)
    return bail(fail(c, LPSIM_E_INVALID_ARG, "signal cycle shorter than two steps"));
  P.seed_lo = (uint32_t)(C.seed & 0xFFFFFFFFu);
  P.seed_hi = (uint32_t)(C.seed >> 32);
  P.flags = C.flags;
  P.sort_every = C.sort_every > 0 ? (uint32_t)C.sort_every : 0u;

  // ---- device, stream ----
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) return bail(fail(c, LPSIM_E_CUDA, "no CUDA device"));
  if (C.device < 0 || C.device >= ndev) return bail(fail(c, LPSIM_E_INVALID_ARG, "device %d out of range", C.device));
  c->device = C.device;
  if (cudaSetDevice(c->device) != cudaSuccess) return bail(fail(c, LPSIM_E_CUDA, "cudaSetDevice failed"));
  if (C.stream) {
    c->stream = (cudaStream_t)C.stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
      return bail(fail(c, LPSIM_E_CUDA, "stream create failed"));
    c->own_stream = true;
  }
  cudaEventCreate(&c->ev0);
  cudaEventCreate(&c->ev1);

  // ---- a0 lane-map builder on the device: cells, exclusive scan -> base ----
  lpsim_status s;
  c->meta.assign((size_t)E, 0);
  for (int32_t e = 0; e < E; ++e) {
    const int32_t u = c->src[e], w = c->dst[e];
    const uint32_t rank = (uint32_t)(e - c->row_ptr[u]);
    const uint32_t kout = (uint32_t)(c->row_ptr[w + 1] - c->row_ptr[w]);
    c->meta[e] = rank | (kout << META_KOUT_SHIFT);
  }
  if (P.sig_cycle > 0) {
    // Q30: nodes with >= 3 in-edges are signalised; an approach's phase is 0 if it runs east-west
    // (|dx| >= |dy| from its source to its destination node, fp32), else 1; without coordinates,
    // the parity of its rank among the node's in-edges in edge-id order
    std::vector<int32_t> indeg((size_t)N, 0), inrank((size_t)std::max(E, 1), 0);
    for (int32_t e = 0; e < E; ++e) inrank[e] = indeg[c->dst[e]]++;
    for (int32_t e = 0; e < E; ++e) {
      const int32_t u = c->src[e], w = c->dst[e];
      if (indeg[w] < 3) continue;
      uint32_t ph;
      if (g->node_xy) {
        const float dx = g->node_xy[2 * w] - g->node_xy[2 * u], dy = g->node_xy[2 * w + 1] - g->node_xy[2 * u + 1];
        ph = std::fabs(dx) >= std::fabs(dy) ? 0u : 1u;
      } else {
        ph = (uint32_t)(inrank[e] & 1);
      }
      c->meta[e] |= META_SIG | (ph ? META_PHASE : 0u);
    }
  }
  uint64_t *d_cells = nullptr, *d_sums = nullptr, *d_total = nullptr;
  if ((s = upload(c, &c->d_length, c->length.data(), E)) || (s = upload(c, &c->d_lanes, c->lanes.data(), E)) ||
      (s = upload(c, &c->d_v0, c->v0.data(), E)) || (s = dalloc(c, &d_cells, E)) ||
      (s = dalloc(c, &c->d_ncells, E)) || (s = dalloc(c, &c->d_gbase, E)) ||
      (s = dalloc(c, &d_sums, (E + SCAN_BLOCK - 1) / SCAN_BLOCK + 1)) || (s = dalloc(c, &d_total, 1)))
    return bail(s);
  const int nsb = (E + SCAN_BLOCK - 1) / SCAN_BLOCK;
  if (E > 0) {
    k_edge_cells<<<grid_for(E), 256, 0, c->stream>>>(c->d_length, c->d_lanes, d_cells, c->d_ncells, E);
    k_scan_blocks<<<nsb, SCAN_BLOCK, 0, c->stream>>>(d_cells, c->d_gbase, d_sums, E);
    k_scan_sums<<<1, 32, 0, c->stream>>>(d_sums, nsb, d_total);
    k_scan_add<<<nsb, SCAN_BLOCK, 0, c->stream>>>(c->d_gbase, d_sums, E);
  } else {
    cudaMemsetAsync(d_total, 0, sizeof(uint64_t), c->stream);
  }
  cudaError_t ce = cudaMemcpyAsync(&c->total_cells, d_total, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(c->stream);
  if (ce != cudaSuccess) return bail(fail(c, LPSIM_E_CUDA, "lane-map builder failed: %s", cudaGetErrorString(ce)));
  if (c->total_cells >= (uint64_t)CELL_MASK - 64) return bail(fail(c, LPSIM_E_CAPACITY, "lane map exceeds 2^31 cells"));
  c->gbase.resize(E);
  c->ncells.resize(E);
  if (E) {
    CU(cudaMemcpyAsync(c->gbase.data(), c->d_gbase, sizeof(uint64_t) * E, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(c->ncells.data(), c->d_ncells, sizeof(uint32_t) * E, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  if (g->node_xy) c->node_xy.assign(g->node_xy, g->node_xy + 2 * (size_t)N);
  if (C.node_part) {
    c->node_part.assign(C.node_part, C.node_part + N);
    for (int32_t u = 0; u < N; ++u)
      if (c->node_part[u] < 0 || c->node_part[u] >= c->K)
        return bail(fail(c, LPSIM_E_INVALID_ARG, "node_part out of range (node %d)", u));
  }
  if ((s = dalloc(c, &c->d_err, 1))) return bail(s);
  CU(cudaMemsetAsync(c->d_err, 0, sizeof(ErrCtl), c->stream));
  if ((s = dalloc(c, &c->d_digest_log, c->digest_cap))) return bail(s);

  // ---- tiles per GPU: every CTA of the persistent kernel resident (cooperative launch) ----
  int bpsm = 0, bpsm_full = 0, nsm = 0;
  const size_t dyn = tile_dyn_smem();
  CU(cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  CU(cudaFuncSetAttribute(k_tile_full, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm, k_tile, TILE_BS, dyn));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm_full, k_tile_full, TILE_BS, dyn));
  bpsm = std::min(bpsm, bpsm_full);
  CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
  if (bpsm < 1) return bail(fail(c, LPSIM_E_CUDA, "step kernel cannot be resident"));
  c->max_tiles = std::min(bpsm, TILE_MINB) * nsm;
  if (const char* mb = std::getenv("LPSIM_MAX_BLOCKS")) {  // fewer tiles (tests; processes sharing a GPU)
    const int cap = std::atoi(mb);
    if (cap > 0) c->max_tiles = std::min(c->max_tiles, cap);
  }
  tm.mark("create (graph, lane-map layout)");
  *out = c;
  return LPSIM_OK;
}

lpsim_status lpsim_load_demand(lpsim_ctx* c, int64_t n, const double* depart_s, const int64_t* route_ptr,
                               const int32_t* route_edges, const int32_t* origin, const int32_t* destination) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (c->loaded) return fail(c, LPSIM_E_STATE, "demand already loaded");
  if (n < 0 || (n > 0 && (!depart_s || !route_ptr || !route_edges)))
    return fail(c, LPSIM_E_INVALID_ARG, "null array or negative size");
  if (n >= (int64_t)0x7FFFFFF0ll) return fail(c, LPSIM_E_CAPACITY, "too many trips");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  StageTimer tm;
  const int32_t E = c->n_edges, NN = c->n_nodes;
  // ---- validation ----
  if (n > 0 && route_ptr[0] != 0) return fail(c, LPSIM_E_INVALID_DEMAND, "route_ptr[0] != 0 (trip 0)");
  auto trip_ok = [&](int64_t i) {
    if (!(depart_s[i] >= 0.0) || !std::isfinite(depart_s[i]) || route_ptr[i + 1] <= route_ptr[i]) return false;
    for (int64_t r = route_ptr[i]; r < route_ptr[i + 1]; ++r) {
      const int32_t e = route_edges[r];
      if (e < 0 || e >= E) return false;
      if (r > route_ptr[i] && c->dst[route_edges[r - 1]] != c->src[e]) return false;
    }
    const int32_t o = c->src[route_edges[route_ptr[i]]], d = c->dst[route_edges[route_ptr[i + 1] - 1]];
    if (origin && origin[i] != o) return false;
    if (destination && destination[i] != d) return false;
    if (origin && destination && origin[i] == destination[i]) return false;
    return true;
  };
  std::vector<int64_t> first_bad(64, n);
  parallel_for(n, [&](int64_t a, int64_t b, int t) {
    for (int64_t i = a; i < b; ++i)
      if (!trip_ok(i)) { first_bad[t] = i; break; }
  });
  const int64_t bad0 = *std::min_element(first_bad.begin(), first_bad.end());
  for (int64_t i = bad0; i < std::min(n, bad0 + 1); ++i) {  // the offending trip: the message
    if (!(depart_s[i] >= 0.0) || !std::isfinite(depart_s[i])) return fail(c, LPSIM_E_INVALID_DEMAND, "bad depart_s (trip %lld)", (long long)i);
    if (route_ptr[i + 1] <= route_ptr[i]) return fail(c, LPSIM_E_INVALID_DEMAND, "empty route (trip %lld)", (long long)i);
    for (int64_t r = route_ptr[i]; r < route_ptr[i + 1]; ++r) {
      const int32_t e = route_edges[r];
      if (e < 0 || e >= E) return fail(c, LPSIM_E_INVALID_DEMAND, "route edge out of range (trip %lld)", (long long)i);
      if (r > route_ptr[i] && c->dst[route_edges[r - 1]] != c->src[e])
        return fail(c, LPSIM_E_INVALID_DEMAND, "route not connected (trip %lld)", (long long)i);
    }
    const int32_t o = c->src[route_edges[route_ptr[i]]], d = c->dst[route_edges[route_ptr[i + 1] - 1]];
    if (origin && origin[i] != o) return fail(c, LPSIM_E_INVALID_DEMAND, "origin != from(first edge) (trip %lld)", (long long)i);
    if (destination && destination[i] != d) return fail(c, LPSIM_E_INVALID_DEMAND, "destination != to(last edge) (trip %lld)", (long long)i);
    if (origin && destination && origin[i] == destination[i]) return fail(c, LPSIM_E_INVALID_DEMAND, "origin == destination (trip %lld)", (long long)i);
  }
  const int64_t R = n > 0 ? route_ptr[n] : 0;
  if (R >= (int64_t)0x7FFFFFF0ll) return fail(c, LPSIM_E_CAPACITY, "route entries exceed 2^31");
  const float dt = c->cfg.dt_s;
  tm.mark("validate demand");

  // ---- packed routes: edge | last << 31; departure steps (Q22); route visits per node ----
  std::unique_ptr<uint32_t[]> route_buf(new uint32_t[(size_t)std::max<int64_t>(R, 1)]);
  uint32_t* route = route_buf.get();
  std::vector<uint32_t> rstart((size_t)std::max<int64_t>(n, 1));
  std::vector<int64_t> dstep((size_t)std::max<int64_t>(n, 1));
  const int64_t NT = par_threads(n);
  std::vector<int64_t> tmax((size_t)NT, -1);
  // node weights for the partition ("route choice in a time window"): route visits, each
  // weighted by the free-flow time spent on the edge that enters the node, i.e. the vehicle-seconds
  // the node's tile will simulate (a visit to a 2 km freeway link costs ~20x a 100 m street link)
  std::vector<std::vector<double>> vis_t((size_t)NT);
  std::vector<double> tff((size_t)std::max(E, 1));
  for (int32_t e = 0; e < E; ++e) tff[e] = 1.0 + (double)c->ncells[e] / (double)c->v0[e];
  parallel_for(n, [&](int64_t a, int64_t b, int t) {
    std::vector<double>& w = vis_t[t];
    w.assign((size_t)NN, 0.0);
    for (int64_t i = a; i < b; ++i) {
      rstart[i] = (uint32_t)route_ptr[i];
      w[c->src[route_edges[route_ptr[i]]]] += 1.0;
      for (int64_t r = route_ptr[i]; r < route_ptr[i + 1]; ++r) {
        const int32_t e = route_edges[r];
        route[r] = (uint32_t)e | (r + 1 == route_ptr[i + 1] ? LAST_BIT : 0u);
        w[c->dst[e]] += tff[e];
      }
      dstep[i] = depart_step_of(depart_s[i], dt);
      tmax[t] = std::max(tmax[t], dstep[i]);
    }
  });
  std::vector<double> visits((size_t)NN, 0.0);
  for (auto& w : vis_t)
    for (int32_t u = 0; u < NN && !w.empty(); ++u) visits[u] += w[u];
  vis_t.clear();
  const int64_t max_step = n ? *std::max_element(tmax.begin(), tmax.end()) : 0;
  tm.mark("pack routes");
  if (max_step >= (int64_t)0xFFFFFFF0ll - 2) return fail(c, LPSIM_E_CAPACITY, "departure step exceeds 2^32");

  // ---- parts (§8(e)): route-weighted multilevel unless the caller gave one ----
  const int32_t K = c->K;
  c->part_of.assign((size_t)NN, 0);
  if (K > 1) {
    if (!c->node_part.empty()) {
      c->part_of = c->node_part;
    } else {
      lpsim_graph gg;
      std::memset(&gg, 0, sizeof(gg));
      gg.struct_size = sizeof(gg);
      gg.num_nodes = NN;
      gg.num_edges = E;
      gg.row_ptr = c->row_ptr.data();
      gg.dst = c->dst.data();
      gg.lanes = c->lanes.data();
      if (NN < 8 * K || lpsim_partition_multilevel(&gg, visits.data(), nullptr, K, 0.05, 1, c->part_of.data()) != LPSIM_OK)
        lpsim_partition_rcb(NN, c->node_xy.empty() ? nullptr : c->node_xy.data(), visits.data(), K, c->part_of.data());
    }
  }
  // ---- tiles: each part split into as many tiles as one GPU keeps resident (one CTA each) ----
  {
    const int32_t per_part = c->world > 1 ? c->max_tiles : std::max(1, c->max_tiles / K);
    std::vector<std::vector<int32_t>> nodes((size_t)K);
    for (int32_t u = 0; u < NN; ++u) nodes[c->part_of[u]].push_back(u);
    c->tile_of_node.assign((size_t)NN, 0);
    c->part_tile0.assign((size_t)K + 1, 0);
    c->tile_part.clear();
    std::vector<int32_t> lt;
    for (int32_t p = 0; p < K; ++p) {
      const int32_t nt = std::max<int32_t>(1, std::min<int32_t>(per_part, (int32_t)nodes[p].size()));
      tile_part_nodes(c, nodes[p], nt, visits, lt);
      // renumber densely (a partitioner may leave a tile empty)
      std::vector<int32_t> ren((size_t)nt, -1);
      int32_t used = 0;
      for (size_t i = 0; i < nodes[p].size(); ++i) {
        int32_t& r = ren[lt[i]];
        if (r < 0) r = used++;
      }
      const int32_t base = c->part_tile0[p];
      for (size_t i = 0; i < nodes[p].size(); ++i) c->tile_of_node[nodes[p][i]] = base + ren[lt[i]];
      c->part_tile0[p + 1] = base + std::max(used, 1);
      for (int32_t t = 0; t < std::max(used, 1); ++t) c->tile_part.push_back((uint8_t)p);
    }
    c->n_tiles = c->part_tile0[K];
  }
  const int32_t T = c->n_tiles;
  tm.mark("partition, tiles");
  auto tile_of_edge = [&](int32_t e) { return c->tile_of_node[c->dst[e]]; };
  auto tile_up = [&](int32_t e) { return c->tile_of_node[c->src[e]]; };
  // ---- neighbour tables: tiles joined by an edge, both directions ----
  std::vector<std::vector<int32_t>> nbl((size_t)T);
  for (int32_t e = 0; e < E; ++e) {
    const int32_t a = tile_up(e), b = tile_of_edge(e);
    if (a == b) continue;
    nbl[a].push_back(b);
    nbl[b].push_back(a);
  }
  std::vector<uint32_t> nb0((size_t)T + 1, 0);
  for (int32_t X = 0; X < T; ++X) {
    auto& v = nbl[X];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    if (v.size() > MAX_NB)
      return fail(c, LPSIM_E_CAPACITY, "tile %d has %zu neighbour tiles (max %u): use fewer tiles", X, v.size(), MAX_NB);
    nb0[X + 1] = nb0[X] + (uint32_t)v.size();
  }
  const uint32_t nbt = nb0[T];
  std::vector<uint32_t> nb_tile((size_t)std::max<uint32_t>(nbt, 1)), nb_back((size_t)std::max<uint32_t>(nbt, 1));
  auto nb_index = [&](int32_t X, int32_t N) -> uint32_t {  // position of N in X's list
    const auto& v = nbl[X];
    return (uint32_t)(std::lower_bound(v.begin(), v.end(), N) - v.begin());
  };
  for (int32_t X = 0; X < T; ++X)
    for (size_t i = 0; i < nbl[X].size(); ++i) {
      const int32_t N = nbl[X][i];
      nb_tile[nb0[X] + i] = (uint32_t)N;
      nb_back[nb0[X] + i] = nb0[N] + nb_index(N, X);
    }
  // channels: entry j of tile D for neighbour N holds the entrants of the edges N -> D (one per lane
  // and step at most: one vehicle per cell); offsets within D's part
  std::vector<uint32_t> ch_cap((size_t)std::max<uint32_t>(nbt, 1), 0), ch_off((size_t)std::max<uint32_t>(nbt, 1), 0);
  std::vector<uint32_t> li((size_t)std::max(E, 1), LI_SAME);
  for (int32_t e = 0; e < E; ++e) {
    const int32_t a = tile_up(e), b = tile_of_edge(e);
    if (a == b) continue;
    li[e] = nb_index(a, b);
    ch_cap[nb0[b] + nb_index(b, a)] += c->lanes[e];
  }
  std::vector<uint64_t> chan_part((size_t)K, 0);
  for (int32_t X = 0; X < T; ++X)
    for (uint32_t j = nb0[X]; j < nb0[X + 1]; ++j) {
      uint64_t& acc = chan_part[c->tile_part[X]];
      ch_off[j] = (uint32_t)acc;
      acc += ch_cap[j];
    }
  uint64_t chan_total = 1;
  for (uint64_t x : chan_part) chan_total = std::max(chan_total, x);
  if (chan_total >= 0x7FFFFFF0ull) return fail(c, LPSIM_E_CAPACITY, "channels too large");
  // edge ownership by part, mirrors of cut edges (§8(e))
  c->edge_opart.assign((size_t)std::max(E, 1), 0);
  std::vector<uint8_t> edge_mpart((size_t)std::max(E, 1), 0);
  for (int32_t e = 0; e < E; ++e) {
    const int32_t pa = c->tile_part[tile_up(e)], pb = c->tile_part[tile_of_edge(e)];
    c->edge_opart[e] = (uint8_t)pb;
    edge_mpart[e] = (uint8_t)pa;
    if (pa != pb) c->meta[e] |= META_MIRROR;
  }
  tm.mark("neighbours, channels");

  // ---- departure slots (A7): slot = (first edge, lane id mod lanes) on tile(from(first edge)) ----
  std::vector<uint64_t> slot_start_of_edge((size_t)E + 1, 0);
  for (int32_t e = 0; e < E; ++e) slot_start_of_edge[e + 1] = slot_start_of_edge[e] + c->lanes[e];
  std::vector<uint32_t> slot_of_key((size_t)std::max<uint64_t>(slot_start_of_edge[E], 1), NONE);
  std::vector<uint32_t> trip_slot((size_t)std::max<int64_t>(n, 1)), trip_rank((size_t)std::max<int64_t>(n, 1));
  std::vector<uint4> slot_a;
  std::vector<uint2> slot_b;
  std::vector<uint32_t> slot_n, slot_tile;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t e1 = route_edges[route_ptr[i]];
    const uint32_t l0 = (uint32_t)(i % c->lanes[e1]);
    const uint64_t key = slot_start_of_edge[e1] + l0;
    uint32_t sl = slot_of_key[key];
    if (sl == NONE) {
      sl = (uint32_t)slot_a.size();
      slot_of_key[key] = sl;
      slot_a.push_back(make_uint4((uint32_t)c->gbase[e1] + l0 * c->ncells[e1], 0, 0, 0));
      slot_b.push_back(make_uint2((uint32_t)e1 | (route_ptr[i + 1] - route_ptr[i] == 1 ? LAST_BIT : 0u),
                                  l0 | (li[e1] << 8)));
      slot_n.push_back(0);
      slot_tile.push_back((uint32_t)tile_up(e1));
    }
    trip_slot[i] = sl;
    trip_rank[i] = slot_n[sl]++;  // trips visited in id order: rank = order of ids
  }
  const uint32_t S = (uint32_t)slot_a.size();
  // slot_b's "last" bit is per trip, not per slot (two trips of one slot may have different route
  // lengths): the resolver takes the edge from it only for the digest, so keep the edge id alone
  for (auto& b : slot_b) b.x &= EDGE_MASK;
  uint64_t bm_words = 0;
  std::vector<uint32_t> soff((size_t)S + 1, 0);
  for (uint32_t q = 0; q < S; ++q) {
    if (bm_depth_host(slot_n[q]) > 4) return fail(c, LPSIM_E_CAPACITY, "more than 2^20 trips start on one (edge, lane) slot");
    soff[q + 1] = soff[q] + slot_n[q];
    slot_a[q].y = (uint32_t)bm_words;
    slot_a[q].z = slot_n[q];
    slot_a[q].w = soff[q];
    bm_words += bm_total_words(slot_n[q]);
  }
  if (bm_words >= 0xFFFFFFF0ull) return fail(c, LPSIM_E_CAPACITY, "departure bitmap too large");
  std::vector<uint32_t> strip((size_t)std::max<uint32_t>(soff[S], 1));
  parallel_for(n, [&](int64_t a, int64_t b, int) {
    for (int64_t i = a; i < b; ++i) strip[soff[trip_slot[i]] + trip_rank[i]] = (uint32_t)i;
  });
  // releases {slot, rank, step} grouped by tile, in step order: counting sort by step, then a stable
  // counting sort by tile
  std::vector<uint4> rel_step((size_t)std::max<int64_t>(n, 1));
  {
    const uint32_t ns = (uint32_t)max_step + 2;
    std::vector<uint32_t> cnt(ns + 1, 0);
    for (int64_t i = 0; i < n; ++i) cnt[dstep[i] + 1]++;
    for (uint32_t k = 0; k < ns; ++k) cnt[k + 1] += cnt[k];
    for (int64_t i = 0; i < n; ++i)
      rel_step[cnt[dstep[i]]++] = make_uint4(trip_slot[i], trip_rank[i], (uint32_t)dstep[i], (uint32_t)i);
  }
  std::vector<uint32_t> rel_tile0((size_t)T + 1, 0);
  c->rel_h.assign((size_t)std::max<int64_t>(n, 1), make_uint4(0, 0, 0, 0));
  {
    for (int64_t i = 0; i < n; ++i) rel_tile0[slot_tile[rel_step[i].x] + 1]++;
    for (int32_t X = 0; X < T; ++X) rel_tile0[X + 1] += rel_tile0[X];
    std::vector<uint32_t> pos(rel_tile0.begin(), rel_tile0.end() - 1);
    for (int64_t i = 0; i < n; ++i) c->rel_h[pos[slot_tile[rel_step[i].x]]++] = rel_step[i];
  }
  rel_step.clear();
  rel_step.shrink_to_fit();
  // pending-slot segments: the slots each tile owns
  std::vector<uint32_t> pcap((size_t)T, 0);
  for (uint32_t q = 0; q < S; ++q) pcap[slot_tile[q]]++;
  tm.mark("slots, releases");

  // ---- vehicle record capacity per tile: alive inputs + entrants of a step <= 2 x min(cells of the
  //      tile's edges, trips whose route visits the tile) ----
  std::vector<uint64_t> tcells((size_t)T, 0);
  for (int32_t e = 0; e < E; ++e) tcells[tile_of_edge(e)] += (uint64_t)c->lanes[e] * c->ncells[e];
  std::vector<std::vector<uint32_t>> touch_t((size_t)NT);
  parallel_for(n, [&](int64_t a, int64_t b, int t) {
    std::vector<uint32_t>& h = touch_t[t];
    h.assign((size_t)T, 0);
    for (int64_t i = a; i < b; ++i) {
      int32_t prev = -1;
      for (int64_t r = route_ptr[i]; r < route_ptr[i + 1]; ++r) {
        const int32_t X = tile_of_edge(route_edges[r]);
        if (X != prev) { h[X]++; prev = X; }
      }
    }
  });
  c->tinfo.assign((size_t)T, TileInfo{});
  uint64_t seg = 0, pseg = 0;
  for (int32_t X = 0; X < T; ++X) {
    uint64_t touch = 0;
    for (auto& h : touch_t) touch += h.empty() ? 0 : h[X];
    const uint64_t cap = std::min<uint64_t>(2 * tcells[X], 2 * touch) + 64;
    TileInfo& I = c->tinfo[X];
    I.seg = (uint32_t)seg;
    I.cap = (uint32_t)cap;
    I.pseg = (uint32_t)pseg;
    I.pcap = pcap[X];
    I.rel0 = rel_tile0[X];
    I.rel1 = rel_tile0[X + 1];
    I.nb0 = nb0[X];
    I.nnb = nb0[X + 1] - nb0[X];
    seg += cap;
    pseg += pcap[X];
    if (seg >= 0xFFFFFFF0ull) return fail(c, LPSIM_E_CAPACITY, "vehicle records exceed 2^32");
  }
  touch_t.clear();
  tm.mark("record capacities");

  // ---- device allocations and uploads ----
  lpsim_status s;
  const size_t nn = (size_t)std::max<int64_t>(n, 1);
  if ((s = upload(c, &c->d_route, route, (size_t)std::max<int64_t>(R, 1))) ||
      (s = upload(c, &c->d_trip_rstart, rstart.data(), nn)) || (s = dalloc(c, &c->d_arrival, nn)))
    return s;
  route_buf.reset();
  if (n) CU(cudaMemsetAsync(c->d_arrival, 0xFF, n * sizeof(int32_t), c->stream));
  c->r_total = R;
  if (c->P.flags & LPSIM_FLAG_EDGE_TIMES) {
    TRY(dalloc(c, &c->d_edge_entry, (size_t)std::max<int64_t>(R, 1)));
    CU(cudaMemsetAsync(c->d_edge_entry, 0xFF, (size_t)std::max<int64_t>(R, 1) * sizeof(int32_t), c->stream));
  }
  // edge records (a0 + ownership)
  uint32_t *d_li = nullptr, *d_meta = nullptr;
  if ((s = upload(c, &d_li, li.data(), (size_t)std::max(E, 1))) ||
      (s = upload(c, &d_meta, c->meta.data(), (size_t)std::max(E, 1))) || (s = dalloc(c, &c->d_edges, (size_t)std::max(E, 1))) ||
      (s = upload(c, &c->d_edge_mpart, edge_mpart.data(), edge_mpart.size())) ||
      (s = upload(c, &c->d_edge_opart, c->edge_opart.data(), c->edge_opart.size())))
    return s;
  if (E > 0)
    k_build_edges<<<grid_for(E), 256, 0, c->stream>>>(E, c->d_gbase, c->d_ncells, c->d_lanes, c->d_v0, d_li, d_meta,
                                                       c->d_edges);
  {
    std::vector<uint32_t> toe((size_t)std::max(E, 1), 0);
    for (int32_t e = 0; e < E; ++e) toe[e] = (uint32_t)tile_of_edge(e);
    TRY(upload(c, &c->d_tile_of_edge, toe.data(), toe.size()));
  }
  // tiles
  uint32_t *d_nb_tile = nullptr, *d_nb_back = nullptr, *d_ch_off = nullptr, *d_ch_cap = nullptr;
  if ((s = upload(c, &c->d_tinfo, c->tinfo.data(), (size_t)T)) || (s = dalloc(c, &c->d_tctl, (size_t)T)) ||
      (s = upload(c, &c->d_tile_part, c->tile_part.data(), (size_t)T)) ||
      (s = upload(c, &d_nb_tile, nb_tile.data(), nb_tile.size())) ||
      (s = upload(c, &d_nb_back, nb_back.data(), nb_back.size())) ||
      (s = upload(c, &d_ch_off, ch_off.data(), ch_off.size())) ||
      (s = upload(c, &d_ch_cap, ch_cap.data(), ch_cap.size())))
    return s;
  {
    std::vector<TileCtl> tc((size_t)T);
    std::memset(tc.data(), 0, tc.size() * sizeof(TileCtl));
    for (int32_t X = 0; X < T; ++X) tc[X].rel_cur = c->tinfo[X].rel0;
    CU(cudaMemcpyAsync(c->d_tctl, tc.data(), tc.size() * sizeof(TileCtl), cudaMemcpyHostToDevice, c->stream));
  }
  // parts: this process's memory (one part per process in multi-process mode, all of them otherwise)
  c->parts.assign((size_t)K, PartPtrs{});
  for (int32_t p = 0; p < K; ++p) {
    if (!c->is_local(p)) continue;
    PartPtrs& M = c->parts[p];
    for (int b = 0; b < 3; ++b) {
      TRY(dalloc(c, &M.map[b], c->total_cells + 64));  // +64: vector over-read pad
      k_fill_u8<<<grid_for(c->total_cells + 64), 256, 0, c->stream>>>(M.map[b], 255, c->total_cells + 64);
    }
    TRY(dalloc(c, &M.flag, 2 * (size_t)std::max<uint32_t>(nbt, 1)));
    CU(cudaMemsetAsync(M.flag, 0, 2 * (size_t)std::max<uint32_t>(nbt, 1) * sizeof(unsigned long long), c->stream));
    TRY(dalloc(c, &M.chan, 2 * (size_t)chan_total));
    TRY(dalloc(c, &M.ctx, nn));
  }
  TRY(dalloc(c, &c->d_parts, (size_t)K));
  // vehicle records (segments of the local tiles)
  const int32_t lt0 = c->t0(), lt1 = c->t1();
  const uint64_t rec0 = c->tinfo[lt0].seg, rec1 = lt1 < T ? c->tinfo[lt1].seg : seg;
  const uint64_t ps0 = c->tinfo[lt0].pseg, ps1 = lt1 < T ? c->tinfo[lt1].pseg : pseg;
  const size_t nrec = (size_t)std::max<uint64_t>(rec1 - rec0, 1), npend = (size_t)std::max<uint64_t>(ps1 - ps0, 1);
  Global& G = c->G;
  for (int b = 0; b < 2; ++b) {
    if ((s = dalloc(c, &G.rid[b], nrec)) || (s = dalloc(c, &G.rln[b], nrec)) || (s = dalloc(c, &G.rpos[b], nrec)) ||
        (s = dalloc(c, &G.rv[b], nrec)) || (s = dalloc(c, &G.rcell[b], nrec)) || (s = dalloc(c, &G.rpcell[b], nrec)) ||
        (s = dalloc(c, &G.rc4[b], nrec)) || (s = dalloc(c, &G.plist[b], npend)))
      return s;
    // the arrays are indexed with the global segment offsets of the tiles
    G.rid[b] -= rec0; G.rln[b] -= rec0; G.rpos[b] -= rec0; G.rv[b] -= rec0;
    G.rcell[b] -= rec0; G.rpcell[b] -= rec0; G.rc4[b] -= rec0; G.plist[b] -= ps0;
  }
  TRY(dalloc(c, &G.cl, nrec));
  G.cl -= rec0;
  TRY(dalloc(c, &G.adm, npend));
  G.adm -= ps0;
  // departures
  uint32_t* d_slot_trip = nullptr;
  uint4 *d_slot_a = nullptr, *d_rel = nullptr, *d_rinfo = nullptr;
  uint2 *d_slot_b = nullptr, *d_dep = nullptr;
  uint32_t *d_bm = nullptr, *d_nrel = nullptr, *d_cand = nullptr, *d_cid = nullptr;
  if (S == 0) {  // keep the uploads non-empty
    slot_a.push_back(make_uint4(0, 0, 0, 0));
    slot_b.push_back(make_uint2(0, 0));
  }
  if ((s = upload(c, &d_slot_a, slot_a.data(), slot_a.size())) ||
      (s = upload(c, &d_slot_b, slot_b.data(), slot_b.size())) ||
      (s = upload(c, &d_slot_trip, strip.data(), strip.size())) || (s = dalloc(c, &d_bm, (size_t)bm_words)) ||
      (s = dalloc(c, &d_nrel, (size_t)std::max<uint32_t>(S, 1))) ||
      (s = dalloc(c, &d_cand, (size_t)std::max<uint32_t>(S, 1))) ||
      (s = dalloc(c, &d_cid, (size_t)std::max<uint32_t>(S, 1))) ||
      (s = upload(c, &d_rel, c->rel_h.data(), c->rel_h.size())) || (s = dalloc(c, &d_dep, nn)) ||
      (s = dalloc(c, &d_rinfo, (size_t)std::max<int64_t>(R, 1))))
    return s;
  if (S) CU(cudaMemsetAsync(d_cid, 0xFF, S * sizeof(uint32_t), c->stream));
  if (R > 0) k_route_info<<<grid_for(R), 256, 0, c->stream>>>(c->d_route, c->d_edges, R, d_rinfo);
  if (bm_words) CU(cudaMemsetAsync(d_bm, 0, bm_words * sizeof(uint32_t), c->stream));
  if (S) CU(cudaMemsetAsync(d_nrel, 0, S * sizeof(uint32_t), c->stream));
  if (S) CU(cudaMemsetAsync(d_cand, 0xFF, S * sizeof(uint32_t), c->stream));
  tm.mark("device allocations, uploads");

  G.tile0 = (uint32_t)lt0;
  G.n_parts = (uint32_t)K;
  G.nbt = nbt;
  G.chan_total = (uint32_t)chan_total;
  G.world = (uint32_t)c->world;
  G.tinfo = c->d_tinfo;
  G.tctl = c->d_tctl;
  G.tile_part = c->d_tile_part;
  G.nb_tile = d_nb_tile;
  G.nb_back = d_nb_back;
  G.ch_off = d_ch_off;
  G.ch_cap = d_ch_cap;
  G.parts = c->d_parts;
  G.edges = c->d_edges;
  G.edge_mpart = c->d_edge_mpart;
  G.route = c->d_route;
  G.trip_rstart = c->d_trip_rstart;
  G.arrival_step = c->d_arrival;
  G.edge_entry = (c->P.flags & LPSIM_FLAG_EDGE_TIMES) ? c->d_edge_entry : nullptr;
  G.slot_a = d_slot_a;
  G.slot_b = d_slot_b;
  G.slot_trip = d_slot_trip;
  G.bm = d_bm;
  G.slot_nrel = d_nrel;
  G.slot_cand = d_cand;
  G.rel = d_rel;
  G.dep = d_dep;
  G.rinfo = d_rinfo;
  G.slot_cid = d_cid;
  G.digest_log = c->d_digest_log;
  G.digest_cap = c->digest_cap;
  G.err = c->d_err;
  TRY(upload_parts(c));
  // departure contexts of the trips (first edge) into the part that owns the first edge
  if (n > 0)
    k_trip_ctx<<<grid_for(n), 256, 0, c->stream>>>(c->d_edges, c->d_route, d_rinfo, c->d_trip_rstart,
                                                    c->d_edge_opart, c->d_parts, (unsigned)K, n, d_dep);
  c->trip_first_edge.resize(nn);
  for (int64_t i = 0; i < n; ++i) c->trip_first_edge[i] = (uint32_t)route_edges[route_ptr[i]];
  c->n_trips = n;
  CU(cudaStreamSynchronize(c->stream));
  CU(cudaGetLastError());
  tm.mark("device setup kernels");
  c->loaded = true;
  c->step = 0;
  return LPSIM_OK;
}

static lpsim_status check_device_error(lpsim_ctx* c) {
  ErrCtl e;
  CU(cudaMemcpy(&e, c->d_err, sizeof(e), cudaMemcpyDeviceToHost));
  if (e.error) {
    c->failed = true;
    if (e.error == ERR_CAPACITY)
      return fail(c, LPSIM_E_CAPACITY, "device capacity exceeded (site %u, step %u, tile %u)", e.info, e.step, e.tile);
    if (e.error == ERR_TIMEOUT)
      return fail(c, LPSIM_E_COMM, "neighbour tile %u made no progress (step %u, tile %u)", e.info, e.step, e.tile);
    return fail(c, LPSIM_E_INVARIANT, "invariant violated: two vehicles in cell %u (step %u, tile %u)", e.info, e.step,
                e.tile);
  }
  return LPSIM_OK;
}

static lpsim_status run_steps(lpsim_ctx* c, int64_t n) {
  Params P = c->P;
  unsigned long long k0 = (unsigned long long)c->step;
  unsigned ns = (unsigned)n;
  Global G = c->G;
  void* args[] = {&G, &P, &k0, &ns};
  const bool full = (P.flags & (LPSIM_FLAG_DIGESTS | LPSIM_FLAG_TIMING)) != 0u;
  void* fn = full ? (void*)k_tile_full : (void*)k_tile;
  const unsigned grid = (unsigned)(c->t1() - c->t0());
  CU(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(TILE_BS), args, tile_dyn_smem(), c->stream));
  c->launches += 1;
  return LPSIM_OK;
}

static lpsim_status occupancy(lpsim_ctx* c, unsigned which, unsigned long long* out);

lpsim_status lpsim_step(lpsim_ctx* c, int64_t n) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "lpsim_step before lpsim_load_demand");
  if (c->failed) return fail(c, LPSIM_E_STATE, "a previous device error left the context unusable: destroy it");
  if (n < 0) return fail(c, LPSIM_E_INVALID_ARG, "n < 0");
  if (c->world > 1 && !c->attached) return fail(c, LPSIM_E_STATE, "multi-process mode: lpsim_ipc_attach first");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  const bool digests = (c->P.flags & LPSIM_FLAG_DIGESTS) != 0;
  c->last_digests.clear();
  c->launches = 0;
  CU(cudaEventRecord(c->ev0, c->stream));
  int64_t done = 0;
  while (done < n) {
    int64_t chunk = n - done;
    if (digests) {
      chunk = std::min<int64_t>(chunk, c->digest_cap);
      CU(cudaMemsetAsync(c->d_digest_log, 0, chunk * sizeof(unsigned long long), c->stream));
    }
    chunk = std::min<int64_t>(chunk, 1 << 20);
    TRY(run_steps(c, chunk));
    if (digests) {
      std::vector<uint64_t> d((size_t)chunk);
      CU(cudaMemcpyAsync(d.data(), c->d_digest_log, chunk * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      c->last_digests.insert(c->last_digests.end(), d.begin(), d.end());
    }
    c->step += chunk;
    done += chunk;
  }
  CU(cudaEventRecord(c->ev1, c->stream));
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    c->failed = true;
    return fail(c, LPSIM_E_CUDA, "step failed: %s", cudaGetErrorString(e));
  }
  TRY(check_device_error(c));
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  c->last_step_ms = ms;
  if ((c->P.flags & LPSIM_FLAG_CHECKS) && c->world == 1) {
    // a7 invariant after the call: occupied cells of M_k == on-road vehicles, M_{k+1} clean
    unsigned long long occ[2] = {0, 0};
    TRY(occupancy(c, 0, &occ[0]));
    TRY(occupancy(c, 1, &occ[1]));
    lpsim_stats st;
    st.struct_size = sizeof(st);
    TRY(lpsim_stats_get(c, &st));
    if ((int64_t)occ[0] != st.on_road || occ[1] != 0) {
      c->failed = true;
      return fail(c, LPSIM_E_INVARIANT, "lane map holds %llu occupied cells for %lld on-road vehicles at step %lld "
                  "(%llu in the next buffer)", occ[0], (long long)st.on_road, (long long)c->step, occ[1]);
    }
  }
  return LPSIM_OK;
}

lpsim_status lpsim_set_flags(lpsim_ctx* c, uint32_t flags) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "lpsim_set_flags before lpsim_load_demand");
  if ((flags & LPSIM_FLAG_EDGE_TIMES) && !c->d_edge_entry)
    return fail(c, LPSIM_E_STATE, "LPSIM_FLAG_EDGE_TIMES must be set at lpsim_create");
  c->P.flags = flags;
  c->cfg.flags = flags;
  c->G.edge_entry = (flags & LPSIM_FLAG_EDGE_TIMES) ? c->d_edge_entry : nullptr;
  return LPSIM_OK;
}

lpsim_status lpsim_stats_get(lpsim_ctx* c, lpsim_stats* out) {
  if (!c || !out) return LPSIM_E_INVALID_ARG;
  if (out->struct_size != sizeof(lpsim_stats)) return fail(c, LPSIM_E_INVALID_ARG, "struct_size mismatch");
  lpsim_stats s;
  std::memset(&s, 0, sizeof(s));
  s.struct_size = sizeof(s);
  s.step = c->step;
  s.num_parts = (int64_t)c->K;
  s.device_bytes = c->device_bytes;
  s.step_ms = c->last_step_ms;
  s.kernel_launches = c->launches;
  s.tiles = c->loaded ? (int64_t)(c->t1() - c->t0()) : 0;
  if (c->loaded) {
    if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
    const int32_t t0 = c->t0(), t1 = c->t1();
    std::vector<TileCtl> tc((size_t)(t1 - t0));
    if (t1 > t0) CU(cudaMemcpy(tc.data(), c->d_tctl + t0, tc.size() * sizeof(TileCtl), cudaMemcpyDeviceToHost));
    unsigned long long tw = 0, tmv = 0, trs = 0, tst = 0;
    for (const TileCtl& x : tc) {
      s.updates += (int64_t)x.ctr[C_UPD];
      s.departures += (int64_t)x.ctr[C_DEP];
      s.transitions += (int64_t)x.ctr[C_TRANS];
      s.lane_changes += (int64_t)x.ctr[C_LC];
      s.arrivals += (int64_t)x.ctr[C_ARR];
      s.lost_claims += (int64_t)x.ctr[C_LOST];
      tw += x.t[0]; tmv += x.t[1]; trs += x.t[2]; tst = std::max(tst, x.t[3]);
    }
    // every departed trip is on the road until it arrives
    s.on_road = c->on_road_base + s.departures - s.arrivals;
    s.finished = s.arrivals;
    s.waiting = c->n_trips - s.on_road - s.finished;
    if (!tc.empty()) {  // LPSIM_FLAG_TIMING: mean per tile (ns), over the steps run with timing
      s.phase_ns[0] = (int64_t)(tw / tc.size());
      s.phase_ns[1] = (int64_t)(tmv / tc.size());
      s.phase_ns[2] = (int64_t)(trs / tc.size());
      s.exchange_ms = (double)(tw / tc.size()) / 1e6;
    }
    (void)tst;
    if (!c->last_digests.empty()) s.digest = c->last_digests.back();
  }
  *out = s;
  return LPSIM_OK;
}

lpsim_status lpsim_debug_block_times(lpsim_ctx* c, uint64_t* out, int64_t n) {
  if (!c || !out) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "no demand loaded");
  const int32_t t0 = c->t0(), t1 = c->t1();
  if (n != (int64_t)24 * (t1 - t0)) return fail(c, LPSIM_E_INVALID_ARG, "n must be 24 x %d", t1 - t0);
  std::vector<TileCtl> tc((size_t)(t1 - t0));
  CU(cudaMemcpy(tc.data(), c->d_tctl + t0, tc.size() * sizeof(TileCtl), cudaMemcpyDeviceToHost));
  std::memset(out, 0, (size_t)n * sizeof(uint64_t));
  for (size_t b = 0; b < tc.size(); ++b) {
    const TileInfo& I = c->tinfo[t0 + b];
    for (int w = 0; w < 4; ++w) out[24 * b + w] = tc[b].t[w];
    out[24 * b + 4] = tc[b].n[c->step & 1];
    out[24 * b + 5] = I.nnb;
    out[24 * b + 6] = I.cap;
    out[24 * b + 7] = tc[b].ctr[C_UPD];
  }
  return LPSIM_OK;
}

lpsim_status lpsim_digests(lpsim_ctx* c, uint64_t* out, int64_t n) {
  if (!c || (!out && n)) return LPSIM_E_INVALID_ARG;
  if ((size_t)n > c->last_digests.size()) return fail(c, LPSIM_E_INVALID_ARG, "only %zu digests recorded", c->last_digests.size());
  std::memcpy(out, c->last_digests.data(), (size_t)n * sizeof(uint64_t));
  return LPSIM_OK;
}

static lpsim_status trip_views(lpsim_ctx* c, int32_t* d_status, int32_t* d_edge, int32_t* d_lane, float* d_pos,
                               float* d_v, int64_t* d_cur) {
  const int64_t n = c->n_trips;
  // defaults: waiting (route[0], lane 0, 0, 0, 0); finished from the arrival array
  std::vector<int32_t> arr((size_t)std::max<int64_t>(n, 1));
  CU(cudaMemcpyAsync(arr.data(), c->d_arrival, n * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  std::vector<int32_t> st((size_t)std::max<int64_t>(n, 1)), ed((size_t)std::max<int64_t>(n, 1));
  for (int64_t i = 0; i < n; ++i) {
    st[i] = arr[i] >= 0 ? 2 : 0;
    ed[i] = (int32_t)c->trip_first_edge[i];
  }
  CU(cudaMemcpyAsync(d_status, st.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemcpyAsync(d_edge, ed.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemsetAsync(d_lane, 0, n * sizeof(int32_t), c->stream));
  CU(cudaMemsetAsync(d_pos, 0, n * sizeof(float), c->stream));
  CU(cudaMemsetAsync(d_v, 0, n * sizeof(float), c->stream));
  CU(cudaMemsetAsync(d_cur, 0, n * sizeof(int64_t), c->stream));
  const int32_t t0 = c->t0(), t1 = c->t1();
  if (t1 > t0)
    k_scatter_trips<<<std::min(t1 - t0, 148 * 4), 256, 0, c->stream>>>(c->G, (uint32_t)t0, (uint32_t)t1,
                                                                       (unsigned long long)c->step, d_status, d_edge,
                                                                       d_lane, d_pos, d_v, d_cur);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(c->stream));  // the host vectors above go out of scope
  return LPSIM_OK;
}

lpsim_status lpsim_trip_state(lpsim_ctx* c, int64_t n, int32_t* status, int32_t* edge, int32_t* lane, float* pos,
                              float* v, int64_t* cursor) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "no demand loaded");
  if (n != c->n_trips) return fail(c, LPSIM_E_INVALID_ARG, "num_trips mismatch");
  if (n == 0) return LPSIM_OK;
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  int32_t *ds = nullptr, *de = nullptr, *dl = nullptr;
  float *dp = nullptr, *dv = nullptr;
  int64_t* dc = nullptr;
  CU(cudaMalloc(&ds, n * 4)); CU(cudaMalloc(&de, n * 4)); CU(cudaMalloc(&dl, n * 4));
  CU(cudaMalloc(&dp, n * 4)); CU(cudaMalloc(&dv, n * 4)); CU(cudaMalloc(&dc, n * 8));
  lpsim_status s = trip_views(c, ds, de, dl, dp, dv, dc);
  if (s == LPSIM_OK) {
    if (status) cudaMemcpy(status, ds, n * 4, cudaMemcpyDeviceToHost);
    if (edge) cudaMemcpy(edge, de, n * 4, cudaMemcpyDeviceToHost);
    if (lane) cudaMemcpy(lane, dl, n * 4, cudaMemcpyDeviceToHost);
    if (pos) cudaMemcpy(pos, dp, n * 4, cudaMemcpyDeviceToHost);
    if (v) cudaMemcpy(v, dv, n * 4, cudaMemcpyDeviceToHost);
    if (cursor) cudaMemcpy(cursor, dc, n * 8, cudaMemcpyDeviceToHost);
  }
  cudaFree(ds); cudaFree(de); cudaFree(dl); cudaFree(dp); cudaFree(dv); cudaFree(dc);
  return s;
}

lpsim_status lpsim_restore(lpsim_ctx* c, int64_t step, int64_t n, const int32_t* status, const int32_t* edge,
                           const int32_t* lane, const float* pos, const float* v, const int64_t* cursor,
                           const int64_t* arrival_step, const int64_t* counters, const int32_t* edge_entry) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "lpsim_restore before lpsim_load_demand");
  if (c->step != 0 || c->restored || c->failed) return fail(c, LPSIM_E_STATE, "lpsim_restore needs a freshly loaded context");
  if (n != c->n_trips) return fail(c, LPSIM_E_INVALID_ARG, "num_trips mismatch");
  if (step < 0 || step >= (int64_t)0x7FFFFFF0ll) return fail(c, LPSIM_E_INVALID_ARG, "step out of range");
  if (n > 0 && (!status || !edge || !lane || !pos || !v || !cursor || !arrival_step))
    return fail(c, LPSIM_E_INVALID_ARG, "null array");
  if (edge_entry && !c->d_edge_entry) return fail(c, LPSIM_E_STATE, "edge entries given without LPSIM_FLAG_EDGE_TIMES");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  // host checks before any device write (first offending trip): status, arrival step, cursor within
  // the route and on the given edge, lane, position, speed
  std::vector<uint32_t> rstart((size_t)std::max<int64_t>(n, 1));
  CU(cudaMemcpy(rstart.data(), c->d_trip_rstart, (size_t)std::max<int64_t>(n, 1) * 4, cudaMemcpyDeviceToHost));
  std::vector<uint32_t> rte((size_t)std::max<int64_t>(c->r_total, 1));
  if (c->r_total) CU(cudaMemcpy(rte.data(), c->d_route, (size_t)c->r_total * 4, cudaMemcpyDeviceToHost));
  std::vector<int32_t> arr32((size_t)std::max<int64_t>(n, 1));
  int64_t on_road = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t st = status[i];
    if (st < 0 || st > 2) return fail(c, LPSIM_E_INVALID_ARG, "bad status (trip %lld)", (long long)i);
    if ((st == 2) != (arrival_step[i] >= 0) || arrival_step[i] > step)
      return fail(c, LPSIM_E_INVALID_ARG, "arrival step inconsistent with status (trip %lld)", (long long)i);
    arr32[i] = (int32_t)arrival_step[i];
    if (st == 1) {
      ++on_road;
      const int32_t e = edge[i];
      const int64_t rlen = (i + 1 < n ? (int64_t)rstart[i + 1] : c->r_total) - (int64_t)rstart[i];
      if (e < 0 || e >= c->n_edges || lane[i] < 0 || lane[i] >= c->lanes[e] || cursor[i] < 0 || cursor[i] >= rlen ||
          (int32_t)(rte[rstart[i] + cursor[i]] & ROUTE_EDGE_MASK) != e ||
          !(pos[i] >= 0.0f && pos[i] < (float)c->ncells[e]) || !(v[i] >= 0.0f && v[i] <= 254.0f))
        return fail(c, LPSIM_E_INVALID_ARG, "bad on-road state (trip %lld)", (long long)i);
    }
  }
  const unsigned cb = (unsigned)(step & 1), mk = (unsigned)(step % 3);
  int32_t *d_st = nullptr, *d_ed = nullptr, *d_ln = nullptr;
  float *d_pos = nullptr, *d_v = nullptr;
  int64_t* d_cur = nullptr;
  uint32_t* d_err = nullptr;
  const size_t nn = (size_t)std::max<int64_t>(n, 1);
  cudaError_t ce = cudaSuccess;
  auto cm = [&](void** p, size_t b) { if (ce == cudaSuccess) ce = cudaMalloc(p, b); };
  cm((void**)&d_st, nn * 4); cm((void**)&d_ed, nn * 4); cm((void**)&d_ln, nn * 4); cm((void**)&d_pos, nn * 4);
  cm((void**)&d_v, nn * 4); cm((void**)&d_cur, nn * 8); cm((void**)&d_err, 4);
  const int32_t t0 = c->t0(), t1 = c->t1();
  const unsigned local = c->world > 1 ? (unsigned)c->rank : 0xFFFFFFFFu;  // all parts are local in one process
  if (ce == cudaSuccess && n > 0) {
    cudaMemcpyAsync(d_st, status, n * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(d_ed, edge, n * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(d_ln, lane, n * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(d_pos, pos, n * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(d_v, v, n * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(d_cur, cursor, n * 8, cudaMemcpyHostToDevice, c->stream);
  }
  if (ce == cudaSuccess) {
    // tile state of snapshot `step`: empty lists and pending lists, release cursors at the first
    // release of a step >= `step`, neighbour flags "step done" with no migrants
    std::vector<TileCtl> tc((size_t)c->n_tiles);
    std::memset(tc.data(), 0, tc.size() * sizeof(TileCtl));
    for (int32_t X = 0; X < c->n_tiles; ++X) {
      const TileInfo& I = c->tinfo[X];
      uint32_t lo = I.rel0, hi = I.rel1;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) / 2;
        if (c->rel_h[mid].z < (uint32_t)step) lo = mid + 1; else hi = mid;
      }
      tc[X].rel_cur = lo;
    }
    cudaMemcpyAsync(c->d_tctl, tc.data(), tc.size() * sizeof(TileCtl), cudaMemcpyHostToDevice, c->stream);
    cudaMemsetAsync(d_err, 0xFF, 4, c->stream);
    for (int32_t p = 0; p < c->K; ++p) {
      if (!c->is_local(p)) continue;
      std::vector<unsigned long long> fl(2 * (size_t)std::max<uint32_t>(c->G.nbt, 1), 0ull);
      for (uint32_t j = 0; j < c->G.nbt; ++j) fl[(size_t)cb * c->G.nbt + j] = (unsigned long long)step << 32;
      cudaMemcpyAsync(c->parts[p].flag, fl.data(), fl.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                      c->stream);
      cudaStreamSynchronize(c->stream);
    }
    if (n > 0)
      k_restore_trips<<<grid_for(n), 256, 0, c->stream>>>(c->G, local, mk, cb, c->P.h_max, n, c->d_tile_of_edge, d_st,
                                                           d_ed, d_ln, d_pos, d_v, d_cur, d_err);
    if (t1 > t0)
      k_restore_released<<<std::min(t1 - t0, 148 * 4), 256, 0, c->stream>>>(c->G, (uint32_t)t0, (uint32_t)t1,
                                                                            (uint32_t)step, d_st);
    ce = cudaStreamSynchronize(c->stream);
  }
  uint32_t err = 0xFFFFFFFFu;
  if (ce == cudaSuccess) ce = cudaMemcpy(&err, d_err, 4, cudaMemcpyDeviceToHost);
  cudaFree(d_st); cudaFree(d_ed); cudaFree(d_ln); cudaFree(d_pos); cudaFree(d_v); cudaFree(d_cur); cudaFree(d_err);
  if (ce != cudaSuccess) {
    c->failed = true;
    return fail(c, LPSIM_E_CUDA, "restore failed: %s", cudaGetErrorString(ce));
  }
  if (err != 0xFFFFFFFFu) {  // not reached after the host checks; the device state is partial
    c->failed = true;
    return fail(c, LPSIM_E_CAPACITY, "restore: trip %u does not fit its tile", err);
  }
  // arrivals, t_start per route edge, counters (on the first local tile)
  if (n > 0) CU(cudaMemcpy(c->d_arrival, arr32.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice));
  if (edge_entry && c->r_total > 0)
    CU(cudaMemcpy(c->d_edge_entry, edge_entry, (size_t)c->r_total * sizeof(int32_t), cudaMemcpyHostToDevice));
  c->on_road_base = on_road;
  if (counters && (c->world == 1 || c->rank == 0)) {
    // {updates, departures, transitions, lane_changes, arrivals, lost_claims} -> ctr[C_*]
    unsigned long long ct[C_N];
    ct[C_UPD] = (unsigned long long)counters[0];
    ct[C_DEP] = (unsigned long long)counters[1];
    ct[C_TRANS] = (unsigned long long)counters[2];
    ct[C_LC] = (unsigned long long)counters[3];
    ct[C_ARR] = (unsigned long long)counters[4];
    ct[C_LOST] = (unsigned long long)counters[5];
    CU(cudaMemcpy((char*)(c->d_tctl + t0) + offsetof(TileCtl, ctr), ct, sizeof(ct), cudaMemcpyHostToDevice));
    c->on_road_base = on_road - (int64_t)(counters[1] - counters[4]);
  }
  c->step = step;
  c->restored = true;
  return LPSIM_OK;
}

lpsim_status lpsim_edge_entry_steps(lpsim_ctx* c, int64_t r_total, int32_t* out) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "no demand loaded");
  if (!c->d_edge_entry) return fail(c, LPSIM_E_STATE, "LPSIM_FLAG_EDGE_TIMES was not set at lpsim_create");
  if (r_total != c->r_total || (r_total > 0 && !out)) return fail(c, LPSIM_E_INVALID_ARG, "r_total mismatch");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  if (r_total) CU(cudaMemcpy(out, c->d_edge_entry, (size_t)r_total * sizeof(int32_t), cudaMemcpyDeviceToHost));
  return LPSIM_OK;
}

lpsim_status lpsim_results(lpsim_ctx* c, int64_t n, int64_t* arrival_step, double* arrival_time_s, double* distance_m) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "no demand loaded");
  if (n != c->n_trips) return fail(c, LPSIM_E_INVALID_ARG, "num_trips mismatch");
  if (n == 0) return LPSIM_OK;
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  std::vector<int32_t> arr((size_t)n);
  if (distance_m) {
    int32_t *ds = nullptr, *de = nullptr, *dl = nullptr;
    float *dp = nullptr, *dv = nullptr;
    int64_t* dc = nullptr;
    double* dd = nullptr;
    CU(cudaMalloc(&ds, n * 4)); CU(cudaMalloc(&de, n * 4)); CU(cudaMalloc(&dl, n * 4));
    CU(cudaMalloc(&dp, n * 4)); CU(cudaMalloc(&dv, n * 4)); CU(cudaMalloc(&dc, n * 8)); CU(cudaMalloc(&dd, n * 8));
    lpsim_status s = trip_views(c, ds, de, dl, dp, dv, dc);
    if (s == LPSIM_OK) {
      k_distances<<<grid_for(n), 256, 0, c->stream>>>(n, c->d_route, c->d_trip_rstart, c->d_length, ds, dp, dc,
                                                       c->d_arrival, dd);
      cudaStreamSynchronize(c->stream);
      cudaMemcpy(distance_m, dd, n * 8, cudaMemcpyDeviceToHost);
    }
    cudaFree(ds); cudaFree(de); cudaFree(dl); cudaFree(dp); cudaFree(dv); cudaFree(dc); cudaFree(dd);
    if (s != LPSIM_OK) return s;
  }
  CU(cudaMemcpy(arr.data(), c->d_arrival, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
  const double dt = (double)c->cfg.dt_s;
  for (int64_t i = 0; i < n; ++i) {
    if (arrival_step) arrival_step[i] = arr[i];
    if (arrival_time_s) arrival_time_s[i] = arr[i] >= 0 ? (double)arr[i] * dt : -1.0;
  }
  return LPSIM_OK;
}

int64_t lpsim_lane_map_size(const lpsim_ctx* c) { return c ? (int64_t)c->total_cells : -1; }

lpsim_status lpsim_lane_map(lpsim_ctx* c, uint8_t* out, int64_t size) {
  if (!c || !out) return LPSIM_E_INVALID_ARG;
  if (size != (int64_t)c->total_cells) return fail(c, LPSIM_E_INVALID_ARG, "size != lane map size");
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "no demand loaded");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  uint8_t* d = nullptr;
  CU(cudaMalloc(&d, std::max<int64_t>(size, 1)));
  CU(cudaMemsetAsync(d, 255, std::max<int64_t>(size, 1), c->stream));
  const int b = (int)(c->step % 3);
  for (int32_t p = 0; p < c->K; ++p)
    if (c->is_local(p))
      k_gather_map<<<std::max(1, std::min(c->n_edges, 148 * 8)), 256, 0, c->stream>>>(
          c->parts[p].map[b], c->d_edges, c->d_edge_opart, (unsigned)p, c->n_edges, d);
  cudaStreamSynchronize(c->stream);
  cudaError_t e = cudaMemcpy(out, d, size, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(c, LPSIM_E_CUDA, "lane map copy: %s", cudaGetErrorString(e));
  return LPSIM_OK;
}

// occupied cells of the owned edges of the local parts in M_{k+which}
static lpsim_status occupancy(lpsim_ctx* c, unsigned which, unsigned long long* out) {
  unsigned long long* d = nullptr;
  CU(cudaMalloc(&d, sizeof(unsigned long long)));
  CU(cudaMemsetAsync(d, 0, sizeof(unsigned long long), c->stream));
  for (int32_t p = 0; p < c->K; ++p)
    if (c->is_local(p))
      k_count_occupied<<<std::max(1, std::min(c->n_edges, 148 * 8)), 256, 0, c->stream>>>(
          c->parts[p].map[(c->step + which) % 3], c->d_edges, c->d_edge_opart, (unsigned)p, c->n_edges, d);
  cudaStreamSynchronize(c->stream);
  cudaError_t e = cudaMemcpy(out, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(c, LPSIM_E_CUDA, "occupancy copy: %s", cudaGetErrorString(e));
  return LPSIM_OK;
}

lpsim_status lpsim_debug_map_occupancy(lpsim_ctx* c, uint64_t* out) {
  if (!c || !out) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "lpsim_debug_map_occupancy before lpsim_load_demand");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  unsigned long long h[2] = {0, 0};
  TRY(occupancy(c, 0, &h[0]));
  TRY(occupancy(c, 1, &h[1]));
  out[0] = h[0];
  out[1] = h[1];
  return LPSIM_OK;
}

lpsim_status lpsim_debug_poke_map(lpsim_ctx* c, int64_t cell, uint8_t value) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "no demand loaded");
  if (cell < 0 || cell >= (int64_t)c->total_cells) return fail(c, LPSIM_E_INVALID_ARG, "cell out of range");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  for (int32_t p = 0; p < c->K; ++p)
    if (c->is_local(p)) CU(cudaMemcpy(c->parts[p].map[c->step % 3] + cell, &value, 1, cudaMemcpyHostToDevice));
  return LPSIM_OK;
}

lpsim_status lpsim_lane_map_base(lpsim_ctx* c, uint64_t* base, int64_t num_edges) {
  if (!c || (!base && num_edges)) return LPSIM_E_INVALID_ARG;
  if (num_edges != c->n_edges) return fail(c, LPSIM_E_INVALID_ARG, "num_edges mismatch");
  std::memcpy(base, c->gbase.data(), (size_t)num_edges * sizeof(uint64_t));
  return LPSIM_OK;
}

namespace {
struct IpcBlob {
  uint32_t magic, rank, world, n_tiles, nbt, chan_total;
  cudaIpcMemHandle_t map[3], flag, chan, ctx;
};
static_assert(sizeof(IpcBlob) <= LPSIM_IPC_BLOB_BYTES, "blob size");
constexpr uint32_t IPC_MAGIC = 0x4c505332u;  // "LPS2"
}  // namespace

lpsim_status lpsim_ipc_handle(lpsim_ctx* c, void* blob, int64_t size) {
  if (!c || !blob || size < LPSIM_IPC_BLOB_BYTES) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "lpsim_ipc_handle before lpsim_load_demand");
  if (c->world < 2) return fail(c, LPSIM_E_STATE, "not in multi-process mode");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  IpcBlob b;
  std::memset(&b, 0, sizeof(b));
  b.magic = IPC_MAGIC;
  b.rank = (uint32_t)c->rank;
  b.world = (uint32_t)c->world;
  b.n_tiles = (uint32_t)c->n_tiles;
  b.nbt = c->G.nbt;
  b.chan_total = c->G.chan_total;
  const PartPtrs& M = c->parts[c->rank];
  for (int i = 0; i < 3; ++i) CU(cudaIpcGetMemHandle(&b.map[i], M.map[i]));
  CU(cudaIpcGetMemHandle(&b.flag, M.flag));
  CU(cudaIpcGetMemHandle(&b.chan, M.chan));
  CU(cudaIpcGetMemHandle(&b.ctx, M.ctx));
  std::memset(blob, 0, LPSIM_IPC_BLOB_BYTES);
  std::memcpy(blob, &b, sizeof(b));
  return LPSIM_OK;
}

lpsim_status lpsim_ipc_attach(lpsim_ctx* c, const void* blobs, int64_t size) {
  if (!c || !blobs) return LPSIM_E_INVALID_ARG;
  if (!c->loaded || c->world < 2) return fail(c, LPSIM_E_STATE, "lpsim_ipc_attach needs multi-process mode after load");
  if (c->attached) return fail(c, LPSIM_E_STATE, "already attached");
  if (size != (int64_t)c->world * LPSIM_IPC_BLOB_BYTES) return fail(c, LPSIM_E_INVALID_ARG, "blob size != world x 512");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  for (int32_t q = 0; q < c->world; ++q) {
    IpcBlob b;
    std::memcpy(&b, (const char*)blobs + (size_t)q * LPSIM_IPC_BLOB_BYTES, sizeof(b));
    if (b.magic != IPC_MAGIC || (int32_t)b.rank != q || (int32_t)b.world != c->world)
      return fail(c, LPSIM_E_COMM, "bad IPC record for rank %d", q);
    if (q == c->rank) continue;
    if ((int32_t)b.n_tiles != c->n_tiles || b.nbt != c->G.nbt || b.chan_total != c->G.chan_total)
      return fail(c, LPSIM_E_COMM, "plan mismatch with rank %d (tiles / neighbour tables)", q);
    PartPtrs& M = c->parts[q];
    void* p = nullptr;
    for (int i = 0; i < 3; ++i) {
      CU(cudaIpcOpenMemHandle(&p, b.map[i], cudaIpcMemLazyEnablePeerAccess));
      c->ipc_opened.push_back(p);
      M.map[i] = (uint8_t*)p;
    }
    CU(cudaIpcOpenMemHandle(&p, b.flag, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    M.flag = (unsigned long long*)p;
    CU(cudaIpcOpenMemHandle(&p, b.chan, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    M.chan = (MigRec*)p;
    CU(cudaIpcOpenMemHandle(&p, b.ctx, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    M.ctx = (Ctx*)p;
  }
  TRY(upload_parts(c));
  c->attached = true;
  return LPSIM_OK;
}

void lpsim_destroy(lpsim_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* p : c->allocs) cudaFree(p);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

}  // extern "C"
