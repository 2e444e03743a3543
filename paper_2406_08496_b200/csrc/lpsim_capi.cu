// lpsim_capi.cu — host runtime behind the C ABI of include/lpsim.h.
//
// Validation, device allocation, the departure structures (A7), the launch of
// the persistent step kernel and the result / state queries.  Every step of
// the simulated method runs in the kernels of lpsim_step.cu; this file only
// prepares integer metadata (CSR ranks, slots, release order) and moves data.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstddef>
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

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
};

struct HostPart {
  PartDev d{};  // device pointers (host copy)
  PartCtl* ctl = nullptr;
  uint32_t* sort_bcount = nullptr;  // a9 bucket counts [sort_nb] (zero between sorts)
  uint32_t* sort_bcur = nullptr;    // bucket cursors [sort_nb]
  uint32_t* sort_bsum = nullptr;    // per-CTA segment sums [grid]
  uint32_t* sort_perm = nullptr;    // [veh_cap]
  uint32_t sort_nb = 0;
};

}  // namespace

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
  std::vector<uint64_t> gbase;  // global lane-map layout (a0), from the device builder
  uint64_t total_cells = 0;
  // device graph
  float* d_length = nullptr;
  uint8_t* d_lanes = nullptr;
  uint64_t* d_gbase = nullptr;
  EdgeRec* d_edges = nullptr;
  // demand
  bool loaded = false;
  int64_t n_trips = 0;
  uint32_t* d_route = nullptr;
  uint32_t* d_trip_rstart = nullptr;
  int32_t* d_arrival = nullptr;
  int32_t* d_edge_entry = nullptr;  // LPSIM_FLAG_EDGE_TIMES
  bool restored = false;            // lpsim_restore ran (once, on a freshly loaded context)
  bool failed = false;              // a device error left the state partial: the context is unusable
  int64_t r_total = 0;
  std::vector<uint32_t> meta;       // packed lanes | rank | out-degree per edge
  std::vector<float> node_xy;
  std::vector<int32_t> node_part;   // user partition (optional)
  std::vector<int32_t> part_of;     // partition in use
  // parts
  std::vector<HostPart> parts;
  PartDev* d_parts = nullptr;
  SortBufs* d_sortbufs = nullptr;  // a9 buffers of every partition (entries of other processes' partitions empty)
  bool parts_dirty = false;  // host copies of the descriptors changed (sort buffer swap) since the upload
  GridCtl* d_grid = nullptr;
  unsigned long long* d_digest_log = nullptr;
  uint32_t digest_cap = 4096;
  std::vector<uint64_t> last_digests;
  int64_t step = 0;
  int grid_blocks = 0;
  int sort_blocks = 0;  // cooperative grid of k_bucket_sort
  double last_step_ms = 0.0;
  int64_t device_bytes = 0;
  std::vector<void*> allocs;
  int64_t sort_counter = 0;
  int64_t launches = 0;  // own kernel launches in the last lpsim_step
  std::vector<cudaEvent_t> sort_ev;  // pairs around the sort launches of the last lpsim_step
  int sort_ev_used = 0;
  int64_t last_sort_ns = 0;
  unsigned long long* d_tblock = nullptr;  // LPSIM_FLAG_TIMING per-CTA phase times
  unsigned long long* d_ctr_block = nullptr;  // per-CTA event counters [grid][5]
  // multi-process mode
  int32_t rank = 0, world = 1;
  uint32_t* d_xflag = nullptr;        // [world] barrier flags written by the peers
  uint32_t** d_xflag_peer = nullptr;  // [world] peer flag pointers
  uint32_t* d_mig_cnt = nullptr;      // [2][K][K] migrant counts (Global::mig_cnt), K > 1
  uint32_t** d_mig_cnt_peer = nullptr;  // [world] the peers' copies
  bool attached = false;
  std::vector<void*> ipc_opened;      // peer mappings to close
  bool is_local(int32_t p) const { return world == 1 || p == rank; }
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

template <class T>
lpsim_status dalloc(lpsim_ctx* c, T** p, size_t count) {
  size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  cudaError_t e = cudaMalloc((void**)p, bytes);
  if (e != cudaSuccess) return fail(c, LPSIM_E_NOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
  c->allocs.push_back((void*)*p);
  c->device_bytes += (int64_t)bytes;
  return LPSIM_OK;
}

template <class T>
lpsim_status upload(lpsim_ctx* c, T** p, const T* h, size_t count) {
  lpsim_status s = dalloc(c, p, count);
  if (s != LPSIM_OK) return s;
  if (count) CU(cudaMemcpyAsync(*p, h, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  return LPSIM_OK;
}

int grid_for(size_t n, int bs = 256) {
  size_t g = (n + bs - 1) / bs;
  return (int)std::max<size_t>(1, std::min<size_t>(g, 148 * 16));
}

#define TRY(x)                        \
  do {                                \
    lpsim_status s_ = (x);            \
    if (s_ != LPSIM_OK) return s_;    \
  } while (0)

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

}  // namespace

// host-side preparation of the demand runs on all host cores: [0, n) split into contiguous ranges
static int64_t par_threads(int64_t n, int64_t grain = 65536) {
  const int64_t hw = std::max<int64_t>(1, (int64_t)std::thread::hardware_concurrency());
  return std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(hw, 64), n / grain));
}
template <class F>
static void parallel_for(int64_t n, F fn, int64_t grain = 65536) {
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

static lpsim_status upload_parts(lpsim_ctx* c) {
  std::vector<PartDev> v;
  for (auto& H : c->parts) v.push_back(H.d);
  CU(cudaMemcpyAsync(c->d_parts, v.data(), v.size() * sizeof(PartDev), cudaMemcpyHostToDevice, c->stream));
  c->parts_dirty = false;
  return LPSIM_OK;
}
// before a kernel that reads the device copy of the descriptors (a pageable upload waits for the
// stream, so the step loop defers it: a process with one partition passes its descriptor in the
// step kernel's parameters and never needs it while stepping)
static lpsim_status sync_parts(lpsim_ctx* c) { return c->parts_dirty ? upload_parts(c) : LPSIM_OK; }

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
    if (L > 16777000.0f) return bail(fail(c, LPSIM_E_CAPACITY, "length_m >= 2^24 m (index %d)", e));
    if (g->lanes[e] < 1 || g->lanes[e] > 63) return bail(fail(c, LPSIM_E_INVALID_GRAPH, "lanes not in 1..63 (index %d)", e));
    const float v = g->speed_limit_mps[e];
    if (!(v > 0.0f && v <= 254.0f)) return bail(fail(c, LPSIM_E_INVALID_GRAPH, "speed limit not in (0,254] (index %d)", e));
  }
  const lpsim_config& C = *cfg;
  if (!(C.dt_s > 0) || !(C.a > 0) || !(C.b > 0) || C.delta < 1 || C.h_min < 1 || !(C.x0 > 0) || C.num_parts < 1)
    return bail(fail(c, LPSIM_E_INVALID_ARG, "invalid parameter"));
  if (C.num_parts > 255) return bail(fail(c, LPSIM_E_INVALID_ARG, "num_parts > 255"));
  if (C.world < 1 || C.rank < 0 || C.rank >= C.world || C.world > 255)
    return bail(fail(c, LPSIM_E_INVALID_ARG, "rank / world out of range"));
  if (C.world > 1 && C.num_parts != 1 && C.num_parts != C.world)
    return bail(fail(c, LPSIM_E_INVALID_ARG, "multi-process mode: num_parts must be 1 or world"));
  c->cfg = C;
  c->rank = C.rank;
  c->world = C.world;
  if (C.world > 1) c->cfg.num_parts = C.world;  // one partition per process
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
  // Q30: cycle in steps, rounded in fp32 like the oracle; >= 2 steps (two phases)
  if (!(C.signal_cycle_s >= 0.0f) || !std::isfinite(C.signal_cycle_s))
    return bail(fail(c, LPSIM_E_INVALID_ARG, "signal_cycle_s must be >= 0"));
  P.sig_cycle = C.signal_cycle_s > 0.0f ? (int)std::floor(C.signal_cycle_s / C.dt_s + 0.5f) : 0;
  if (C.signal_cycle_s > 0.0f && P.sig_cycle < 2)
    return bail(fail(c, LPSIM_E_INVALID_ARG, "signal cycle shorter than two steps"));
  P.seed_lo = (uint32_t)(C.seed & 0xFFFFFFFFu);
  P.seed_hi = (uint32_t)(C.seed >> 32);
  P.flags = C.flags;

  // ---- device, stream ----
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0)
    return bail(fail(c, LPSIM_E_CUDA, "no CUDA device"));
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
  std::vector<uint32_t> meta(E);
  for (int32_t e = 0; e < E; ++e) {
    const int32_t u = c->src[e], w = c->dst[e];
    const uint32_t rank = (uint32_t)(e - c->row_ptr[u]);
    const uint32_t kout = (uint32_t)(c->row_ptr[w + 1] - c->row_ptr[w]);
    meta[e] = (uint32_t)c->lanes[e] | (rank << META_RANK_SHIFT) | (kout << META_KOUT_SHIFT);
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
      meta[e] |= META_SIG | (ph ? META_PHASE : 0u);
    }
  }
  uint64_t *d_cells = nullptr, *d_sums = nullptr, *d_total = nullptr;
  uint32_t *d_ncells = nullptr, *d_meta = nullptr;
  float* d_v0 = nullptr;
  if ((s = upload(c, &c->d_length, c->length.data(), E)) || (s = upload(c, &c->d_lanes, c->lanes.data(), E)) ||
      (s = upload(c, &d_v0, c->v0.data(), E)) || (s = upload(c, &d_meta, meta.data(), E)) ||
      (s = dalloc(c, &d_cells, E)) || (s = dalloc(c, &d_ncells, E)) || (s = dalloc(c, &c->d_gbase, E)) ||
      (s = dalloc(c, &d_sums, (E + SCAN_BLOCK - 1) / SCAN_BLOCK + 1)) || (s = dalloc(c, &d_total, 1)) ||
      (s = dalloc(c, &c->d_edges, E)))
    return bail(s);
  const int nsb = (E + SCAN_BLOCK - 1) / SCAN_BLOCK;
  if (E > 0) {
    k_edge_cells<<<grid_for(E), 256, 0, c->stream>>>(c->d_length, c->d_lanes, d_cells, d_ncells, E);
    k_scan_blocks<<<nsb, SCAN_BLOCK, 0, c->stream>>>(d_cells, c->d_gbase, d_sums, E);
    k_scan_sums<<<1, 32, 0, c->stream>>>(d_sums, nsb, d_total);
    k_scan_add<<<nsb, SCAN_BLOCK, 0, c->stream>>>(c->d_gbase, d_sums, E);
  } else {
    cudaMemsetAsync(d_total, 0, sizeof(uint64_t), c->stream);
  }
  cudaError_t ce = cudaMemcpyAsync(&c->total_cells, d_total, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(c->stream);
  if (ce != cudaSuccess) return bail(fail(c, LPSIM_E_CUDA, "lane-map builder failed: %s", cudaGetErrorString(ce)));
  if (c->total_cells >= 0xFFFFFFF0ull) return bail(fail(c, LPSIM_E_CAPACITY, "lane map exceeds 2^32 cells"));
  c->gbase.resize(E);
  if (E) cudaMemcpy(c->gbase.data(), c->d_gbase, sizeof(uint64_t) * E, cudaMemcpyDeviceToHost);
  if (E > 0) k_build_edges<<<grid_for(E), 256, 0, c->stream>>>(E, c->d_gbase, d_ncells, d_v0, d_meta, c->d_edges);

  // per-partition state (lane maps, claims, vehicles) is built by lpsim_load_demand,
  // once the route-weighted partition is known
  c->meta = meta;
  if (g->node_xy) c->node_xy.assign(g->node_xy, g->node_xy + 2 * (size_t)N);
  if (C.node_part) {
    c->node_part.assign(C.node_part, C.node_part + N);
    for (int32_t u = 0; u < N; ++u)
      if (c->node_part[u] < 0 || c->node_part[u] >= c->cfg.num_parts)
        return bail(fail(c, LPSIM_E_INVALID_ARG, "node_part out of range (node %d)", u));
  }
  if ((s = dalloc(c, &c->d_grid, 1))) return bail(s);
  {
    GridCtl g0;
    std::memset(&g0, 0, sizeof(g0));
    g0.err_step = 0xFFFFFFFFu;
    CU(cudaMemcpyAsync(c->d_grid, &g0, sizeof(g0), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  if ((s = dalloc(c, &c->d_digest_log, c->digest_cap))) return bail(s);
  CU(cudaStreamSynchronize(c->stream));

  int bpsm = 0, nsm = 0;
  int bpsm_full = 0;
  const size_t dyn = step_dyn_smem();
  CU(cudaFuncSetAttribute(k_run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  CU(cudaFuncSetAttribute(k_run_full, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  CU(cudaFuncSetAttribute(k_run_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  int bpsm_multi = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm, k_run, STEP_BS, dyn));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm_full, k_run_full, STEP_BS, dyn));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm_multi, k_run_multi, STEP_BS, dyn));
  bpsm = std::min(bpsm, std::min(bpsm_full, bpsm_multi));
  CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
  if (bpsm < 1) return bail(fail(c, LPSIM_E_CUDA, "step kernel cannot be resident"));
  c->grid_blocks = bpsm * nsm;
  if (const char* mb = std::getenv("LPSIM_MAX_BLOCKS")) {  // e.g. several processes sharing one GPU (tests)
    const int cap = std::atoi(mb);
    if (cap > 0) c->grid_blocks = std::min(c->grid_blocks, cap);
  }
  {
    int bps = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_bucket_sort, 256, 0));
    if (bps < 1) return bail(fail(c, LPSIM_E_CUDA, "sort kernel cannot be resident"));
    c->sort_blocks = std::min(bps * nsm, c->grid_blocks);  // <= grid_blocks: sort_bsum is sized by it
  }
  tm.mark("create (graph, lane maps)");
  if ((s = dalloc(c, &c->d_ctr_block, 5 * (size_t)c->grid_blocks))) return bail(s);
  CU(cudaMemsetAsync(c->d_ctr_block, 0, 5 * sizeof(unsigned long long) * (size_t)c->grid_blocks, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  *out = c;
  return LPSIM_OK;
}

lpsim_status lpsim_load_demand(lpsim_ctx* c, int64_t n, const double* depart_s, const int64_t* route_ptr,
                               const int32_t* route_edges, const int32_t* origin, const int32_t* destination) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (c->loaded) return fail(c, LPSIM_E_STATE, "demand already loaded");
  if (n < 0 || (n > 0 && (!depart_s || !route_ptr || !route_edges)))
    return fail(c, LPSIM_E_INVALID_ARG, "null array or negative size");
  if (n >= (int64_t)0xFFFFFFF0ll) return fail(c, LPSIM_E_CAPACITY, "too many trips");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  StageTimer tm;
  // ---- validation ----
  if (n > 0 && route_ptr[0] != 0) return fail(c, LPSIM_E_INVALID_DEMAND, "route_ptr[0] != 0 (trip 0)");
  auto trip_ok = [&](int64_t i) {
    if (!(depart_s[i] >= 0.0) || !std::isfinite(depart_s[i]) || route_ptr[i + 1] <= route_ptr[i]) return false;
    for (int64_t r = route_ptr[i]; r < route_ptr[i + 1]; ++r) {
      const int32_t e = route_edges[r];
      if (e < 0 || e >= c->n_edges) return false;
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
      if (e < 0 || e >= c->n_edges) return fail(c, LPSIM_E_INVALID_DEMAND, "route edge out of range (trip %lld)", (long long)i);
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

  // ---- departure steps (Q22); route offsets.  The route table (~1 GB at C4) goes to the device as
  // the caller's edge ids, uploaded by a helper thread while the host builds the tables below, and is
  // packed there (edge | last << 31, k_mark_last) ----
  std::vector<uint32_t> rstart((size_t)std::max<int64_t>(n, 1));
  std::vector<int64_t> dstep((size_t)std::max<int64_t>(n, 1));
  std::vector<int64_t> tmax(64, -1);
  parallel_for(n, [&](int64_t a, int64_t b, int t) {
    for (int64_t i = a; i < b; ++i) {
      rstart[i] = (uint32_t)route_ptr[i];
      dstep[i] = depart_step_of(depart_s[i], dt);
      tmax[t] = std::max(tmax[t], dstep[i]);
    }
  });
  const int64_t max_step = *std::max_element(tmax.begin(), tmax.end());
  {
    lpsim_status s0;
    if ((s0 = dalloc(c, &c->d_route, (size_t)std::max<int64_t>(R, 1))) ||
        (s0 = dalloc(c, &c->d_trip_rstart, (size_t)std::max<int64_t>(n, 1))))
      return s0;
  }
  // joined before any use of the device route table and on every return path
  struct Uploader {
    std::thread t;
    cudaError_t err = cudaSuccess;
    ~Uploader() { if (t.joinable()) t.join(); }
    cudaError_t join() { if (t.joinable()) t.join(); return err; }
  } up;
  up.t = std::thread([&] {
    cudaError_t e = cudaSetDevice(c->device);
    if (e == cudaSuccess && R > 0)
      e = cudaMemcpyAsync(c->d_route, route_edges, (size_t)R * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess && n > 0)
      e = cudaMemcpyAsync(c->d_trip_rstart, rstart.data(), (size_t)n * sizeof(uint32_t), cudaMemcpyHostToDevice,
                          c->stream);
    if (e == cudaSuccess && n > 0) {
      k_mark_last<<<grid_for(n), 256, 0, c->stream>>>(n, R, c->d_trip_rstart, c->d_route);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);  // (rstart is read by the copy)
    up.err = e;
  });
  tm.mark("pack routes");
  if (max_step >= (int64_t)0xFFFFFFF0ll - 2) return fail(c, LPSIM_E_CAPACITY, "departure step exceeds 2^32");
  // ---- partition (§8(e)): route-weighted multilevel unless the caller gave one ----
  const int32_t K = c->cfg.num_parts;
  const int32_t E = c->n_edges;
  if ((int64_t)n * K >= (int64_t)0xFFFFFFF0ll) return fail(c, LPSIM_E_CAPACITY, "too many trips x parts");
  c->part_of.assign((size_t)c->n_nodes, 0);
  if (K > 1) {
    if (!c->node_part.empty()) {
      c->part_of = c->node_part;
    } else {
      std::vector<double> w((size_t)c->n_nodes, 0.0);  // route visits
      for (int64_t i = 0; i < n; ++i) {
        w[c->src[route_edges[route_ptr[i]]]] += 1.0;
        for (int64_t r = route_ptr[i]; r < route_ptr[i + 1]; ++r) w[c->dst[route_edges[r]]] += 1.0;
      }
      // balanced multilevel k-way on the route-visit weights (§8(f) item 1): on C4 it
      // cuts 10-90x fewer lanes than RCB (tools/partition_compare.py); RCB for tiny graphs
      lpsim_graph gg;
      std::memset(&gg, 0, sizeof(gg));
      gg.struct_size = sizeof(gg);
      gg.num_nodes = c->n_nodes;
      gg.num_edges = E;
      gg.row_ptr = c->row_ptr.data();
      gg.dst = c->dst.data();
      gg.lanes = c->lanes.data();
      if (c->n_nodes < 8 * K ||
          lpsim_partition_multilevel(&gg, w.data(), nullptr, K, 0.05, 1, c->part_of.data()) != LPSIM_OK)
        lpsim_partition_rcb(c->n_nodes, c->node_xy.empty() ? nullptr : c->node_xy.data(), w.data(), K,
                            c->part_of.data());
    }
  }
  const int h_max = c->P.h_max;
  std::vector<uint32_t> Lc((size_t)std::max(E, 1));
  for (int32_t e = 0; e < E; ++e) Lc[e] = (uint32_t)std::ceil(c->length[e]);
  auto owner = [&](int32_t e) { return c->part_of[c->dst[e]]; };
  auto upstream = [&](int32_t e) { return c->part_of[c->src[e]]; };
  // ---- local lane-map layouts: owned edges (dst owned) then entry halos of cut out-edges ----
  std::vector<std::vector<uint64_t>> base((size_t)K, std::vector<uint64_t>((size_t)std::max(E, 1), 0));
  std::vector<uint64_t> cells((size_t)K, 0);
  for (int32_t p = 0; p < K; ++p) {
    uint64_t acc = 0;
    for (int32_t e = 0; e < E; ++e)
      if (owner(e) == p) {
        base[p][e] = K == 1 ? c->gbase[e] : acc;  // K = 1: the a0 layout built on the device
        acc += (uint64_t)c->lanes[e] * Lc[e];
      }
    if (K == 1) acc = c->total_cells;
    for (int32_t e = 0; e < E; ++e)
      if (upstream(e) == p && owner(e) != p) {
        base[p][e] = acc;
        acc += (uint64_t)c->lanes[e] * (uint64_t)h_max;
      }
    if (acc >= 0xFFFFFFF0ull) return fail(c, LPSIM_E_CAPACITY, "partition %d lane map exceeds 2^32 cells", p);
    cells[p] = acc;
  }
  // ---- exchange plan (§8(e)): receive queues with one region per sender (one slot per cut lane:
  // at most one vehicle enters a lane per step), the owner's cell 0 of each halo edge, the
  // upstream halo of each owned cut edge (its mirror) ----
  std::vector<std::vector<uint64_t>> ncut((size_t)K, std::vector<uint64_t>((size_t)K, 0));  // [sender][receiver]
  std::vector<std::vector<uint2>> halo_dst((size_t)K), mirror((size_t)K);
  if (K > 1)
    for (int32_t p = 0; p < K; ++p) {
      halo_dst[p].assign((size_t)std::max(E, 1), make_uint2(NONE, NONE));
      mirror[p].assign((size_t)std::max(E, 1), make_uint2(NONE, NONE));
    }
  for (int32_t e = 0; e < E; ++e) {
    const int32_t q = owner(e), p = upstream(e);
    if (p == q) continue;
    ncut[p][q] += c->lanes[e];
    halo_dst[p][e] = make_uint2((uint32_t)q, (uint32_t)base[q][e]);
    mirror[q][e] = make_uint2((uint32_t)p, (uint32_t)base[p][e]);
  }
  std::vector<std::vector<uint32_t>> rq_off((size_t)K, std::vector<uint32_t>((size_t)K + 1, 0));
  std::vector<std::vector<uint32_t>> send_off((size_t)K, std::vector<uint32_t>((size_t)K, 0));
  for (int32_t q = 0; q < K; ++q) {
    uint64_t acc = 0;
    for (int32_t u = 0; u < K; ++u) {
      rq_off[q][u] = (uint32_t)acc;
      send_off[u][q] = (uint32_t)acc;
      acc += u == q ? 0 : ncut[u][q];
    }
    if (acc >= (1u << 24)) return fail(c, LPSIM_E_CAPACITY, "too many cut lanes");
    rq_off[q][K] = (uint32_t)acc;
  }
  // ---- departure slots (A7): slot = (first edge, lane id mod lanes), on the origin's part ----
  std::vector<uint64_t> slot_start_of_edge((size_t)E + 1, 0);
  for (int32_t e = 0; e < E; ++e) slot_start_of_edge[e + 1] = slot_start_of_edge[e] + c->lanes[e];
  const uint64_t max_slots = slot_start_of_edge[E];
  std::vector<uint32_t> slot_of_key((size_t)std::max<uint64_t>(max_slots, 1), NONE);
  std::vector<uint32_t> trip_slot((size_t)std::max<int64_t>(n, 1)), trip_rank((size_t)std::max<int64_t>(n, 1));
  std::vector<std::vector<uint32_t>> slot_cell((size_t)K), slot_n((size_t)K);
  {
    // a trip's rank in its slot = the number of lower ids in the slot (id order, A9): per-thread key
    // counts over contiguous id ranges, an exclusive prefix over the threads per key, then each thread
    // numbers its own trips; slots are numbered per part in key (edge, lane) order
    std::vector<uint32_t> tkey((size_t)std::max<int64_t>(n, 1));
    const int64_t grain = std::max<int64_t>(65536, n / 16 + 1);  // <= 16 histograms of the key space
    std::vector<std::vector<uint32_t>> kh((size_t)par_threads(n, grain));
    parallel_for(n, [&](int64_t a, int64_t b, int t) {
      kh[t].assign((size_t)std::max<uint64_t>(max_slots, 1), 0u);
      for (int64_t i = a; i < b; ++i) {
        const int32_t e1 = route_edges[route_ptr[i]];
        const uint32_t key = (uint32_t)(slot_start_of_edge[e1] + (uint64_t)(i % c->lanes[e1]));
        tkey[i] = key;
        kh[t][key]++;
      }
    }, grain);
    std::vector<uint32_t> ktot((size_t)std::max<uint64_t>(max_slots, 1), 0u);
    parallel_for((int64_t)max_slots, [&](int64_t a, int64_t b, int) {
      for (int64_t key = a; key < b; ++key) {
        uint32_t run = 0;
        for (auto& h : kh) {
          const uint32_t x = h[key];
          h[key] = run;
          run += x;
        }
        ktot[key] = run;
      }
    });
    for (int32_t e = 0; e < E; ++e) {
      const int32_t p = upstream(e);
      const uint32_t stride = owner(e) == p ? Lc[e] : (uint32_t)h_max;
      for (uint32_t l0 = 0; l0 < c->lanes[e]; ++l0) {
        const uint64_t key = slot_start_of_edge[e] + l0;
        if (!ktot[key]) continue;
        slot_of_key[key] = (uint32_t)slot_cell[p].size();
        slot_cell[p].push_back((uint32_t)base[p][e] + l0 * stride);
        slot_n[p].push_back(ktot[key]);
      }
    }
    parallel_for(n, [&](int64_t a, int64_t b, int t) {
      for (int64_t i = a; i < b; ++i) {
        const uint32_t key = tkey[i];
        trip_slot[i] = slot_of_key[key];
        trip_rank[i] = kh[t][key]++;  // trips of this range in id order after the lower ranges'
      }
    }, grain);
  }
  tm.mark("partition, layout, slots");
  const uint32_t rel_steps = (uint32_t)(max_step + 1);
  c->parts.assign((size_t)K, HostPart());
  lpsim_status s;
  if ((s = dalloc(c, &c->d_arrival, (size_t)std::max<int64_t>(n, 1)))) return s;
  if (n) CU(cudaMemsetAsync(c->d_arrival, 0xFF, n * sizeof(int32_t), c->stream));
  c->r_total = R;
  if (c->P.flags & LPSIM_FLAG_EDGE_TIMES) {
    if ((s = dalloc(c, &c->d_edge_entry, (size_t)std::max<int64_t>(R, 1)))) return s;
    CU(cudaMemsetAsync(c->d_edge_entry, 0xFF, (size_t)std::max<int64_t>(R, 1) * sizeof(int32_t), c->stream));
  }
  std::vector<int32_t> trip_part((size_t)std::max<int64_t>(n, 1), 0);  // partition of each trip's origin
  if (K > 1)
    parallel_for(n, [&](int64_t a, int64_t b, int) {
      for (int64_t i = a; i < b; ++i) trip_part[i] = upstream(route_edges[route_ptr[i]]);
    });
  // visit runs of the trips per part: a trip counts once per maximal run of its route on the part's
  // edges (its departure counts on the origin's part)
  std::vector<uint64_t> touch((size_t)K, 0);
  if (K == 1) {
    touch[0] = (uint64_t)n;
  } else {
    std::vector<std::vector<uint64_t>> th((size_t)par_threads(n), std::vector<uint64_t>((size_t)K, 0));
    parallel_for(n, [&](int64_t a, int64_t b, int t) {
      for (int64_t i = a; i < b; ++i) {
        int32_t prev = trip_part[i];
        th[t][prev]++;
        for (int64_t r = route_ptr[i]; r < route_ptr[i + 1]; ++r) {
          const int32_t q = owner(route_edges[r]);
          if (q != prev) { th[t][q]++; prev = q; }
        }
      }
    });
    for (auto& v : th)
      for (int32_t q = 0; q < K; ++q) touch[q] += v[q];
  }
  tm.mark("upload routes");
  for (int32_t p = 0; p < K; ++p) {
    HostPart& H = c->parts[p];
    PartDev& D = H.d;
    D.n_in = rq_off[p][K];  // plan data, known for every partition
    if (!c->is_local(p)) continue;  // simulated by another process; peer pointers come from lpsim_ipc_attach
    const uint32_t S = (uint32_t)slot_cell[p].size();
    // edge records of this part's view (a0; META_HALO / META_REMOTE)
    std::vector<EdgeRec> er((size_t)std::max(E, 1));
    for (int32_t e = 0; e < E; ++e) {
      EdgeRec& r = er[e];
      r.base = (uint32_t)base[p][e];
      r.ncells = Lc[e];
      r.v0 = c->v0[e];
      r.meta = c->meta[e];
      if (owner(e) != p) r.meta |= (upstream(e) == p) ? META_HALO : META_REMOTE;
      else if (upstream(e) != p) r.meta |= META_MIRROR;
    }
    std::vector<uint32_t> soff(S + 1, 0), sbm(S + 1, 0);
    uint64_t bm_words = 0;
    for (uint32_t q = 0; q < S; ++q) {
      soff[q + 1] = soff[q] + slot_n[p][q];
      sbm[q] = (uint32_t)bm_words;
      bm_words += bm_total_words(slot_n[p][q]);
    }
    if (bm_words >= 0xFFFFFFF0ull) return fail(c, LPSIM_E_CAPACITY, "departure bitmap too large");
    for (uint32_t q = 0; q < S; ++q)  // the step kernel's departure search handles bitmaps up to 4 levels
      if (bm_depth_host(slot_n[p][q]) > 4)
        return fail(c, LPSIM_E_CAPACITY, "more than 2^20 trips start on one (edge, lane) slot");
    // trips of this part: slot members in id order (each trip writes its own entry), releases in
    // depart-step order (stable counting sort with per-thread histograms), all on the host cores
    tm.mark("  part: edge records, slot offsets");
    std::vector<uint32_t> strip((size_t)std::max<uint32_t>(soff[S], 1));
    const int64_t NT = par_threads(n);
    std::vector<std::vector<uint32_t>> hist((size_t)NT, std::vector<uint32_t>(rel_steps + 1, 0));
    parallel_for(n, [&](int64_t a, int64_t b, int t) {
      for (int64_t i = a; i < b; ++i) {
        if (trip_part[i] != p) continue;
        strip[soff[trip_slot[i]] + trip_rank[i]] = (uint32_t)i;
        hist[t][dstep[i]]++;
      }
    });
    std::vector<uint32_t> rel_ptr(rel_steps + 2, 0);
    uint64_t np_trips = 0;
    for (uint32_t k = 0; k <= rel_steps; ++k) {
      rel_ptr[k] = (uint32_t)np_trips;
      for (int64_t t = 0; t < NT; ++t) {  // hist becomes each thread's write offset
        const uint32_t h = hist[t][k];
        hist[t][k] = (uint32_t)np_trips;
        np_trips += h;
      }
    }
    rel_ptr[rel_steps + 1] = rel_ptr[rel_steps];
    tm.mark("  part: slot members, release histogram");
    std::vector<uint4> rel4((size_t)std::max<uint64_t>(np_trips, 1));
    parallel_for(n, [&](int64_t a, int64_t b, int t) {
      for (int64_t i = a; i < b; ++i) {
        if (trip_part[i] != p) continue;
        const uint32_t q = trip_slot[i];
        rel4[hist[t][dstep[i]]++] = make_uint4(q, trip_rank[i], sbm[q], slot_n[p][q]);
      }
    });
    // per slot {entry cell, bitmap offset, width, trip offset}; per step the distinct released slots
    // with the lowest rank released (two passes over step ranges, thread-local "seen at step" marks)
    tm.mark("  part: release list");
    std::vector<uint4> sinfo((size_t)std::max<uint32_t>(S, 1));
    for (uint32_t q = 0; q < S; ++q) sinfo[q] = make_uint4(slot_cell[p][q], sbm[q], slot_n[p][q], soff[q]);
    std::vector<uint32_t> rs_ptr(rel_steps + 2, 0), rs_cnt(rel_steps + 1, 0);
    parallel_for(rel_steps, [&](int64_t ka, int64_t kb, int) {
      std::vector<uint32_t> seen_at((size_t)std::max<uint32_t>(S, 1), NONE);
      for (int64_t k = ka; k < kb; ++k)
        for (uint32_t j = rel_ptr[k]; j < rel_ptr[k + 1]; ++j) {
          const uint32_t q = rel4[j].x;
          if (seen_at[q] != (uint32_t)k) { seen_at[q] = (uint32_t)k; rs_cnt[k]++; }
        }
    }, 512);
    uint32_t max_rs = 0;
    for (uint32_t k = 0; k < rel_steps; ++k) {
      rs_ptr[k + 1] = rs_ptr[k] + rs_cnt[k];
      max_rs = std::max(max_rs, rs_cnt[k]);
    }
    rs_ptr[rel_steps + 1] = rs_ptr[rel_steps];
    const size_t nrs = std::max<size_t>(rs_ptr[rel_steps], 1);
    std::vector<uint32_t> rs_slot(nrs, 0);
    std::vector<uint4> rs_info(nrs, make_uint4(0, 0, 0, 0));
    std::vector<uint2> rs_cand(nrs, make_uint2(NONE, NONE));  // lowest rank released at the step, its trip id
    std::vector<uint32_t> rs_r2(nrs, NONE);                   // second lowest rank released at the step
    parallel_for(rel_steps, [&](int64_t ka, int64_t kb, int) {
      std::vector<uint32_t> seen_at((size_t)std::max<uint32_t>(S, 1), NONE), pos_of((size_t)std::max<uint32_t>(S, 1));
      for (int64_t k = ka; k < kb; ++k) {
        uint32_t pos = rs_ptr[k];
        for (uint32_t j = rel_ptr[k]; j < rel_ptr[k + 1]; ++j) {
          const uint32_t q = rel4[j].x, r = rel4[j].y;
          if (seen_at[q] == (uint32_t)k) {
            uint2& m = rs_cand[pos_of[q]];
            uint32_t& m2 = rs_r2[pos_of[q]];
            if (r < m.x) {
              m2 = m.x;
              m = make_uint2(r, strip[soff[q] + r]);
            } else if (r < m2) {
              m2 = r;
            }
            continue;
          }
          seen_at[q] = (uint32_t)k;
          pos_of[q] = pos;
          rs_slot[pos] = q;
          rs_info[pos] = sinfo[q];
          rs_cand[pos] = make_uint2(r, strip[soff[q] + r]);
          ++pos;
        }
      }
    }, 512);
    tm.mark("  part: released slots per step");
    uint64_t owned_cells = 0;
    for (int32_t e = 0; e < E; ++e)
      if (owner(e) == p) owned_cells += (uint64_t)c->lanes[e] * Lc[e];
    // SoA capacity: live entries (<= cells, <= trips visiting the part) plus the dead entries left
    // between two compactions (a9) by trips that arrived or moved to another part (<= visit runs)
    const uint64_t cap = std::min<uint64_t>(touch[p], owned_cells) + touch[p] + 64;
    const uint32_t nin = rq_off[p][K];
    // sharded lists: a shard holds ~2x its fair share (pushes are spread by work index)
    const uint32_t slot_shcap = (uint32_t)std::min<uint64_t>(S, 2 * ((uint64_t)S + NSH - 1) / NSH + 64);
    tm.mark("  part: host tables");
    EdgeRec* d_er = nullptr;
    if ((s = upload(c, &d_er, er.data(), (size_t)std::max(E, 1))) ||
        (s = upload(c, (uint4**)&D.slot_info, sinfo.data(), sinfo.size())) ||
        (s = upload(c, (uint32_t**)&D.slot_trip, strip.data(), strip.size())) ||
        (s = dalloc(c, &D.bm, bm_words)) || (s = dalloc(c, &D.slot_list[0], (size_t)NSH * slot_shcap)) ||
        (s = dalloc(c, &D.slot_list[1], (size_t)NSH * slot_shcap)) ||
        (s = dalloc(c, &D.slot_li[0], (size_t)NSH * slot_shcap)) ||
        (s = dalloc(c, &D.slot_li[1], (size_t)NSH * slot_shcap)) ||
        (s = dalloc(c, &D.slot_lc[0], (size_t)NSH * slot_shcap)) ||
        (s = dalloc(c, &D.slot_lc[1], (size_t)NSH * slot_shcap)) ||
        (s = dalloc(c, &D.slot_cw, (size_t)std::max<uint32_t>(S, 1))) ||
        (s = dalloc(c, &D.slot_nrel, (size_t)std::max<uint32_t>(S, 1))) ||
        (s = dalloc(c, &D.slot_relk, (size_t)std::max<uint32_t>(S, 1))) ||
        (s = dalloc(c, &D.slot_cand, (size_t)NSH * slot_shcap + max_rs)) ||
        (s = dalloc(c, &D.slot_ci, (size_t)NSH * slot_shcap + max_rs)) ||
        (s = upload(c, (uint2**)&D.rs_cand, rs_cand.data(), rs_cand.size())) ||
        (s = upload(c, (uint32_t**)&D.rs_r2, rs_r2.data(), rs_r2.size())) ||
        (s = dalloc(c, (uint4**)&D.slot_cs, (size_t)NSH * slot_shcap + max_rs)) ||
        (s = upload(c, (uint32_t**)&D.rs_ptr, rs_ptr.data(), rs_ptr.size())) ||
        (s = upload(c, (uint32_t**)&D.rs_slot, rs_slot.data(), rs_slot.size())) ||
        (s = upload(c, (uint4**)&D.rs_info, rs_info.data(), rs_info.size())) ||
        (s = dalloc(c, &D.tel, (size_t)std::max<int64_t>(n, 1))) || (s = dalloc(c, &D.tx[0], (size_t)std::max<int64_t>(n, 1))) ||
        (s = dalloc(c, &D.tx[1], (size_t)std::max<int64_t>(n, 1))) || (s = dalloc(c, &D.tx[2], (size_t)std::max<int64_t>(n, 1))) ||
        (s = dalloc(c, &D.tx[3], (size_t)std::max<int64_t>(n, 1))) || (s = dalloc(c, &D.tx[4], (size_t)std::max<int64_t>(n, 1))) ||
        (s = dalloc(c, &D.tx[5], (size_t)std::max<int64_t>(n, 1))) ||
        (s = dalloc(c, &D.sh_slot[0], NSH * SH_STRIDE)) || (s = dalloc(c, &D.sh_slot[1], NSH * SH_STRIDE)) ||
        (s = dalloc(c, &D.cbits[0], cap / 32 + 2)) || (s = dalloc(c, &D.cbits[1], cap / 32 + 2)) ||
        (s = upload(c, (uint4**)&D.rel4, rel4.data(), rel4.size())) ||
        (s = upload(c, (uint32_t**)&D.rel_ptr, rel_ptr.data(), rel_ptr.size())) ||
        (s = dalloc(c, &D.inq[0], 2 * (size_t)std::max<uint32_t>(nin, 1))) ||
        (s = upload(c, (uint32_t**)&D.rq_off, rq_off[p].data(), rq_off[p].size())) ||
        (s = upload(c, (uint32_t**)&D.send_off, send_off[p].data(), send_off[p].size())) ||
        (K > 1 && (s = upload(c, (uint2**)&D.halo_dst, halo_dst[p].data(), halo_dst[p].size()))) ||
        (K > 1 && (s = upload(c, (uint2**)&D.mirror, mirror[p].data(), mirror[p].size()))) ||
        (s = dalloc(c, &D.claim, cells[p])) || (s = dalloc(c, &H.ctl, 1)))
      return s;
    tm.mark("  part: uploads + allocs");
    D.edges = d_er;
    D.ncells = (uint32_t)cells[p];
    D.n_in = nin;
    D.inq[1] = D.inq[0] + std::max<uint32_t>(nin, 1);
    D.halo_lo = (uint32_t)cells[p];  // owned cells first, then the entry halos
    for (int32_t e = 0; e < E; ++e)
      if (upstream(e) == p && owner(e) != p) D.halo_lo = std::min(D.halo_lo, (uint32_t)base[p][e]);
    for (int b = 0; b < 2; ++b) {
      if ((s = dalloc(c, &D.map[b], cells[p] + 64))) return s;  // +64: vector over-read pad
      k_fill_u8<<<grid_for(cells[p] + 64), 256, 0, c->stream>>>(D.map[b], 255, cells[p] + 64);
    }
    k_fill_u32<<<grid_for(cells[p]), 256, 0, c->stream>>>(D.claim, NONE, cells[p]);
    for (int b = 0; b < 2; ++b) {
      const uint64_t capp = cap + 16;  // the step kernel's TMA staging reads up to 3 entries past the count
      if ((s = dalloc(c, &D.vid[b], capp)) || (s = dalloc(c, &D.vel[b], capp)) || (s = dalloc(c, &D.vpos[b], capp)) ||
          (s = dalloc(c, &D.vv[b], capp)) || (s = dalloc(c, &D.vcur[b], capp)) || (s = dalloc(c, &D.vpcell[b], capp)) ||
          (s = dalloc(c, &D.vcell[b], capp)) || (s = dalloc(c, &D.crec[b], capp)) || (s = dalloc(c, &D.xc0[b], capp)) ||
          (s = dalloc(c, &D.xv0[b], capp)) || (s = dalloc(c, &D.xc2[b], capp)) || (s = dalloc(c, &D.xc3[b], capp)) ||
          (s = dalloc(c, &D.xc4[b], capp)) || (s = dalloc(c, &D.xrn[b], capp)))
        return s;
    }
    tm.mark("  part: maps, SoA allocs");
    D.veh_cap = (uint32_t)cap;
    D.slot_shcap = std::max<uint32_t>(slot_shcap, 1);
    D.n_slot_total = S;
    D.rel_steps = rel_steps;
    D.ctl = H.ctl;
    CU(cudaMemsetAsync(H.ctl, 0, sizeof(PartCtl), c->stream));
    if (bm_words) CU(cudaMemsetAsync(D.bm, 0, bm_words * sizeof(uint32_t), c->stream));
    if (S) CU(cudaMemsetAsync(D.slot_relk, 0xFF, S * sizeof(uint32_t), c->stream));
    if (S) CU(cudaMemsetAsync(D.slot_cw, 0xFF, S * sizeof(uint2), c->stream));  // every slot empty
    if (S) CU(cudaMemsetAsync(D.slot_nrel, 0, S * sizeof(uint32_t), c->stream));
    for (int b = 0; b < 2; ++b) {
      CU(cudaMemsetAsync(D.sh_slot[b], 0, NSH * SH_STRIDE * sizeof(uint32_t), c->stream));
    }
    {
      // buckets cover the cells (locality) and the SoA indices (compaction-only mode)
      const uint64_t nb = (std::max<uint64_t>(cells[p], cap) >> SORT_SHIFT) + 1;
      H.sort_nb = (uint32_t)nb;
      if ((s = dalloc(c, &H.sort_bcount, nb)) || (s = dalloc(c, &H.sort_bcur, nb)) ||
          (s = dalloc(c, &H.sort_bsum, (size_t)c->grid_blocks)) || (s = dalloc(c, &H.sort_perm, cap)))
        return s;
      CU(cudaMemsetAsync(H.sort_bcount, 0, nb * sizeof(uint32_t), c->stream));
    }
  }
  if ((s = dalloc(c, &c->d_parts, c->parts.size()))) return s;
  {
    std::vector<SortBufs> sb(c->parts.size());
    for (size_t p = 0; p < c->parts.size(); ++p) {
      const HostPart& H = c->parts[p];
      sb[p] = SortBufs{H.sort_bcount, H.sort_bcur, H.sort_bsum, H.sort_perm, H.sort_nb, 0u};
    }
    if ((s = dalloc(c, &c->d_sortbufs, sb.size()))) return s;
    CU(cudaMemcpyAsync(c->d_sortbufs, sb.data(), sb.size() * sizeof(SortBufs), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));  // (sb is a host temporary)
  }
  tm.mark("  part: sort buffers");
  TRY(upload_parts(c));
  if (up.join() != cudaSuccess) return fail(c, LPSIM_E_CUDA, "route upload failed: %s", cudaGetErrorString(up.err));
  // departure state of each trip on its origin partition (a kernel; the edge context needs the local layout)
  for (int32_t p = 0; p < K; ++p) {
    if (!c->is_local(p)) continue;
    std::vector<uint32_t> own;
    for (int64_t i = 0; i < n; ++i)
      if (trip_part[i] == p) own.push_back((uint32_t)i);
    if (own.empty()) continue;
    uint32_t* d_own = nullptr;
    if ((s = upload(c, &d_own, own.data(), own.size()))) return s;
    k_trip_ctx<<<grid_for(own.size()), 256, 0, c->stream>>>(c->d_parts, (unsigned)p, c->d_route, c->d_trip_rstart, d_own,
                                                             (uint32_t)own.size(), h_max);
  }
  c->n_trips = n;
  if (c->world > 1) {
    if ((s = dalloc(c, &c->d_xflag, (size_t)c->world)) || (s = dalloc(c, &c->d_xflag_peer, (size_t)c->world)) ||
        (s = dalloc(c, &c->d_mig_cnt_peer, (size_t)c->world)))
      return s;
    CU(cudaMemsetAsync(c->d_xflag, 0, c->world * sizeof(uint32_t), c->stream));
  }
  if (K > 1) {
    if ((s = dalloc(c, &c->d_mig_cnt, 2 * (size_t)K * K))) return s;
    CU(cudaMemsetAsync(c->d_mig_cnt, 0, 2 * (size_t)K * K * sizeof(uint32_t), c->stream));
  }
  tm.mark("per-partition setup + upload");
  // releases (depart step k) are applied by the step kernel in phase A of step k
  CU(cudaStreamSynchronize(c->stream));
  tm.mark("device setup kernels");
  c->loaded = true;
  c->step = 0;
  return LPSIM_OK;
}

static lpsim_status run_steps(lpsim_ctx* c, int64_t n, bool digests) {
  Global G{};
  G.route = c->d_route;
  G.trip_rstart = c->d_trip_rstart;
  G.arrival_step = c->d_arrival;
  G.edge_entry = (c->P.flags & LPSIM_FLAG_EDGE_TIMES) ? c->d_edge_entry : nullptr;
  G.digest_log = c->d_digest_log;
  G.digest_cap = c->digest_cap;
  G.n_parts = (uint32_t)c->parts.size();
  G.part0 = c->world > 1 ? (uint32_t)c->rank : 0u;
  G.n_local = c->world > 1 ? 1u : (uint32_t)c->parts.size();
  G.world = (uint32_t)c->world;
  G.rank = (uint32_t)c->rank;
  G.xflag_local = c->d_xflag;
  G.xflag_peer = c->d_xflag_peer;
  G.mig_cnt = c->d_mig_cnt;
  G.mig_cnt_peer = c->d_mig_cnt_peer;
  G.parts = c->d_parts;
  G.grid = c->d_grid;
  G.ctr_block = c->d_ctr_block;
  Params P = c->P;
  unsigned long long k0 = (unsigned long long)c->step;
  unsigned ns = (unsigned)n;
  if (G.n_local > 1u) TRY(sync_parts(c));  // the step kernel reads G.parts[part]
  PartParam PP{};
  PP.mk = (uint32_t)(k0 & 1ull);
  if (G.n_local == 1u) {
    PP.valid = 1u;
    PP.d = c->parts[G.part0].d;
  }
  void* args[] = {&G, &P, &PP, &k0, &ns};
  // the instrumented instantiation only when digests or timing are requested
  const bool full = (P.flags & (LPSIM_FLAG_DIGESTS | LPSIM_FLAG_TIMING)) != 0u;
  void* fn = full ? (void*)k_run_full : G.n_parts > 1u ? (void*)k_run_multi : (void*)k_run;
  CU(cudaLaunchCooperativeKernel(fn, dim3(c->grid_blocks), dim3(STEP_BS), args, step_dyn_smem(), c->stream));
  c->launches += 1;
  (void)digests;
  return LPSIM_OK;
}

static lpsim_status check_device_error(lpsim_ctx* c) {
  GridCtl g;
  CU(cudaMemcpy(&g, c->d_grid, sizeof(g), cudaMemcpyDeviceToHost));
  if (g.error) {
    PartCtl pc;
    std::memset(&pc, 0, sizeof(pc));
    for (auto& H : c->parts)
      if (H.ctl) { CU(cudaMemcpy(&pc, H.ctl, sizeof(pc), cudaMemcpyDeviceToHost)); if (pc.error) break; }
    c->failed = true;  // the state of the failed step is partial
    if (g.error == ERR_CAPACITY) return fail(c, LPSIM_E_CAPACITY, "device capacity exceeded (site %u, step %u)", pc.error_info, g.err_step);
    if (g.error == ERR_TIMEOUT) return fail(c, LPSIM_E_COMM, "no progress of a peer GPU (step %u)", g.err_step);
    return fail(c, LPSIM_E_INVARIANT, "invariant violated at step %u: a second vehicle written into occupied cell %u "
                "of M_{k+1} (P:L248)", g.err_step, pc.error_info);
  }
  return LPSIM_OK;
}

// a9: periodic locality sort of the active SoA by lane-map cell (radix sort)
// a9: periodic locality sort of the active SoA by lane-map cell (radix sort);
// dead entries (vehicles that left) get the largest key and are cut off, so
// the sort is also the compaction.  With LPSIM_FLAG_NO_SORT only the
// compaction runs (a 1-bit stable sort: live first, order kept).
static lpsim_status sort_vehicles_launch(lpsim_ctx* c, bool locality);
// a9 with its device time recorded (an event pair per sort of the call)
static lpsim_status sort_vehicles(lpsim_ctx* c, bool locality) {
  if ((size_t)c->sort_ev_used + 2 > c->sort_ev.size()) {
    for (int i = 0; i < 2; ++i) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      c->sort_ev.push_back(e);
    }
  }
  CU(cudaEventRecord(c->sort_ev[c->sort_ev_used], c->stream));
  TRY(sort_vehicles_launch(c, locality));
  CU(cudaEventRecord(c->sort_ev[c->sort_ev_used + 1], c->stream));
  c->sort_ev_used += 2;
  return LPSIM_OK;
}

static lpsim_status sort_vehicles_launch(lpsim_ctx* c, bool locality) {
  // the process's partitions in one cooperative kernel (CTAs split among them; one launch per
  // partition when they would get fewer than 8 CTAs each); the counts stay on the device (no host
  // round trip).  The kernel reads the descriptors from the device copy: current before the launch.
  const unsigned buf = (unsigned)(c->step & 1);
  unsigned mode = locality ? 0u : 1u;
  unsigned p0 = c->world > 1 ? (unsigned)c->rank : 0u;
  const unsigned nl = c->world > 1 ? 1u : (unsigned)c->parts.size();
  TRY(sync_parts(c));
  const unsigned per = nl * 8u <= (unsigned)c->sort_blocks ? nl : 1u;  // partitions per launch
  for (unsigned q = 0; q < nl; q += per) {
    unsigned pq = p0 + q;
    unsigned nq = per;
    void* args[] = {&c->d_parts, &c->d_sortbufs, &pq, &nq, (void*)&buf, &mode};
    CU(cudaLaunchCooperativeKernel((void*)k_bucket_sort, dim3(c->sort_blocks), dim3(256), args, 0, c->stream));
    c->launches += 1;
  }
  bool any = false;
  for (size_t p = 0; p < c->parts.size(); ++p) {
    HostPart& H = c->parts[p];
    if (!H.ctl) continue;  // a partition of another process
    // the sorted copy lives in buffer buf^1: swap the buffer roles
    PartDev& Dh = H.d;
    std::swap(Dh.vid[0], Dh.vid[1]);
    std::swap(Dh.vel[0], Dh.vel[1]);
    std::swap(Dh.vpos[0], Dh.vpos[1]);
    std::swap(Dh.vv[0], Dh.vv[1]);
    std::swap(Dh.vcur[0], Dh.vcur[1]);
    std::swap(Dh.vpcell[0], Dh.vpcell[1]);
    std::swap(Dh.vcell[0], Dh.vcell[1]);
    Dh.xb ^= 1u;  // the gathered context lives in the other context buffer
    any = true;
  }
  if (any) c->parts_dirty = true;
  CU(cudaGetLastError());
  return LPSIM_OK;
}

lpsim_status lpsim_step(lpsim_ctx* c, int64_t n) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "lpsim_step before lpsim_load_demand");
  if (c->failed) return fail(c, LPSIM_E_STATE, "a previous device error left the context unusable: destroy it");
  if (n < 0) return fail(c, LPSIM_E_INVALID_ARG, "n < 0");
  if (c->world > 1 && !c->attached) return fail(c, LPSIM_E_STATE, "multi-process mode: lpsim_ipc_attach first");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  const bool digests = (c->P.flags & LPSIM_FLAG_DIGESTS) != 0;
  const bool sorting = (c->P.flags & LPSIM_FLAG_NO_SORT) == 0;
  const int64_t sort_every = c->cfg.sort_every > 0 ? c->cfg.sort_every : 256;
  c->last_digests.clear();
  c->launches = 0;
  c->sort_ev_used = 0;
  if (c->P.flags & LPSIM_FLAG_TIMING) {
    unsigned long long z[4] = {0, 0, 0, 0};
    CU(cudaMemcpyAsync((char*)c->d_grid + offsetof(GridCtl, t_phase), z, sizeof(z), cudaMemcpyHostToDevice, c->stream));
    if (!c->d_tblock) {
      lpsim_status s2 = dalloc(c, &c->d_tblock, TB_N * (size_t)c->grid_blocks);
      if (s2 != LPSIM_OK) return s2;
      CU(cudaMemcpyAsync((char*)c->d_grid + offsetof(GridCtl, t_block), &c->d_tblock, sizeof(void*),
                         cudaMemcpyHostToDevice, c->stream));
    }
    CU(cudaMemsetAsync(c->d_tblock, 0, TB_N * sizeof(unsigned long long) * (size_t)c->grid_blocks, c->stream));
  }
  CU(cudaEventRecord(c->ev0, c->stream));
  int64_t done = 0;
  while (done < n) {
    int64_t chunk = n - done;
    if (digests) chunk = std::min<int64_t>(chunk, c->digest_cap);
    chunk = std::min<int64_t>(chunk, sort_every - (c->step % sort_every));
    chunk = std::min<int64_t>(chunk, 1 << 20);
    TRY(run_steps(c, chunk, digests));
    if (digests) {
      std::vector<uint64_t> d((size_t)chunk);
      CU(cudaMemcpyAsync(d.data(), c->d_digest_log, chunk * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      c->last_digests.insert(c->last_digests.end(), d.begin(), d.end());
    }
    c->step += chunk;
    done += chunk;
    if (c->step % sort_every == 0) TRY(sort_vehicles(c, sorting));
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
  c->last_sort_ns = 0;
  for (int i = 0; i + 1 < c->sort_ev_used; i += 2) {
    float sm = 0.0f;
    cudaEventElapsedTime(&sm, c->sort_ev[i], c->sort_ev[i + 1]);
    c->last_sort_ns += (int64_t)(sm * 1e6);
  }
  if ((c->P.flags & LPSIM_FLAG_CHECKS) && c->world == 1) {
    // a7 after the call: the occupied cells of M_k are the on-road
    // vehicles, the other buffer is clean
    uint64_t occ[2] = {0, 0};
    TRY(lpsim_debug_map_occupancy(c, occ));
    lpsim_stats st;
    st.struct_size = sizeof(st);
    TRY(lpsim_stats_get(c, &st));
    if ((int64_t)occ[0] != st.on_road || occ[1] != 0) {
      c->failed = true;
      return fail(c, LPSIM_E_INVARIANT, "invariant violated at step %lld: M_k holds %llu occupied cells for %lld "
                  "on-road vehicles, the other lane map %llu", (long long)c->step, (unsigned long long)occ[0],
                  (long long)st.on_road, (unsigned long long)occ[1]);
    }
  }
  return LPSIM_OK;
}

lpsim_status lpsim_debug_poke_map(lpsim_ctx* c, int64_t cell, uint8_t value) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "no demand loaded");
  if (c->parts.size() != 1) return fail(c, LPSIM_E_STATE, "lpsim_debug_poke_map needs a single-partition context");
  if (cell < 0 || cell >= (int64_t)c->total_cells) return fail(c, LPSIM_E_INVALID_ARG, "cell out of range");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  CU(cudaMemcpyAsync(c->parts[0].d.map[c->step & 1] + cell, &value, 1, cudaMemcpyHostToDevice, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return LPSIM_OK;
}

lpsim_status lpsim_set_flags(lpsim_ctx* c, uint32_t flags) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "lpsim_set_flags before lpsim_load_demand");
  if ((flags & LPSIM_FLAG_EDGE_TIMES) && !c->d_edge_entry)
    return fail(c, LPSIM_E_STATE, "LPSIM_FLAG_EDGE_TIMES must be set at lpsim_create");
  c->P.flags = flags;
  c->cfg.flags = flags;
  return LPSIM_OK;
}

lpsim_status lpsim_stats_get(lpsim_ctx* c, lpsim_stats* out) {
  if (!c || !out) return LPSIM_E_INVALID_ARG;
  if (out->struct_size != sizeof(lpsim_stats)) return fail(c, LPSIM_E_INVALID_ARG, "struct_size mismatch");
  lpsim_stats s;
  std::memset(&s, 0, sizeof(s));
  s.struct_size = sizeof(s);
  s.step = c->step;
  s.num_parts = (int64_t)c->parts.size();
  s.device_bytes = c->device_bytes;
  s.step_ms = c->last_step_ms;
  s.kernel_launches = c->launches;
  s.sort_ns = c->last_sort_ns;
  if (c->loaded && (c->P.flags & LPSIM_FLAG_TIMING)) {
    GridCtl g;
    CU(cudaMemcpy(&g, c->d_grid, sizeof(g), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 3; ++i) s.phase_ns[i] = (int64_t)g.t_phase[i];
    s.exchange_ms = (double)g.t_phase[2] / 1e6;
  }
  if (c->loaded) {
    if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
    const unsigned buf = (unsigned)(c->step & 1);
    const int64_t K = (int64_t)c->parts.size();
    std::vector<uint32_t> mc;
    if (K > 1) {  // migrants in the receive queues of snapshot k are on the road (§8(e))
      mc.resize((size_t)(K * K));
      CU(cudaMemcpy(mc.data(), c->d_mig_cnt + (size_t)buf * K * K, mc.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    }
    for (int64_t p = 0; p < K; ++p) {
      HostPart& H = c->parts[p];
      if (!H.ctl) continue;
      PartCtl pc;
      CU(cudaMemcpy(&pc, H.ctl, sizeof(pc), cudaMemcpyDeviceToHost));
      for (int64_t u = 0; u < K && K > 1; ++u)
        if (u != p) s.on_road += (int64_t)mc[(size_t)(u * K + p)];
      s.on_road += (int64_t)pc.n_veh[buf] - (int64_t)pc.n_dead[buf];
      s.soa_entries += (int64_t)pc.n_veh[buf];
      s.updates += (int64_t)pc.updates;
      s.departures += (int64_t)pc.departures;
      s.transitions += (int64_t)pc.transitions;
      s.lane_changes += (int64_t)pc.lane_changes;
      s.arrivals += (int64_t)pc.arrivals;
      s.lost_claims += (int64_t)pc.lost_claims;
    }
    {
      std::vector<unsigned long long> cb(5 * (size_t)c->grid_blocks);
      CU(cudaMemcpy(cb.data(), c->d_ctr_block, cb.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      for (int b = 0; b < c->grid_blocks; ++b) {
        s.transitions += (int64_t)cb[5 * b + 0];
        s.lane_changes += (int64_t)cb[5 * b + 1];
        s.lost_claims += (int64_t)cb[5 * b + 2];
        s.departures += (int64_t)cb[5 * b + 3];
        s.arrivals += (int64_t)cb[5 * b + 4];
      }
    }
    s.finished = s.arrivals;
    s.waiting = c->n_trips - s.on_road - s.finished;
    if (!c->last_digests.empty()) s.digest = c->last_digests.back();
  }
  *out = s;
  return LPSIM_OK;
}

lpsim_status lpsim_debug_block_times(lpsim_ctx* c, uint64_t* out, int64_t n) {
  if (!c || !out) return LPSIM_E_INVALID_ARG;
  if (!c->d_tblock) return fail(c, LPSIM_E_STATE, "run lpsim_step with LPSIM_FLAG_TIMING first");
  if (n != (int64_t)TB_N * c->grid_blocks) return fail(c, LPSIM_E_INVALID_ARG, "n must be 24 x %d", c->grid_blocks);
  CU(cudaMemcpy(out, c->d_tblock, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
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
  // defaults on the device: waiting (route[0], lane 0, 0, 0, 0); finished from the arrival array
  if (n > 0)
    k_trip_defaults<<<grid_for(n), 256, 0, c->stream>>>(n, c->d_arrival, c->d_route, c->d_trip_rstart, d_status,
                                                         d_edge, d_lane, d_pos, d_v, d_cur);
  const unsigned buf = (unsigned)(c->step & 1);
  TRY(sync_parts(c));
  k_scatter_trips<<<grid_for(n), 256, 0, c->stream>>>(c->d_parts, (unsigned)c->parts.size(), buf, c->d_mig_cnt,
                                                       c->d_trip_rstart, d_status, d_edge, d_lane, d_pos, d_v, d_cur);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(c->stream));
  return LPSIM_OK;
}

lpsim_status lpsim_trip_state(lpsim_ctx* c, int64_t n, int32_t* status, int32_t* edge, int32_t* lane, float* pos,
                              float* v, int64_t* cursor) {
  if (!c) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "no demand loaded");
  if (n != c->n_trips) return fail(c, LPSIM_E_INVALID_ARG, "num_trips mismatch");
  if (n == 0) return LPSIM_OK;
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  int32_t *ds, *de, *dl;
  float *dp, *dv;
  int64_t* dc;
  CU(cudaMalloc(&ds, n * 4)); CU(cudaMalloc(&de, n * 4)); CU(cudaMalloc(&dl, n * 4));
  CU(cudaMalloc(&dp, n * 4)); CU(cudaMalloc(&dv, n * 4)); CU(cudaMalloc(&dc, n * 8));
  lpsim_status s = trip_views(c, ds, de, dl, dp, dv, dc);
  if (s == LPSIM_OK) {
    cudaStreamSynchronize(c->stream);
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
  // the trip's route and on the given edge, lane, position, speed
  std::vector<uint32_t> rstart((size_t)std::max<int64_t>(n, 1));
  std::vector<uint32_t> rte((size_t)std::max<int64_t>(c->r_total, 1));
  if (n) CU(cudaMemcpyAsync(rstart.data(), c->d_trip_rstart, (size_t)n * 4, cudaMemcpyDeviceToHost, c->stream));
  if (c->r_total) CU(cudaMemcpyAsync(rte.data(), c->d_route, (size_t)c->r_total * 4, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  std::vector<int32_t> arr32((size_t)std::max<int64_t>(n, 1));
  for (int64_t i = 0; i < n; ++i) {
    const int32_t st = status[i];
    if (st < 0 || st > 2) return fail(c, LPSIM_E_INVALID_ARG, "bad status (trip %lld)", (long long)i);
    if ((st == 2) != (arrival_step[i] >= 0) || arrival_step[i] > step)
      return fail(c, LPSIM_E_INVALID_ARG, "arrival step inconsistent with status (trip %lld)", (long long)i);
    arr32[i] = (int32_t)arrival_step[i];
    if (st == 1) {
      const int32_t e = edge[i];
      const int64_t rlen = (i + 1 < n ? (int64_t)rstart[i + 1] : c->r_total) - (int64_t)rstart[i];
      if (e < 0 || e >= c->n_edges || lane[i] < 0 || lane[i] >= c->lanes[e] || cursor[i] < 0 || cursor[i] >= rlen ||
          (int32_t)(rte[rstart[i] + cursor[i]] & ROUTE_EDGE_MASK) != e ||
          !(pos[i] >= 0.0f && pos[i] < (float)std::ceil(c->length[e])) || !(v[i] >= 0.0f && v[i] <= 254.0f))
        return fail(c, LPSIM_E_INVALID_ARG, "bad on-road state (trip %lld)", (long long)i);
    }
  }
  TRY(sync_parts(c));
  const unsigned buf = (unsigned)(step & 1), mk = (unsigned)(step & 1);
  const unsigned np = (unsigned)c->parts.size();
  std::vector<int32_t> owner((size_t)std::max(c->n_edges, 1)), up((size_t)std::max(c->n_edges, 1));
  for (int32_t e = 0; e < c->n_edges; ++e) {
    owner[e] = c->part_of[c->dst[e]];
    up[e] = c->part_of[c->src[e]];
  }
  int32_t *d_st = nullptr, *d_ed = nullptr, *d_ln = nullptr, *d_own = nullptr, *d_up = nullptr;
  float *d_pos = nullptr, *d_v = nullptr;
  int64_t* d_cur = nullptr;
  uint32_t* d_err = nullptr;
  const size_t nn = (size_t)std::max<int64_t>(n, 1), ne = (size_t)std::max(c->n_edges, 1);
  cudaError_t ce = cudaSuccess;
  auto cm = [&](void** p, size_t b) { if (ce == cudaSuccess) ce = cudaMalloc(p, b); };
  cm((void**)&d_st, nn * 4); cm((void**)&d_ed, nn * 4); cm((void**)&d_ln, nn * 4); cm((void**)&d_pos, nn * 4);
  cm((void**)&d_v, nn * 4); cm((void**)&d_cur, nn * 8); cm((void**)&d_own, ne * 4); cm((void**)&d_up, ne * 4);
  cm((void**)&d_err, 4);
  lpsim_status rs = LPSIM_OK;
  // copies and the memset ordered on the context's stream with the restore kernels
  if (ce == cudaSuccess && n > 0) {
    cudaMemcpyAsync(d_st, status, n * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(d_ed, edge, n * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(d_ln, lane, n * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(d_pos, pos, n * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(d_v, v, n * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(d_cur, cursor, n * 8, cudaMemcpyHostToDevice, c->stream);
  }
  if (ce == cudaSuccess) {
    cudaMemcpyAsync(d_own, owner.data(), ne * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(d_up, up.data(), ne * 4, cudaMemcpyHostToDevice, c->stream);
    cudaMemsetAsync(d_err, 0xFF, 4, c->stream);
    if (n > 0)
      k_restore_trips<<<grid_for(n), 256, 0, c->stream>>>(c->d_parts, np, buf, mk, c->P.h_max, n, c->d_route,
                                                           c->d_trip_rstart, d_own, d_up, d_st, d_ed, d_ln, d_pos,
                                                           d_v, d_cur, d_err);
    for (unsigned p = 0; p < np; ++p) {
      if (!c->parts[p].ctl) continue;
      k_mark_release_list<<<64, 256, 0, c->stream>>>(c->d_parts, p, (uint32_t)step);
      k_restore_released<<<grid_for(n), 256, 0, c->stream>>>(c->d_parts, p, (uint32_t)step, d_st);
      k_restore_slots<<<grid_for(std::max<uint32_t>(c->parts[p].d.n_slot_total, 1)), 256, 0, c->stream>>>(
          c->d_parts, p, (uint32_t)step, d_err);
    }
    ce = cudaStreamSynchronize(c->stream);
  }
  uint32_t err = 0xFFFFFFFFu;
  if (ce == cudaSuccess) ce = cudaMemcpy(&err, d_err, 4, cudaMemcpyDeviceToHost);
  cudaFree(d_st); cudaFree(d_ed); cudaFree(d_ln); cudaFree(d_pos); cudaFree(d_v); cudaFree(d_cur);
  cudaFree(d_own); cudaFree(d_up); cudaFree(d_err);
  if (ce != cudaSuccess) {
    c->failed = true;
    return fail(c, LPSIM_E_CUDA, "restore failed: %s", cudaGetErrorString(ce));
  }
  // (not reached after the host checks): the device state is partial, the context unusable
  if (err == 0xFFFFFFFEu) rs = fail(c, LPSIM_E_CAPACITY, "restore: admit list capacity");
  else if (err != 0xFFFFFFFFu) rs = fail(c, LPSIM_E_INVALID_ARG, "bad on-road state (trip %u)", err);
  if (rs != LPSIM_OK) {
    c->failed = true;
    return rs;
  }
  // arrivals, t_start per route edge, counters (on the first local partition / CTA 0's slots)
  if (n > 0) CU(cudaMemcpy(c->d_arrival, arr32.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice));
  if (edge_entry && c->r_total > 0)
    CU(cudaMemcpy(c->d_edge_entry, edge_entry, (size_t)c->r_total * sizeof(int32_t), cudaMemcpyHostToDevice));
  if (counters && (c->world == 1 || c->rank == 0)) {
    for (auto& H : c->parts) {
      if (!H.ctl) continue;
      const unsigned long long upd = (unsigned long long)counters[0];
      CU(cudaMemcpy((char*)H.ctl + offsetof(PartCtl, updates), &upd, sizeof(upd), cudaMemcpyHostToDevice));
      break;
    }
    // C_TRANS, C_LC, C_LOST, C_DEP, C_ARR of CTA 0 (the host sums the per-CTA slots)
    const unsigned long long cb[5] = {(unsigned long long)counters[2], (unsigned long long)counters[3],
                                      (unsigned long long)counters[5], (unsigned long long)counters[1],
                                      (unsigned long long)counters[4]};
    CU(cudaMemcpy(c->d_ctr_block, cb, sizeof(cb), cudaMemcpyHostToDevice));
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
    int32_t *ds, *de, *dl;
    float *dp, *dv;
    int64_t* dc;
    double* dd;
    CU(cudaMalloc(&ds, n * 4)); CU(cudaMalloc(&de, n * 4)); CU(cudaMalloc(&dl, n * 4));
    CU(cudaMalloc(&dp, n * 4)); CU(cudaMalloc(&dv, n * 4)); CU(cudaMalloc(&dc, n * 8)); CU(cudaMalloc(&dd, n * 8));
    lpsim_status s = trip_views(c, ds, de, dl, dp, dv, dc);
    if (s == LPSIM_OK) {
      k_distances<<<148 * 8, 256, 0, c->stream>>>(n, c->d_route, (int64_t)c->r_total, c->d_trip_rstart, c->d_length,
                                                  ds, dp, dc, c->d_arrival, dd);
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
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  uint8_t* d;
  CU(cudaMalloc(&d, std::max<int64_t>(size, 1)));
  const int b = (int)(c->step & 1);
  for (auto& H : c->parts)
    if (H.ctl) k_gather_map<<<std::max(1, std::min(c->n_edges, 148 * 8)), 256, 0, c->stream>>>(H.d.map[b], c->d_gbase, H.d.edges,
                                                                                  c->n_edges, d, c->d_lanes);
  cudaStreamSynchronize(c->stream);
  cudaError_t e = cudaMemcpy(out, d, size, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(c, LPSIM_E_CUDA, "lane map copy: %s", cudaGetErrorString(e));
  return LPSIM_OK;
}

lpsim_status lpsim_debug_map_occupancy(lpsim_ctx* c, uint64_t* out) {
  if (!c || !out) return LPSIM_E_INVALID_ARG;
  if (!c->loaded) return fail(c, LPSIM_E_STATE, "lpsim_debug_map_occupancy before lpsim_load_demand");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, LPSIM_E_CUDA, "cudaSetDevice failed");
  unsigned long long* d;
  CU(cudaMalloc(&d, 2 * sizeof(unsigned long long)));
  CU(cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), c->stream));
  for (auto& H : c->parts)
    if (H.ctl)
      for (int w = 0; w < 2; ++w)  // w = 0: M_k, w = 1: the other buffer (M_{k+1} before it is written)
        k_count_occupied<<<std::max(1, std::min(c->n_edges, 148 * 8)), 256, 0, c->stream>>>(
            H.d.map[(c->step + w) & 1], H.d.edges, c->n_edges, c->d_lanes, d + w);
  unsigned long long h[2] = {0, 0};
  cudaStreamSynchronize(c->stream);
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(c, LPSIM_E_CUDA, "occupancy copy: %s", cudaGetErrorString(e));
  out[0] = h[0];
  out[1] = h[1];
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
  uint32_t magic, rank, world, nin;
  cudaIpcMemHandle_t inq, map[2], xflag, mig_cnt;
};
static_assert(sizeof(IpcBlob) <= LPSIM_IPC_BLOB_BYTES, "blob size");
constexpr uint32_t IPC_MAGIC = 0x4c505331u;  // "LPS1"
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
  const PartDev& D = c->parts[c->rank].d;
  b.nin = D.n_in;
  CU(cudaIpcGetMemHandle(&b.inq, D.inq[0]));
  CU(cudaIpcGetMemHandle(&b.mig_cnt, c->d_mig_cnt));
  for (int i = 0; i < 2; ++i) CU(cudaIpcGetMemHandle(&b.map[i], D.map[i]));
  CU(cudaIpcGetMemHandle(&b.xflag, c->d_xflag));
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
  std::vector<uint32_t*> peer_flags((size_t)c->world, nullptr), peer_cnt((size_t)c->world, nullptr);
  peer_flags[c->rank] = c->d_xflag;
  peer_cnt[c->rank] = c->d_mig_cnt;
  for (int32_t q = 0; q < c->world; ++q) {
    IpcBlob b;
    std::memcpy(&b, (const char*)blobs + (size_t)q * LPSIM_IPC_BLOB_BYTES, sizeof(b));
    if (b.magic != IPC_MAGIC || (int32_t)b.rank != q || (int32_t)b.world != c->world)
      return fail(c, LPSIM_E_COMM, "bad IPC record for rank %d", q);
    if (q == c->rank) continue;
    if (b.nin != c->parts[q].d.n_in) return fail(c, LPSIM_E_COMM, "plan mismatch with rank %d (queue size)", q);
    void* p = nullptr;
    CU(cudaIpcOpenMemHandle(&p, b.inq, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    c->parts[q].d.inq[0] = (MigSlot*)p;
    c->parts[q].d.inq[1] = (MigSlot*)p + std::max<uint32_t>(b.nin, 1);
    CU(cudaIpcOpenMemHandle(&p, b.mig_cnt, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    peer_cnt[q] = (uint32_t*)p;
    for (int i = 0; i < 2; ++i) {
      CU(cudaIpcOpenMemHandle(&p, b.map[i], cudaIpcMemLazyEnablePeerAccess));
      c->ipc_opened.push_back(p);
      c->parts[q].d.map[i] = (uint8_t*)p;
    }
    CU(cudaIpcOpenMemHandle(&p, b.xflag, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    peer_flags[q] = (uint32_t*)p;
  }
  CU(cudaMemcpyAsync(c->d_xflag_peer, peer_flags.data(), c->world * sizeof(uint32_t*), cudaMemcpyHostToDevice,
                     c->stream));
  CU(cudaMemcpyAsync(c->d_mig_cnt_peer, peer_cnt.data(), c->world * sizeof(uint32_t*), cudaMemcpyHostToDevice,
                     c->stream));
  TRY(upload_parts(c));
  CU(cudaStreamSynchronize(c->stream));
  c->attached = true;
  return LPSIM_OK;
}

void lpsim_destroy(lpsim_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* p : c->allocs) cudaFree(p);
  for (cudaEvent_t e : c->sort_ev) cudaEventDestroy(e);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

}  // extern "C"
