// lpsim_kernels.h — kernel declarations (definitions in lpsim_step.cu).
#pragma once
#include <cuda_runtime.h>

#include "lpsim_dev.h"

namespace lpsim {
#ifndef LPSIM_BS
#define LPSIM_BS 512
#endif
#ifndef LPSIM_MINB
#define LPSIM_MINB 2  // resident CTAs (tiles) per SM the register budget is sized for
#endif
#ifndef LPSIM_HT_BITS
#define LPSIM_HT_BITS 12
#endif
constexpr int TILE_BS = LPSIM_BS;       // threads per CTA (tile) of the step kernel
constexpr int TILE_MINB = LPSIM_MINB;
constexpr unsigned TILE_HT_BITS = LPSIM_HT_BITS;
constexpr int SCAN_BLOCK = 1024;
size_t tile_dyn_smem();  // dynamic shared memory bytes of the step kernel (per CTA)
// the step kernel: lean (digest and timing code compiled out) and instrumented (k_tile_full)
__global__ void k_tile(Global G, Params P, unsigned long long k0, unsigned nsteps);
__global__ void k_tile_full(Global G, Params P, unsigned long long k0, unsigned nsteps);
__global__ void k_fill_u8(uint8_t* p, uint8_t v, size_t n);
__global__ void k_fill_u32(uint32_t* p, uint32_t v, size_t n);
__global__ void k_edge_cells(const float* length, const uint8_t* lanes, uint64_t* cells, uint32_t* ncells, int E);
__global__ void k_scan_blocks(const uint64_t* in, uint64_t* out, uint64_t* sums, int n);
__global__ void k_scan_sums(uint64_t* sums, int nb, uint64_t* total);
__global__ void k_scan_add(uint64_t* out, const uint64_t* sums, int n);
__global__ void k_build_edges(int E, const uint64_t* base, const uint32_t* ncells, const uint8_t* lanes, const float* v0,
                              const uint32_t* li, const uint32_t* meta, EdgeRec* out);
// departure contexts: ctx of the first edge into the context array of the part owning it, the entry
// cell of the second edge for the departure lane
__global__ void k_trip_ctx(const EdgeRec* edges, const uint32_t* route, const uint4* rinfo,
                           const uint32_t* trip_rstart, const uint8_t* edge_opart, const PartPtrs* parts,
                           unsigned n_parts, int64_t n, uint2* dep);
// the route-position table: per route entry j (not last), the next edge's data (Global::rinfo)
__global__ void k_route_info(const uint32_t* route, const EdgeRec* edges, int64_t R, uint4* rinfo);
// per-trip view of the on-road vehicles of the tiles [t0, t1) at snapshot k (records + migrants in flight)
__global__ void k_scatter_trips(Global G, uint32_t t0, uint32_t t1, unsigned long long k, int32_t* status,
                                int32_t* edge, int32_t* lane, float* pos, float* v, int64_t* cursor);
__global__ void k_distances(int64_t n, const uint32_t* route, const uint32_t* trip_rstart, const float* length,
                            const int32_t* status, const float* pos, const int64_t* cursor, const int32_t* arrival,
                            double* dist);
// cells of the edges owned by part p (edge_opart[e] == p): copy map -> out (global layout) / count occupied
__global__ void k_gather_map(const uint8_t* map, const EdgeRec* edges, const uint8_t* edge_opart, unsigned p, int E,
                             uint8_t* out);
__global__ void k_count_occupied(const uint8_t* map, const EdgeRec* edges, const uint8_t* edge_opart, unsigned p,
                                 int E, unsigned long long* out);
// restore (§8(f) checkpoint): on-road trips into the records of their edge's tile + their byte in M_k
// (local_part = 0xFFFFFFFF: every part is simulated by this process)
__global__ void k_restore_trips(Global G, unsigned local_part, unsigned mk, unsigned cb, int h_max, int64_t n,
                                const uint32_t* tile_of_edge, const int32_t* status, const int32_t* edge,
                                const int32_t* lane, const float* pos, const float* v, const int64_t* cursor,
                                uint32_t* err);
// waiting trips released before step k: bits, counts, candidates, pending lists of the tiles [t0, t1)
__global__ void k_restore_released(Global G, uint32_t t0, uint32_t t1, uint32_t k, const int32_t* status);
}  // namespace lpsim
