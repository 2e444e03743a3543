// lpsim_kernels.h — kernel declarations (definitions in lpsim_step.cu).
#pragma once
#include <cuda_runtime.h>

#include "lpsim_dev.h"

namespace lpsim {
#ifndef LPSIM_BS
#define LPSIM_BS 256
#endif
constexpr int STEP_BS = LPSIM_BS;  // threads per CTA of the step kernel
constexpr int SCAN_BLOCK = 1024;
size_t step_dyn_smem();  // dynamic shared memory bytes of the step kernel (per CTA)
// the descriptor of a process's single partition travels in the launch parameters (constant bank):
// the CTAs stage it in shared memory without a dependent global load at launch start
struct PartParam {
  uint32_t valid;  // 1: use d, else read G.parts[part] (several partitions in one process)
  uint32_t mk;     // k0 & 1 (lane map M_k of the first step)
  PartDev d;
};
// the step kernel: lean for one partition (k_run: digest, timing and exchange code compiled out), lean for
// several partitions (k_run_multi), instrumented (k_run_full)
__global__ void k_run(Global G, Params P, PartParam PP, unsigned long long k0, unsigned nsteps);
__global__ void k_run_full(Global G, Params P, PartParam PP, unsigned long long k0, unsigned nsteps);
__global__ void k_run_multi(Global G, Params P, PartParam PP, unsigned long long k0, unsigned nsteps);
__global__ void k_fill_u8(uint8_t* p, uint8_t v, size_t n);
__global__ void k_fill_u32(uint32_t* p, uint32_t v, size_t n);
__global__ void k_edge_cells(const float* length, const uint8_t* lanes, uint64_t* cells, uint32_t* ncells, int E);
__global__ void k_scan_blocks(const uint64_t* in, uint64_t* out, uint64_t* sums, int n);
__global__ void k_scan_sums(uint64_t* sums, int nb, uint64_t* total);
__global__ void k_scan_add(uint64_t* out, const uint64_t* sums, int n);
__global__ void k_scatter_trips(PartDev* parts, unsigned np, unsigned buf, const uint32_t* mig_cnt,
                                const uint32_t* trip_rstart, int32_t* status, int32_t* edge, int32_t* lane, float* pos,
                                float* v, int64_t* cursor);
__global__ void k_mark_last(int64_t n, int64_t R, const uint32_t* trip_rstart, uint32_t* route);
__global__ void k_trip_defaults(int64_t n, const int32_t* arrival, const uint32_t* route, const uint32_t* trip_rstart,
                                int32_t* status, int32_t* edge, int32_t* lane, float* pos, float* v, int64_t* cur);
__global__ void k_distances(int64_t n, const uint32_t* route, int64_t R, const uint32_t* trip_rstart,
                            const float* length, const int32_t* status, const float* pos, const int64_t* cursor,
                            const int32_t* arrival, double* dist);
__global__ void k_gather_map(const uint8_t* local, const uint64_t* gbase, const EdgeRec* edges, int E, uint8_t* out,
                             const uint8_t* lanes);
__global__ void k_count_occupied(const uint8_t* map, const EdgeRec* edges, int E, const uint8_t* lanes,
                                 unsigned long long* out);
constexpr unsigned SORT_SHIFT = 8;  // a9: the locality sort orders by cell >> SORT_SHIFT (k_bucket_sort)
// a9 work buffers of one partition
struct SortBufs {
  uint32_t* bcount;  // bucket counts [nb] (zero between sorts)
  uint32_t* bcur;    // bucket cursors [nb]
  uint32_t* bsum;    // per-CTA segment sums [grid]
  uint32_t* perm;    // [veh_cap]
  uint32_t nb, pad;
};
// partitions p0 .. p0+nl-1 in one cooperative launch (the CTAs split among them, as in the step kernel)
__global__ void k_bucket_sort(const PartDev* parts, const SortBufs* sb, unsigned p0, unsigned nl, unsigned buf,
                              unsigned mode);
__global__ void k_restore_trips(PartDev* parts, unsigned np, uint32_t buf, uint32_t mk, int h_max, int64_t n,
                                const uint32_t* route, const uint32_t* trip_rstart, const int32_t* edge_owner,
                                const int32_t* edge_up, const int32_t* status, const int32_t* edge,
                                const int32_t* lane, const float* pos, const float* v, const int64_t* cursor,
                                uint32_t* err);
__global__ void k_restore_released(PartDev* parts, unsigned p, uint32_t k, const int32_t* status);
__global__ void k_restore_slots(PartDev* parts, unsigned p, uint32_t k, uint32_t* err);
__global__ void k_mark_release_list(PartDev* parts, unsigned p, uint32_t k);
__global__ void k_trip_ctx(PartDev* parts, unsigned p, const uint32_t* route, const uint32_t* trip_rstart,
                           const uint32_t* trips, uint32_t n, int h_max);
__global__ void k_build_edges(int E, const uint64_t* base, const uint32_t* ncells, const float* v0,
                              const uint32_t* meta, EdgeRec* out);
}  // namespace lpsim
