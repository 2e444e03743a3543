// Microbenchmark, second round: grid-barrier variants at the step kernel's
// launch shape (148 SMs x 3 CTAs x 256 threads).
//   mode 2: cooperative_groups grid.sync() (one counter, all CTAs arrive on it)
//   mode 3: striped monotone counters (NS counters 128 B apart; CTA b adds to
//           stripe b % NS with red.release; lanes of warp 0 poll all stripes)
//   mode 4: cluster-hierarchical: hardware cluster barrier, one arrival per
//           cluster on the striped counters, cluster barrier again
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/barrier_bench2 tools/barrier_bench2.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int STRIDE = 32;  // u32 words between stripes (128 B)

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_hw() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ unsigned cluster_id_x() {
  unsigned r; asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r)); return r;
}
__device__ __forceinline__ unsigned n_clusters_x() {
  unsigned r; asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r)); return r;
}

// arrivals: `unit` = this arriving unit's index, `nunits` = number of units; stripe s
// receives units u with u % NS == s, i.e. (nunits - s + NS - 1) / NS of them per barrier
template <int NS>
__device__ __forceinline__ void striped_barrier(unsigned* cnt, unsigned unit, unsigned nunits, unsigned gen) {
  if (threadIdx.x == 0) red_release_add(cnt + (unit % NS) * STRIDE, 1u);
  if (threadIdx.x < 32) {
    const unsigned s = threadIdx.x;
    const unsigned per = s < NS ? (nunits - s + NS - 1) / NS : 0u;
    const unsigned target = per * gen;
    bool ok = s >= NS;
    while (!__all_sync(0xffffffffu, ok)) {
      if (!ok) ok = (int)(ld_acquire(cnt + s * STRIDE) - target) >= 0;
    }
  }
}

template <int MODE, int NS>
__global__ void k_bar(unsigned* cnt, int iters, unsigned* sink) {
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 2) {
      cg::this_grid().sync();
    } else if (MODE == 3) {
      __syncthreads();
      striped_barrier<NS>(cnt, blockIdx.x, gridDim.x, (unsigned)it + 1u);
      __syncthreads();
    } else {
      cluster_sync_hw();
      if (cluster_rank() == 0) striped_barrier<NS>(cnt, cluster_id_x(), n_clusters_x(), (unsigned)it + 1u);
      cluster_sync_hw();
    }
    acc += threadIdx.x;
  }
  if (acc == 0xFFFFFFFF) *sink = acc;
}

template <int MODE, int NS>
void run(int blocks, int threads, int cluster, unsigned* cnt, unsigned* sink) {
  int iters = 4000;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = cluster;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if (cluster > 1) {
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, k_bar<MODE, NS>, &cfg);
    if (ncl * cluster < blocks) {
      printf("mode %d NS %2d blocks %4d cluster %d: only %d clusters co-resident, skipped\n", MODE, NS, blocks,
             cluster, ncl);
      return;
    }
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(cnt, 0, 64 * STRIDE * 4);
    cudaEventRecord(e0);
    cudaError_t le = cudaLaunchKernelEx(&cfg, k_bar<MODE, NS>, cnt, iters, sink);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    if (le != cudaSuccess || err != cudaSuccess) {
      printf("mode %d NS %2d blocks %4d cluster %d: error %s / %s\n", MODE, NS, blocks, cluster,
             cudaGetErrorString(le), cudaGetErrorString(err));
      cudaGetLastError();
      return;
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("mode %d NS %2d blocks %4d threads %d cluster %d: %.3f us/barrier\n", MODE, NS, blocks, threads, cluster,
         1e3 * best / iters);
}

int main() {
  unsigned *cnt, *sink;
  cudaMalloc(&cnt, 64 * STRIDE * 4); cudaMalloc(&sink, 4);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int bps : {1, 2, 3}) {
    const int b = nsm * bps;
    run<2, 1>(b, 256, 1, cnt, sink);
    run<3, 1>(b, 256, 1, cnt, sink);
    run<3, 4>(b, 256, 1, cnt, sink);
    run<3, 8>(b, 256, 1, cnt, sink);
    run<3, 16>(b, 256, 1, cnt, sink);
    run<3, 32>(b, 256, 1, cnt, sink);
    run<4, 8>(b, 256, 2, cnt, sink);
    run<4, 8>(b, 256, 4, cnt, sink);
    run<4, 4>(b, 256, 4, cnt, sink);
    run<4, 16>(b, 256, 2, cnt, sink);
  }
  return 0;
}
