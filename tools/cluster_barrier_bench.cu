// Microbenchmark: grid-wide barrier of the step kernel's grid (444 CTAs x 256 threads, all resident)
// - cooperative_groups grid.sync() (the step kernel's barrier)
// - hierarchical: thread-block clusters of C CTAs (barrier.cluster in hardware), one CTA per cluster
//   arrives on a global flip-bit counter and polls it, then a second cluster barrier releases the cluster
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(256, 3) k_cg(int iters, unsigned* sink) {
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    cg::this_grid().sync();
    acc += threadIdx.x;
  }
  if (acc == 0xFFFFFFFF) *sink = acc;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned nclusters() {
  unsigned r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}

__global__ void __launch_bounds__(256, 3) k_hier(unsigned* ctr, int iters, unsigned* sink) {
  unsigned acc = 0;
  const bool leader = cluster_rank() == 0 && threadIdx.x == 0;
  const unsigned ncl = nclusters();
  const bool master = leader && cluster_id() == 0;
  for (int it = 0; it < iters; ++it) {
    cluster_sync_all();
    if (leader) {
      const unsigned add = master ? 0x80000000u - (ncl - 1u) : 1u;
      unsigned old;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(ctr), "r"(add) : "memory");
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(ctr) : "memory");
      } while (((old ^ cur) & 0x80000000u) == 0u);
    }
    cluster_sync_all();
    acc += threadIdx.x;
  }
  if (acc == 0xFFFFFFFF) *sink = acc;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = 3 * nsm, threads = 256;
  unsigned *sink, *ctr;
  cudaMalloc(&sink, 4); cudaMalloc(&ctr, 4);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4000;
  for (int rep = 0; rep < 2; ++rep) {
    void* args[] = {(void*)&iters, &sink};
    cudaEventRecord(a, st);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k_cg, blocks, threads, args, 0, st);
    cudaEventRecord(b, st);
    cudaStreamSynchronize(st);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cg grid.sync, %d CTAs: %.3f us per barrier (%s)\n", blocks, ms * 1e3 / iters, cudaGetErrorString(e));
  }
  for (int csz : {2, 4, 6, 3}) {
    if (blocks % csz) continue;
    for (int coop = 1; coop >= 0; --coop) {
      cudaMemset(ctr, 0, 4);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = 0; cfg.stream = st;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
      cfg.attrs = at; cfg.numAttrs = coop ? 2 : 1;
      int ncl = 0;
      cudaOccupancyMaxActiveClusters(&ncl, (void*)k_hier, &cfg);
      cudaEventRecord(a, st);
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_hier, ctr, iters, sink);
      cudaEventRecord(b, st);
      cudaError_t e2 = cudaStreamSynchronize(st);
      float ms = 0; cudaEventElapsedTime(&ms, a, b);
      printf("cluster %d (%s launch; max active clusters %d, needed %d): %.3f us per barrier (%s / %s)\n", csz,
             coop ? "cooperative" : "plain", ncl, blocks / csz, ms * 1e3 / iters, cudaGetErrorString(e), cudaGetErrorString(e2));
      if (e2 != cudaSuccess) return 1;
    }
  }
  return 0;
}
