// Microbenchmark: cost of one grid-wide barrier on B200 for several grid
// sizes and implementations (atomic counter + generation spin, with plain
// fences or release/acquire PTX; cooperative_groups grid.sync()).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

struct Bar { unsigned count, gen; };

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old; asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory"); return old;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MODE>
__global__ void k_bar(Bar* b, int iters, unsigned* sink) {
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 2) {
      cg::this_grid().sync();
    } else {
      __syncthreads();
      if (threadIdx.x == 0) {
        if (MODE == 1) {
          const unsigned g = ld_acquire(&b->gen);
          if (atom_add_acq_rel(&b->count, 1u) == gridDim.x - 1) { b->count = 0; st_release(&b->gen, g + 1); }
          else while (ld_acquire(&b->gen) == g) {}
        } else {
          volatile unsigned* gp = &b->gen;
          const unsigned g = *gp;
          __threadfence();
          if (atomicAdd(&b->count, 1u) == gridDim.x - 1) { b->count = 0; __threadfence(); atomicAdd(&b->gen, 1u); }
          else while (*gp == g) {}
          __threadfence();
        }
      }
      __syncthreads();
    }
    acc += threadIdx.x;
  }
  if (acc == 0xFFFFFFFF) *sink = acc;
}

template <int MODE>
void run(int blocks, int threads, Bar* b, unsigned* sink) {
  int iters = 2000;
  void* args[] = {&b, &iters, &sink};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchCooperativeKernel((void*)k_bar<MODE>, blocks, threads, args, 0, 0);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  cudaLaunchCooperativeKernel((void*)k_bar<MODE>, blocks, threads, args, 0, 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("mode %d blocks %4d threads %4d: %.3f us/barrier %s\n", MODE, blocks, threads, 1e3 * ms / iters,
         err ? cudaGetErrorString(err) : "");
}

int main() {
  Bar* b; unsigned* sink;
  cudaMalloc(&b, sizeof(Bar)); cudaMemset(b, 0, sizeof(Bar)); cudaMalloc(&sink, 4);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int bps : {1, 2, 4}) for (int t : {256, 512}) {
    if (bps * t > 2048) continue;
    run<0>(nsm * bps, t, b, sink); run<1>(nsm * bps, t, b, sink); run<2>(nsm * bps, t, b, sink);
  }
  return 0;
}
