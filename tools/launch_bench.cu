// Microbenchmark: GPU-side cost of launching the step kernel's grid (444 CTAs x 256 threads on
// B200) with cudaLaunchCooperativeKernel vs a plain launch, measured with CUDA events around the
// launch after a 256 MiB memset on the same stream (the bench's per-step pattern); and the cost
// of a flip-bit grid barrier (the cooperative_groups algorithm, own counter, plain launch) vs
// cooperative_groups grid.sync().
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(256, 3) k_empty(unsigned* sink) {
  if (threadIdx.x == 0 && blockIdx.x == 100000) *sink = 1;
}

__device__ __forceinline__ void flip_barrier(unsigned* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned add = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    __threadfence();
    const unsigned old = atomicAdd(ctr, add);
    volatile unsigned* v = ctr;
    while (((*v ^ old) & 0x80000000u) == 0u) {}
    __threadfence();
  }
  __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(256, 3) k_bar(unsigned* ctr, int iters, unsigned* sink) {
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 2) cg::this_grid().sync();
    else flip_barrier(ctr);
    acc += threadIdx.x;
  }
  if (acc == 0xFFFFFFFF) *sink = acc;
}

__global__ void k_bar2(unsigned* ctr, int iters, unsigned* sink) {
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    cg::this_grid().sync();
    acc += threadIdx.x;
  }
  if (acc == 0xFFFFFFFF) *sink = acc;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = 3 * nsm, threads = 256;
  unsigned *sink, *ctr; void* flush;
  cudaMalloc(&sink, 4); cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
  cudaMalloc(&flush, 256u << 20);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int coop = 1; coop >= 0; --coop) {
    std::vector<float> t;
    for (int r = 0; r < 60; ++r) {
      cudaMemsetAsync(flush, r & 255, 256u << 20, st);
      void* args[] = {&sink};
      cudaEventRecord(e0, st);
      if (coop) cudaLaunchCooperativeKernel((void*)k_empty, blocks, threads, args, 0, st);
      else k_empty<<<blocks, threads, 0, st>>>(sink);
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 10) t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    printf("empty kernel %s launch after a flush: median %.2f us, p10 %.2f, p90 %.2f\n", coop ? "cooperative" : "plain",
           t[t.size() / 2], t[t.size() / 10], t[t.size() * 9 / 10]);
  }
  const int iters = 4000;
  for (int cfg = 0; cfg < 3; ++cfg) {  // the barrier alone for 148 x 768, 296 x 384, 444 x 256 CTAs
    const int bl = cfg == 0 ? nsm : cfg == 1 ? 2 * nsm : 3 * nsm, th = cfg == 0 ? 768 : cfg == 1 ? 384 : 256;
    void* args[] = {&ctr, (void*)&iters, &sink};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a, st);
      cudaLaunchCooperativeKernel((void*)k_bar2, bl, th, args, 0, st);
      cudaEventRecord(b, st);
      cudaError_t err = cudaStreamSynchronize(st);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("cg grid.sync with %d CTAs x %d threads: %.3f us per barrier %s\n", bl, th, 1e3 * ms / iters,
                      err ? cudaGetErrorString(err) : "");
    }
  }
  for (int mode : {2, 3}) {
    void* args[] = {&ctr, (void*)&iters, &sink};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a, st);
      if (mode == 2) cudaLaunchCooperativeKernel((void*)k_bar<2>, blocks, threads, args, 0, st);
      else k_bar<3><<<blocks, threads, 0, st>>>(ctr, iters, sink);
      cudaEventRecord(b, st);
      cudaError_t err = cudaStreamSynchronize(st);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("barrier %s: %.3f us per barrier (%d CTAs) %s\n", mode == 2 ? "cg grid.sync" : "flip-bit, plain launch",
                      1e3 * ms / iters, blocks, err ? cudaGetErrorString(err) : "");
    }
  }
  return 0;
}
