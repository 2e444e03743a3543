// Microbenchmark: what a one-step measurement after an L2 flush pays before the step kernel runs.
// Empty kernel with the step kernel's grid (444 x 256) and shared-memory footprint, timed with CUDA
// events on the stream after: nothing, a cudaMemset flush (256 MiB), or a flush kernel that asks for
// the same shared-memory carveout as the step kernel.
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 3) k_empty(unsigned* sink) {
  extern __shared__ unsigned s[];
  if (threadIdx.x == 0 && blockIdx.x == 100000) { s[0] = 1; *sink = s[1]; }
}
__global__ void __launch_bounds__(256, 3) k_flush(uint4* p, size_t n) {
  extern __shared__ unsigned s[];
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(1, 2, 3, 4);
  if (n == 0) s[threadIdx.x] = 0;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = 3 * nsm, threads = 256;
  unsigned* sink; void* flush;
  cudaMalloc(&sink, 4);
  const size_t fb = 256u << 20;
  cudaMalloc(&flush, fb);
  const int dyn = 45056 + 10240;  // the step kernel's dynamic + static shared memory
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  cudaFuncSetAttribute(k_flush, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"no flush, 0 smem", "no flush, step smem", "memset flush, 0 smem", "memset flush, step smem",
                         "flush kernel (step carveout), step smem", "flush kernel (0 smem), step smem",
                         "memset flush, no kernel (events only)"};
  for (int mode = 0; mode < 7; ++mode) {
    std::vector<float> t;
    for (int r = 0; r < 80; ++r) {
      if (mode >= 2 && mode != 4 && mode != 5) cudaMemsetAsync(flush, r & 255, fb, st);
      if (mode == 4) k_flush<<<blocks, threads, dyn, st>>>((uint4*)flush, fb / 16);
      if (mode == 5) k_flush<<<blocks, threads, 0, st>>>((uint4*)flush, fb / 16);
      cudaEventRecord(e0, st);
      const int sm = (mode == 0 || mode == 2) ? 0 : dyn;
      if (mode != 6) k_empty<<<blocks, threads, sm, st>>>(sink);
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 10) t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    printf("%-45s median %.2f us  p10 %.2f  p90 %.2f\n", names[mode], t[t.size() / 2], t[t.size() / 10], t[t.size() * 9 / 10]);
  }
  return 0;
}
