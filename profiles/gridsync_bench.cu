// Micro-benchmark: cost of cooperative_groups grid.sync() on this GPU with
// one 1024-thread CTA per SM (the persistent PCG launch shape), and of a
// hand-rolled atomic barrier.  Build/run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gs profiles/gridsync_bench.cu && /tmp/gs
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_sync(int iters, double* sink) {
  cg::grid_group g = cg::this_grid();
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    acc += i;
    g.sync();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = acc;
}

__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;

__device__ __forceinline__ void bar_atomic(unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int gen = g_gen;
    __threadfence();
    if (atomicAdd(&g_count, 1u) == nblocks - 1) {
      g_count = 0;
      __threadfence();
      g_gen = gen + 1;
    } else {
      while (g_gen == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_atomic(int iters, double* sink) {
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    acc += i;
    bar_atomic(gridDim.x);
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {256, 1024}) {
    int iters = 2000;
    void* args[] = {&iters, &sink};
    cudaLaunchCooperativeKernel((void*)k_sync, sms, threads, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_sync, sms, threads, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync  blocks=%d threads=%d: %.3f us/sync (%s)\n", sms, threads, ms * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
    cudaLaunchCooperativeKernel((void*)k_atomic, sms, threads, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_atomic, sms, threads, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("atomic bar blocks=%d threads=%d: %.3f us/sync (%s)\n", sms, threads, ms * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
