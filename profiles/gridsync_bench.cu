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

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// the persistent PCG's reduction pattern: block reduce -> partial -> grid
// barrier -> every block sums all partials in order
template <int MODE>
__global__ void k_reduce(int iters, double* part, double* sink) {
  cg::grid_group g = cg::this_grid();
  __shared__ double wred[32];
  __shared__ double bc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
  double acc = 0.0, v = threadIdx.x * 1e-3;
  for (int i = 0; i < iters; ++i) {
    double a = wsum(v);
    if (lane == 0) wred[warp] = a;
    __syncthreads();
    if (warp == 0) {
      double t = lane < (int)(blockDim.x / 32) ? wred[lane] : 0.0;
      t = wsum(t);
      if (lane == 0) part[(i & 1) * G + blockIdx.x] = t;
    }
    g.sync();
    if (MODE == 0) {
      if (warp == 0) {
        double t = 0.0;
        for (int q = lane; q < G; q += 32) t += __ldcg(part + (i & 1) * G + q);
        t = wsum(t);
        if (lane == 0) bc = t;
      }
      __syncthreads();
      acc += bc;
      __syncthreads();
    }
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
  double* part;
  cudaMalloc(&part, 4096 * sizeof(double));
  for (int mode = 0; mode < 2; ++mode) {
    int iters = 2000;
    void* args[] = {&iters, &part, &sink};
    void* fn = mode == 0 ? (void*)k_reduce<0> : (void*)k_reduce<1>;
    cudaLaunchCooperativeKernel(fn, sms, 1024, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel(fn, sms, 1024, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("reduce pattern mode %d (1 = no partial read): %.3f us/iter (%s)\n", mode,
           ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
