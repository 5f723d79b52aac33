// Micro-benchmark: cost of a cluster barrier (barrier.cluster.arrive.release
// + wait.acquire) for one cluster of NC CTAs x T threads, and of a plain
// __syncthreads for comparison.  Build/run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cb profiles/cluster_barrier_bench.cu && /tmp/cb
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_cb(int iters, int mode, double* sink) {
  __shared__ double buf[2048];
  double acc = threadIdx.x;
  buf[threadIdx.x] = acc;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  unsigned nr;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nr));
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  for (int i = 0; i < iters; ++i) {
    acc = acc * 1.0000001 + 1.0;
    if (mode >= 3) {
      // one DSMEM read of the next CTA's buffer (mode 3) or a local read (mode 4), one local write
      const double* p = buf + ((threadIdx.x + i) & 1023);
      uint64_t q;
      asm volatile("mapa.u64 %0, %1, %2;" : "=l"(q) : "l"(p), "r"(mode == 3 ? (rank + 1) % nr : rank));
      acc += *reinterpret_cast<const double*>(q);
      buf[1024 + (threadIdx.x & 1023)] = acc;
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else if (mode == 0) {
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else if (mode == 1) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory");
    } else {
      __syncthreads();
    }
  }
  if (acc == -1.0) *sink = acc;
}

int main() {
  double* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(k_cb, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int nc : {2, 8, 16}) {
    for (int t : {256, 1024}) {
      for (int mode : {0, 1, 2, 3, 4}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(nc);
        cfg.blockDim = dim3(t);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = nc;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const int iters = 2000;
        cudaLaunchKernelEx(&cfg, k_cb, iters, mode, sink);
        cudaEventRecord(a);
        cudaLaunchKernelEx(&cfg, k_cb, iters, mode, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("cluster %2d x %4d threads, mode %s: %.3f us per barrier (%s)\n", nc, t,
               mode == 0 ? "release/acquire" : mode == 1 ? "relaxed        " : mode == 2 ? "syncthreads    " : mode == 3 ? "dsmem rd+bar   " : "local rd+bar   ",
               ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
