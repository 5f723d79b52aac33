// Micro-benchmark: back-to-back launch cost of an empty cluster kernel
// (NC CTAs x T threads, S bytes of dynamic shared memory) vs a plain grid,
// eager and inside a CUDA graph.  Build/run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cl profiles/cluster_launch_bench.cu && /tmp/cl
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(double* sink) {
  extern __shared__ double sm[];
  if (threadIdx.x == 0 && sink == nullptr) sm[0] = 1.0;
}

static float run(int nc, int t, int smem, bool graph, int reps) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nc > 0 ? nc : 16);
  cfg.blockDim = dim3(t);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = nc > 0 ? 1 : 0;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cfg.stream = s;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaGraphExec_t ge = nullptr;
  if (graph) {
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, k_empty, (double*)1);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
  } else {
    for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, k_empty, (double*)1);
  }
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  if (graph) cudaGraphLaunch(ge, s);
  else
    for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, k_empty, (double*)1);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms * 1e3f / reps;
}

int main() {
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int graph : {0, 1})
    for (int nc : {0, 1, 2, 8, 16})
      for (int t : {256, 1024})
        for (int smem : {0, 64 * 1024, 220 * 1024})
          printf("%s cluster %2d x %4d threads, smem %6d: %.2f us per launch\n",
                 graph ? "graph" : "eager", nc, t, smem, run(nc, t, smem, graph, 200));
  return 0;
}
