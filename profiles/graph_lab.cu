// Lab: per-kernel cost of graph replay, plain graph vs conditional WHILE
// body, for tiny kernels (the multigrid's small levels).  Not library code.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o graph_lab profiles/graph_lab.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void tiny(double* x, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 0.5 + 1.0;
}
__global__ void cond_k(cudaGraphConditionalHandle h, int* counter, int reps) {
  if (threadIdx.x == 0) {
    int c = ++(*counter);
    cudaGraphSetConditional(h, c < reps ? 1u : 0u);
  }
}

int main() {
  double* x;
  int* cnt;
  const int n = 4096;
  cudaMalloc(&x, n * 8 * 64);
  cudaMalloc(&cnt, 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int K = 40, REPS = 50;
  for (int blocks : {1, 16, 148, 592}) {
    // plain graph: REPS x K kernels
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int r = 0; r < REPS; ++r)
      for (int k = 0; k < K; ++k) tiny<<<blocks, 256, 0, s>>>(x + (k % 8) * n, blocks * 256 < n ? blocks * 256 : n);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("blocks %4d plain graph:   %.2f us per kernel\n", blocks, ms * 1e3 / (REPS * K));
    // while graph: body of K kernels + cond, REPS passes
    cudaGraph_t wg;
    cudaGraphCreate(&wg, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, wg, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    cudaGraphAddNode(&node, wg, nullptr, 0, &np);
    cudaGraph_t body = np.conditional.phGraph_out[0];
    cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    for (int k = 0; k < K; ++k) tiny<<<blocks, 256, 0, s>>>(x + (k % 8) * n, blocks * 256 < n ? blocks * 256 : n);
    cond_k<<<1, 32, 0, s>>>(h, cnt, REPS);
    cudaStreamEndCapture(s, &body);
    cudaGraphExec_t wge;
    cudaGraphInstantiate(&wge, wg, 0);
    cudaMemsetAsync(cnt, 0, 4, s);
    cudaGraphLaunch(wge, s);
    cudaStreamSynchronize(s);
    cudaMemsetAsync(cnt, 0, 4, s);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(wge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("blocks %4d while graph:   %.2f us per kernel (%s)\n", blocks, ms * 1e3 / (REPS * (K + 1)),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
