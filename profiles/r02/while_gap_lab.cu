// Lab (not library code): GPU idle time between a straight-line graph and a
// following graph holding a conditional WHILE node, measured with
// %globaltimer stamps (no profiler).  Variants: separate graph launches,
// one combined graph (kernels then the WHILE node), explicit upload, PDL.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/wg profiles/r02/while_gap_lab.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// stamp[2*i] = start, stamp[2*i+1] = end of kernel i (block 0, thread 0)
__global__ void work(double* x, int n, unsigned long long* st, int i) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0 && threadIdx.x == 0) st[2 * i] = gtime();
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    x[k] = x[k] * 0.5 + 1.0;
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) st[2 * i + 1] = gtime();
}
__global__ void cond_k(cudaGraphConditionalHandle h, int* counter, int passes) {
  if (threadIdx.x == 0) {
    int c = ++(*counter);
    cudaGraphSetConditional(h, c < passes ? 1u : 0u);
  }
}
__global__ void reset(int* c) { *c = 0; }

static void lk(cudaStream_t s, double* x, int n, unsigned long long* st, int i, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = 148;
  cfg.blockDim = 256;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, work, x, n, st, i);
}

int main() {
  const int n = 1 << 20;
  double* x;
  int* cnt;
  unsigned long long* st;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&cnt, 4);
  cudaMallocManaged(&st, 64 * 8);
  cudaStream_t s, cs;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl) {
    // graph A: reset + 4 kernels (stamps 0..3)
    cudaGraph_t ga;
    cudaGraphExec_t gea;
    cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    reset<<<1, 1, 0, cs>>>(cnt);
    for (int i = 0; i < 4; ++i) lk(cs, x, n, st, i, pdl);
    cudaStreamEndCapture(cs, &ga);
    cudaGraphInstantiate(&gea, ga, 0);
    // plain graph B: 2 kernels (stamps 4, 5)
    cudaGraph_t gb;
    cudaGraphExec_t geb;
    cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    for (int i = 4; i < 6; ++i) lk(cs, x, n, st, i, pdl);
    cudaStreamEndCapture(cs, &gb);
    cudaGraphInstantiate(&geb, gb, 0);
    // while graph W: body = 2 kernels (stamps 4, 5) + cond (1 pass)
    auto make_while = [&](bool with_prefix, bool upload) {
      cudaGraph_t g;
      cudaGraphCreate(&g, 0);
      cudaGraphNode_t last = nullptr;
      if (with_prefix) {
        cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
        reset<<<1, 1, 0, cs>>>(cnt);
        for (int i = 0; i < 4; ++i) lk(cs, x, n, st, i, pdl);
        cudaStreamEndCapture(cs, &g);
        size_t nn = 0;
        cudaGraphGetNodes(g, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        cudaGraphGetNodes(g, nodes.data(), &nn);
        // the sink node (no dependents)
        for (auto nd : nodes) {
          size_t nd_out = 0;
          cudaGraphNodeGetDependentNodes(nd, nullptr, &nd_out);
          if (nd_out == 0) last = nd;
        }
      }
      cudaGraphConditionalHandle h;
      cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
      cudaGraphNodeParams np = {};
      np.type = cudaGraphNodeTypeConditional;
      np.conditional.handle = h;
      np.conditional.type = cudaGraphCondTypeWhile;
      np.conditional.size = 1;
      cudaGraphNode_t node;
      cudaError_t e = cudaGraphAddNode(&node, g, last ? &last : nullptr, last ? 1 : 0, &np);
      if (e) printf("add node: %s\n", cudaGetErrorString(e));
      cudaGraph_t body = np.conditional.phGraph_out[0];
      cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
      for (int i = 4; i < 6; ++i) lk(cs, x, n, st, i, pdl);
      cond_k<<<1, 32, 0, cs>>>(h, cnt, 1);
      cudaGraph_t got;
      cudaStreamEndCapture(cs, &got);
      cudaGraphExec_t ge;
      e = cudaGraphInstantiate(&ge, g, 0);
      if (e) printf("inst: %s\n", cudaGetErrorString(e));
      if (upload) cudaGraphUpload(ge, s);
      return ge;
    };
    cudaGraphExec_t gw = make_while(false, false);
    cudaGraphExec_t gwu = make_while(false, true);
    cudaGraphExec_t gc = make_while(true, true);
    auto run = [&](const char* name, auto&& f) {
      double gap_sum = 0, tot = 0;
      const int R = 50;
      for (int r = 0; r < R + 3; ++r) {
        f();
        cudaStreamSynchronize(s);
        if (r < 3) continue;
        gap_sum += (double)(st[8] - st[7]) / 1e3;  // start of kernel 4 - end of kernel 3
        tot += (double)(st[11] - st[0]) / 1e3;
      }
      printf("pdl=%d %-34s gap k3->k4 %7.2f us   span %7.2f us\n", pdl, name, gap_sum / R, tot / R);
    };
    run("plain A -> plain B", [&] { cudaGraphLaunch(gea, s); cudaGraphLaunch(geb, s); });
    run("plain A -> while W", [&] { cudaGraphLaunch(gea, s); cudaGraphLaunch(gw, s); });
    run("plain A -> while W (uploaded)", [&] { cudaGraphLaunch(gea, s); cudaGraphLaunch(gwu, s); });
    run("combined A+WHILE one graph", [&] { cudaGraphLaunch(gc, s); });
    {
      std::vector<cudaGraphExec_t> ws;
      for (int q = 0; q < 4; ++q) ws.push_back(make_while(false, true));
      int rr = 0;
      run("plain A -> 4 while graphs round-robin", [&] { cudaGraphLaunch(gea, s); cudaGraphLaunch(ws[rr++ % 4], s); });
      std::vector<cudaGraphExec_t> wc;
      for (int q = 0; q < 4; ++q) wc.push_back(make_while(true, true));
      run("4 combined graphs round-robin", [&] { cudaGraphLaunch(wc[rr++ % 4], s); });
      std::vector<cudaGraphExec_t> pb;
      for (int q = 0; q < 4; ++q) {
        cudaGraph_t g2; cudaGraphExec_t e2;
        cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
        for (int i = 4; i < 6; ++i) lk(cs, x, n, st, i, pdl);
        cudaStreamEndCapture(cs, &g2);
        cudaGraphInstantiate(&e2, g2, 0);
        pb.push_back(e2);
      }
      run("plain A -> 4 plain graphs round-robin", [&] { cudaGraphLaunch(gea, s); cudaGraphLaunch(pb[rr++ % 4], s); });
    }
    run("eager A -> while W", [&] {
      reset<<<1, 1, 0, s>>>(cnt);
      for (int i = 0; i < 4; ++i) lk(s, x, n, st, i, pdl);
      cudaGraphLaunch(gwu, s);
    });
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("done: %s\n", cudaGetErrorString(e));
  return 0;
}
