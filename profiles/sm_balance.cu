// Per-SM speed probe: one 1024-thread CTA per SM (cooperative shape, large
// dynamic smem) runs an identical shared-memory + FP64 workload and records
// its duration and %smid.  Reveals SMs that are systematically slower
// (a static row partition waits for the slowest SM at every grid barrier).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smb profiles/sm_balance.cu && /tmp/smb
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
#include <algorithm>

namespace cg = cooperative_groups;

__global__ void k_probe(int iters, int n, double* out_t, int* out_sm, double* sink) {
  extern __shared__ double sm[];
  cg::grid_group g = cg::this_grid();
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  g.sync();
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      int j = (i * 7 + it) % n;
      acc += sm[j] * 1.0000001;
    }
  }
  __syncthreads();
  long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    out_t[blockIdx.x] = (double)(t1 - t0);
    out_sm[blockIdx.x] = (int)smid;
  }
  if (acc == 12345.0) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *t, *sink;
  int* smid;
  cudaMalloc(&t, sms * sizeof(double));
  cudaMalloc(&smid, sms * sizeof(int));
  cudaMalloc(&sink, 8);
  for (int kb : {0, 200}) {
    int n = kb ? kb * 1024 / 8 : 4096;
    size_t smem = (size_t)n * 8;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int iters = 200;
    void* args[] = {&iters, &n, &t, &smid, &sink};
    for (int rep = 0; rep < 2; ++rep)
      cudaLaunchCooperativeKernel((void*)k_probe, sms, 1024, args, smem, 0);
    cudaDeviceSynchronize();
    std::vector<double> ht(sms);
    std::vector<int> hs(sms);
    cudaMemcpy(ht.data(), t, sms * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hs.data(), smid, sms * 4, cudaMemcpyDeviceToHost);
    std::vector<double> srt = ht;
    std::sort(srt.begin(), srt.end());
    int arg = std::max_element(ht.begin(), ht.end()) - ht.begin();
    printf("smem %zu KB: median %.0f ns, max %.0f ns (block %d on SM %d), min %.0f (%s)\n",
           smem / 1024, srt[sms / 2], srt[sms - 1], arg, hs[arg], srt[0],
           cudaGetErrorString(cudaGetLastError()));
    for (int b = 0; b < sms; ++b)
      if (ht[b] > 1.3 * srt[sms / 2]) printf("   slow block %d SM %d: %.0f ns\n", b, hs[b], ht[b]);
  }
  return 0;
}
