// Lab: attainable per-iteration time of the two CG kernels on an
// L2-resident 1M-row problem (2D 7-point P1 stencil, uniform values).
// Not part of the library.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   -o cg_lab profiles/cg_lab.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

constexpr int kB = 256;

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int MODE>  // 0 no reduction, 1 partials only, 2 partials + last block
__global__ void __launch_bounds__(kB) upd(int m, const double* __restrict__ p,
                                          const double* __restrict__ q,
                                          const double* __restrict__ d, double* __restrict__ x,
                                          double* __restrict__ r, double* __restrict__ z,
                                          double alpha, double* part, unsigned* cnt,
                                          double* out) {
  double rho = 0, rr = 0;
  const int T = gridDim.x * blockDim.x;
  for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < m; i0 += 2 * T) {
    double pk[2], qk[2], dk[2], xk[2], rk[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int i = i0 + u * T;
      if (i < m) {
        pk[u] = p[i];
        qk[u] = q[i];
        dk[u] = d[i];
        xk[u] = x[i];
        rk[u] = r[i];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int i = i0 + u * T;
      if (i < m) {
        x[i] = xk[u] + alpha * pk[u];
        double rn = rk[u] - alpha * qk[u];
        r[i] = rn;
        double zn = dk[u] * rn;
        z[i] = zn;
        rho += rn * zn;
        rr += rn * rn;
      }
    }
  }
  if (MODE == 0) return;
  __shared__ double red[8][2];
  rho = wsum(rho);
  rr = wsum(rr);
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5][0] = rho;
    red[threadIdx.x >> 5][1] = rr;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < 8; ++w) {
      a += red[w][0];
      b += red[w][1];
    }
    part[blockIdx.x] = a;
    part[gridDim.x + blockIdx.x] = b;
  }
  if (MODE == 1) return;
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  double a = 0;
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) a += __ldcg(part + b);
  a = wsum(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][0] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < 8; ++w) t += red[w][0];
    *out = t;
    *cnt = 0;
  }
}

// SpMV with on-the-fly p = z + beta pold, uniform 7-point stencil
template <int MODE>
__global__ void __launch_bounds__(kB, 4) spmv(int m, int n1, const double* __restrict__ z,
                                             const double* __restrict__ po, double* __restrict__ pn,
                                             double* __restrict__ q, double beta, double* part) {
  const int off[7] = {-n1 - 1, -n1, -1, 0, 1, n1, n1 + 1};
  const double val[7] = {-0.5, -0.5, -1.0, 4.2, -1.0, -0.5, -0.5};
  double mu = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    double acc = 0;
    double pr = z[i] + beta * po[i];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      int c = i + off[k];
      if (c >= 0 && c < m) acc += val[k] * (z[c] + beta * po[c]);
    }
    pn[i] = pr;
    q[i] = acc;
    mu += pr * acc;
  }
  if (MODE == 0) return;
  __shared__ double red[8];
  mu = wsum(mu);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mu;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0;
    for (int w = 0; w < 8; ++w) a += red[w];
    part[blockIdx.x] = a;
  }
}

// SpMV with smem tile per block: block owns rows [b*R, b*R+R); stages
// p for rows [lo - n1 - 1, hi + n1 + 1] computed once
template <int R>
__global__ void __launch_bounds__(kB) spmv_tile(int m, int n1, const double* __restrict__ z,
                                               const double* __restrict__ po,
                                               double* __restrict__ pn, double* __restrict__ q,
                                               double beta, double* part) {
  extern __shared__ double tile[];
  double mu = 0;
  for (int blk = blockIdx.x; blk * R < m; blk += gridDim.x) {
    const int lo = blk * R, hi = min(m, lo + R);
    const int t0 = lo - n1 - 1, t1 = min(m, hi + n1 + 1);
    __syncthreads();
    for (int c = t0 + threadIdx.x; c < t1; c += blockDim.x)
      tile[c - t0] = c >= 0 ? z[c] + beta * po[c] : 0.0;
    __syncthreads();
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const double* t = tile + (i - t0);
      double pr = t[0];
      double acc = 4.2 * pr - (t[-1] + t[1]) - 0.5 * (t[-n1 - 1] + t[-n1] + t[n1] + t[n1 + 1]);
      pn[i] = pr;
      q[i] = acc;
      mu += pr * acc;
    }
  }
  __shared__ double red[8];
  mu = wsum(mu);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mu;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0;
    for (int w = 0; w < 8; ++w) a += red[w];
    part[blockIdx.x] = a;
  }
}


struct Offs {
  int d[8];
};
// runtime offsets (kernel params), per-slot values from a header array
// (one value per 32-row slice and slot), z/pold separate or interleaved
template <int VAR>
__global__ void __launch_bounds__(kB, 4) spmv_rt(int m, Offs o, int w, const double* __restrict__ hv,
                                                const double* __restrict__ z,
                                                const double* __restrict__ po,
                                                const double2* __restrict__ zp,
                                                double* __restrict__ pn, double* __restrict__ q,
                                                double beta, double* part) {
  double mu = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int sl = i >> 5;
    double acc = 0, pr;
    if (VAR == 0) {
      pr = z[i] + beta * po[i];
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        int c = i + o.d[k];
        if (c >= 0 && c < m) acc += __ldg(hv + sl * 8 + k) * (z[c] + beta * po[c]);
      }
    } else {
      double2 t = zp[i];
      pr = t.x + beta * t.y;
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        int c = i + o.d[k];
        if (c >= 0 && c < m) {
          double2 g = zp[c];
          acc += __ldg(hv + sl * 8 + k) * (g.x + beta * g.y);
        }
      }
    }
    pn[i] = pr;
    q[i] = acc;
    mu += pr * acc;
  }
  __shared__ double red[8];
  mu = wsum(mu);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mu;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0;
    for (int w2 = 0; w2 < 8; ++w2) a += red[w2];
    part[blockIdx.x] = a;
  }
}


// ablation of the library's stencil SpMV main loop (no prologue):
// F bit0: lane-distributed headers + vote + shuffle (else per-thread header loads)
//     bit1: fallback path present
//     bit2: mask load
template <int F>
__global__ void __launch_bounds__(kB, 4) spmv_lib(int m, Offs o, const int* __restrict__ colhdr,
                                                 const double* __restrict__ ua,
                                                 const int* __restrict__ sell_col,
                                                 const double* __restrict__ aval,
                                                 const unsigned char* __restrict__ mask,
                                                 const double* __restrict__ z,
                                                 const double* __restrict__ po,
                                                 double* __restrict__ pn, double* __restrict__ q,
                                                 double beta, double* part) {
  constexpr int W = 7;
  const int lane = threadIdx.x & 31;
  const int nsl = (m + 31) / 32;
  const int wstride = gridDim.x * (blockDim.x / 32);
  double mu = 0.0;
  for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) / 32; sl < nsl; sl += wstride) {
    const int row = sl * 32 + lane;
    const bool valid = row < m;
    const int q0 = sl * W;
    double pr = z[row] + beta * po[row];
    const bool flagged = (F & 4) ? (valid && mask[row]) : false;
    double ps[W];
#pragma unroll
    for (int kk = 0; kk < W; ++kk) {
      const int c = row + o.d[kk];
      ps[kk] = z[c] + beta * po[c];
    }
    double acc = 0.0;
    if (F & 1) {
      const bool hl = lane < W;
      const int hd = hl ? __ldg(colhdr + q0 + lane) : 0;
      const double ha = hl ? __ldg(ua + q0 + lane) : 0.0;
      const bool ok = __all_sync(0xffffffffu, !hl || (hd == o.d[lane < W ? lane : 0] && !isnan(ha)));
      if (ok) {
#pragma unroll
        for (int kk = 0; kk < W; ++kk) acc += __shfl_sync(0xffffffffu, ha, kk) * ps[kk];
      } else if ((F & 2) && valid) {
        const int base = sl * 32 * W;
#pragma unroll
        for (int kk = 0; kk < W; ++kk) {
          const int pos = base + kk * 32 + lane;
          const int c = sell_col[pos];
          acc += aval[pos] * (z[c] + beta * po[c]);
        }
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < W; ++kk) acc += __ldg(ua + q0 + kk) * ps[kk];
    }
    if (flagged) acc = pr;
    if (valid) {
      pn[row] = pr;
      q[row] = acc;
      mu += pr * acc;
    }
  }
  __shared__ double red[8];
  mu = wsum(mu);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mu;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0;
    for (int w2 = 0; w2 < 8; ++w2) a += red[w2];
    part[blockIdx.x] = a;
  }
}

int main() {
  const int n1 = 1025, m = n1 * n1;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *v[8], *part, *out;
  unsigned* cnt;
  for (auto& p : v) {
    cudaMalloc(&p, m * 8);
    cudaMemset(p, 0, m * 8);
  }
  cudaMalloc(&part, 1 << 20);
  cudaMalloc(&out, 64);
  cudaMalloc(&cnt, 64);
  cudaMemset(cnt, 0, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaStream_t cs;
  cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  auto timeit = [&](const char* name, auto launch) {
    // 200 launches captured in one graph: device time without host launch cost
    const int reps = 200;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < reps; ++i) launch(cs);
    cudaStreamEndCapture(cs, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, cs);
    cudaStreamSynchronize(cs);
    cudaEventRecord(e0, cs);
    cudaGraphLaunch(ge, cs);
    cudaEventRecord(e1, cs);
    cudaEventSynchronize(e1);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %8.2f us  %s\n", name, ms * 1e3 / reps, cudaGetErrorString(cudaGetLastError()));
  };
  for (int bps : {4, 8}) {
    int G = sms * bps;
    char nm[64];
    snprintf(nm, 64, "upd no-red G=%d", G);
    timeit(nm, [&](cudaStream_t st) { upd<0><<<G, kB, 0, st>>>(m, v[0], v[1], v[2], v[3], v[4], v[5], 1e-3, part, cnt, out); });
    snprintf(nm, 64, "upd partials G=%d", G);
    timeit(nm, [&](cudaStream_t st) { upd<1><<<G, kB, 0, st>>>(m, v[0], v[1], v[2], v[3], v[4], v[5], 1e-3, part, cnt, out); });
    snprintf(nm, 64, "upd last-block G=%d", G);
    timeit(nm, [&](cudaStream_t st) { upd<2><<<G, kB, 0, st>>>(m, v[0], v[1], v[2], v[3], v[4], v[5], 1e-3, part, cnt, out); });
    snprintf(nm, 64, "spmv gather no-red G=%d", G);
    timeit(nm, [&](cudaStream_t st) { spmv<0><<<G, kB, 0, st>>>(m, n1, v[5], v[0], v[6], v[1], 0.5, part); });
    snprintf(nm, 64, "spmv gather partials G=%d", G);
    timeit(nm, [&](cudaStream_t st) { spmv<1><<<G, kB, 0, st>>>(m, n1, v[5], v[0], v[6], v[1], 0.5, part); });
  }
  {
    int G1 = (m + kB - 1) / kB;
    timeit("upd no-red 1 row/thread", [&](cudaStream_t st) { upd<0><<<G1, kB, 0, st>>>(m, v[0], v[1], v[2], v[3], v[4], v[5], 1e-3, part, cnt, out); });
    timeit("spmv gather 1 row/thread", [&](cudaStream_t st) { spmv<1><<<G1, kB, 0, st>>>(m, n1, v[5], v[0], v[6], v[1], 0.5, part); });
  }
  {
    Offs o{{-n1 - 1, -n1, -1, 0, 1, n1, n1 + 1, 0}};
    double* hv;
    cudaMalloc(&hv, (m / 32 + 1) * 8 * 8);
    cudaMemset(hv, 0, (m / 32 + 1) * 64);
    double2* zp;
    cudaMalloc(&zp, (size_t)m * 16);
    cudaMemset(zp, 0, (size_t)m * 16);
    int G = sms * 4;
    timeit("spmv rt-offsets separate", [&](cudaStream_t st) { spmv_rt<0><<<G, kB, 0, st>>>(m, o, 7, hv, v[5], v[0], zp, v[6], v[1], 0.5, part); });
    int* colhdr; double* ua; int* scol; double* aval; unsigned char* msk;
    {
      int ns = (m + 31) / 32;
      std::vector<int> h((size_t)ns * 7);
      std::vector<double> hv((size_t)ns * 7);
      for (int q0 = 0; q0 < ns; ++q0) for (int k = 0; k < 7; ++k) { h[(size_t)q0 * 7 + k] = o.d[k]; hv[(size_t)q0 * 7 + k] = 0.1 * k; }
      cudaMalloc(&colhdr, h.size() * 4); cudaMemcpy(colhdr, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
      cudaMalloc(&ua, hv.size() * 8); cudaMemcpy(ua, hv.data(), hv.size() * 8, cudaMemcpyHostToDevice);
      cudaMalloc(&scol, (size_t)ns * 32 * 7 * 4); cudaMemset(scol, 0, (size_t)ns * 32 * 7 * 4);
      cudaMalloc(&aval, (size_t)ns * 32 * 7 * 8); cudaMemset(aval, 0, (size_t)ns * 32 * 7 * 8);
      cudaMalloc(&msk, m); cudaMemset(msk, 0, m);
    }
    // z / po with halo: use interior pointers of padded buffers
    double *zb, *pb;
    cudaMalloc(&zb, (size_t)(m + 4096) * 8); cudaMemset(zb, 0, (size_t)(m + 4096) * 8);
    cudaMalloc(&pb, (size_t)(m + 4096) * 8); cudaMemset(pb, 0, (size_t)(m + 4096) * 8);
    double* zz = zb + 2048; double* pp = pb + 2048;
    timeit("lib F=0 (thread headers)", [&](cudaStream_t st) { spmv_lib<0><<<G, kB, 0, st>>>(m, o, colhdr, ua, scol, aval, msk, zz, pp, v[6], v[1], 0.5, part); });
    timeit("lib F=1 (vote+shfl)", [&](cudaStream_t st) { spmv_lib<1><<<G, kB, 0, st>>>(m, o, colhdr, ua, scol, aval, msk, zz, pp, v[6], v[1], 0.5, part); });
    timeit("lib F=3 (vote+fallback)", [&](cudaStream_t st) { spmv_lib<3><<<G, kB, 0, st>>>(m, o, colhdr, ua, scol, aval, msk, zz, pp, v[6], v[1], 0.5, part); });
    timeit("lib F=7 (vote+fallback+mask)", [&](cudaStream_t st) { spmv_lib<7><<<G, kB, 0, st>>>(m, o, colhdr, ua, scol, aval, msk, zz, pp, v[6], v[1], 0.5, part); });
    timeit("lib F=4 (thread headers+mask)", [&](cudaStream_t st) { spmv_lib<4><<<G, kB, 0, st>>>(m, o, colhdr, ua, scol, aval, msk, zz, pp, v[6], v[1], 0.5, part); });
    timeit("spmv rt-offsets interleaved", [&](cudaStream_t st) { spmv_rt<1><<<G, kB, 0, st>>>(m, o, 7, hv, v[5], v[0], zp, v[6], v[1], 0.5, part); });
  }
  for (int R : {1024, 2048, 4096}) {
    size_t sm = (size_t)(R + 2 * n1 + 2) * 8;
    int G = sms * (sm < 50000 ? 4 : 2);
    char nm[64];
    snprintf(nm, 64, "spmv tile R=%d G=%d", R, G);
    if (R == 1024) {
      cudaFuncSetAttribute(spmv_tile<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      timeit(nm, [&](cudaStream_t st) { spmv_tile<1024><<<G, kB, sm, st>>>(m, n1, v[5], v[0], v[6], v[1], 0.5, part); });
    } else if (R == 2048) {
      cudaFuncSetAttribute(spmv_tile<2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      timeit(nm, [&](cudaStream_t st) { spmv_tile<2048><<<G, kB, sm, st>>>(m, n1, v[5], v[0], v[6], v[1], 0.5, part); });
    } else {
      cudaFuncSetAttribute(spmv_tile<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      timeit(nm, [&](cudaStream_t st) { spmv_tile<4096><<<G, kB, sm, st>>>(m, n1, v[5], v[0], v[6], v[1], 0.5, part); });
    }
  }
  return 0;
}
