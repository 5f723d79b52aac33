// Krylov building blocks (K3): fused classical Gram-Schmidt projections,
// orthogonalisation update + norm, basis linear combination, BLAS-1.
//
// Reference anchor: the Arnoldi/Givens arithmetic of fgmres
// (/root/reference/pkg/src/implicitrk/sparsela.py:355-394).  The reference
// uses modified Gram-Schmidt, one vector pass per projection; here the
// projections of one Arnoldi step are computed in ONE pass over the basis
// (classical Gram-Schmidt, optional second pass = CGS2).
//
// All reductions are deterministic: block partials are written to a scratch
// array and summed in block order by the last block to finish.
#include "irk_internal.cuh"

namespace irk {

constexpr int kTileElems = 4;  // elements per thread per tile

struct HostVec {
  double v[kMaxBasis];
};

// Last-block finalisation helper: returns true in the block that finished
// last (all blocks' partial stores are then visible).
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) *counter = 0u;  // re-arm for the next launch
  return is_last;
}

// h[i] = <V_i, w>
__global__ void __launch_bounds__(kBlock)
    k_multidot(int64_t n, int k, const double* __restrict__ V, int64_t ldv,
               const double* __restrict__ w, double* __restrict__ partials,
               unsigned int* counter, double* __restrict__ h) {
  __shared__ double acc[kMaxBasis][kBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < k * (kBlock / 32); i += blockDim.x)
    acc[i / (kBlock / 32)][i % (kBlock / 32)] = 0.0;
  __syncthreads();
  const int64_t tile = (int64_t)kBlock * kTileElems;
  for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < n; t0 += (int64_t)gridDim.x * tile) {
    double wv[kTileElems];
#pragma unroll
    for (int q = 0; q < kTileElems; ++q) {
      int64_t e = t0 + q * kBlock + threadIdx.x;
      wv[q] = e < n ? w[e] : 0.0;
    }
    for (int i = 0; i < k; ++i) {
      const double* vi = V + (int64_t)i * ldv;
      double p = 0.0;
#pragma unroll
      for (int q = 0; q < kTileElems; ++q) {
        int64_t e = t0 + q * kBlock + threadIdx.x;
        if (e < n) p += __ldg(vi + e) * wv[q];
      }
      p = warp_sum(p);
      if (lane == 0) acc[i][warp] += p;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < kBlock / 32; ++q) s += acc[i][q];
    partials[(int64_t)i * gridDim.x + blockIdx.x] = s;
  }
  if (last_block(counter)) {
    for (int i = warp; i < k; i += kBlock / 32) {
      double s = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) s += partials[(int64_t)i * gridDim.x + b];
      s = warp_sum(s);
      if (lane == 0) h[i] = s;
    }
  }
}

// w -= sum_i coef[i] V_i ; out_norm = ||w|| (when out_norm != NULL)
// coef is read from device memory (h) so the projections never leave the GPU.
__global__ void __launch_bounds__(kBlock)
    k_orth_update(int64_t n, int k, const double* __restrict__ V, int64_t ldv,
                  const double* __restrict__ coef, double* __restrict__ w,
                  double* __restrict__ partials, unsigned int* counter,
                  double* __restrict__ out_norm) {
  __shared__ double hc[kMaxBasis];
  __shared__ double red[8];
  for (int i = threadIdx.x; i < k; i += blockDim.x) hc[i] = coef[i];
  __syncthreads();
  double ss = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double x = w[e];
    for (int i = 0; i < k; ++i) x -= hc[i] * __ldg(V + (int64_t)i * ldv + e);
    w[e] = x;
    ss += x * x;
  }
  if (!out_norm) return;
  double v[1] = {ss};
  block_sum<1>(v, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = v[0];
  if (last_block(counter)) {
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) s += partials[b];
      s = warp_sum(s);
      if (lane == 0) *out_norm = sqrt(s);
    }
  }
}

__global__ void k_add_vec(int k, double* __restrict__ h, const double* __restrict__ h2) {
  int i = threadIdx.x;
  if (i < k) h[i] += h2[i];
}

__global__ void k_lincomb(int64_t n, int k, const double* __restrict__ Z, int64_t ldz,
                          const HostVec y, double* __restrict__ x) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double acc = x[e];
    for (int i = 0; i < k; ++i) acc += y.v[i] * __ldg(Z + (int64_t)i * ldz + e);
    x[e] = acc;
  }
}

__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b,
                        double* __restrict__ y) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    y[e] = (b == 0.0) ? a * x[e] : a * x[e] + b * y[e];
}

__global__ void k_scale_dev(int64_t n, const double* __restrict__ num,
                            const double* __restrict__ den, const double* __restrict__ x,
                            double* __restrict__ y) {
  double a = *num / *den;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    y[e] = a * x[e];
}

template <bool NORM>
__global__ void __launch_bounds__(kBlock)
    k_dot(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
          double* __restrict__ partials, unsigned int* counter, double* __restrict__ out) {
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    s += x[e] * y[e];
  double v[1] = {s};
  block_sum<1>(v, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = v[0];
  if (last_block(counter)) {
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
      double t = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) t += partials[b];
      t = warp_sum(t);
      if (lane == 0) *out = NORM ? sqrt(t) : t;
    }
  }
}

__global__ void k_nonfinite(int64_t n, const double* __restrict__ x, int* flag) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[e])) {
      *flag = 1;
      return;
    }
}

}  // namespace irk

using namespace irk;

extern "C" {

int irk_multidot(irk_ctx* ctx, int64_t n, int k, const double* V_dev, int64_t ldv,
                 const double* w_dev, double* h_dev) {
  IRK_REQUIRE(ctx && V_dev && w_dev && h_dev, "irk_multidot: NULL argument");
  IRK_REQUIRE(k >= 1 && k <= kMaxBasis, "irk_multidot: 1 <= k <= %d", kMaxBasis);
  int g = grid_for(ctx, (n + kTileElems - 1) / kTileElems, kBlock, 4);
  IRK_TRY(ensure_red(ctx, (size_t)g * k));
  k_multidot<<<g, kBlock, 0, ctx->stream>>>(n, k, V_dev, ldv, w_dev, ctx->red, ctx->counters + 0,
                                            h_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_orth_update(irk_ctx* ctx, int64_t n, int k, const double* V_dev, int64_t ldv,
                    double* h_dev, double* w_dev, int reorth) {
  IRK_REQUIRE(ctx && V_dev && w_dev && h_dev, "irk_orth_update: NULL argument");
  IRK_REQUIRE(k >= 1 && k < kMaxBasis, "irk_orth_update: 1 <= k < %d", kMaxBasis);
  int g = grid_for(ctx, n, kBlock, 4);
  IRK_TRY(ensure_red(ctx, (size_t)g * kMaxBasis + 2 * kMaxBasis));
  if (reorth) {
    k_orth_update<<<g, kBlock, 0, ctx->stream>>>(n, k, V_dev, ldv, h_dev, w_dev, ctx->red,
                                                 ctx->counters + 1, nullptr);
    IRK_CHECK_LAUNCH(ctx);
    double* h2 = h_dev + kMaxBasis;  // caller provides 2*kMaxBasis scratch
    IRK_TRY(irk_multidot(ctx, n, k, V_dev, ldv, w_dev, h2));
    k_orth_update<<<g, kBlock, 0, ctx->stream>>>(n, k, V_dev, ldv, h2, w_dev, ctx->red,
                                                 ctx->counters + 1, h_dev + k);
    IRK_CHECK_LAUNCH(ctx);
    k_add_vec<<<1, kMaxBasis, 0, ctx->stream>>>(k, h_dev, h2);
    IRK_CHECK_LAUNCH(ctx);
  } else {
    k_orth_update<<<g, kBlock, 0, ctx->stream>>>(n, k, V_dev, ldv, h_dev, w_dev, ctx->red,
                                                 ctx->counters + 1, h_dev + k);
    IRK_CHECK_LAUNCH(ctx);
  }
  return IRK_OK;
}

int irk_lincomb(irk_ctx* ctx, int64_t n, int k, const double* Z_dev, int64_t ldz,
                const double* y_host, double* x_dev) {
  IRK_REQUIRE(ctx && Z_dev && y_host && x_dev, "irk_lincomb: NULL argument");
  IRK_REQUIRE(k >= 0 && k <= kMaxBasis, "irk_lincomb: 0 <= k <= %d", kMaxBasis);
  if (k == 0 || n == 0) return IRK_OK;
  HostVec y{};
  for (int i = 0; i < k; ++i) y.v[i] = y_host[i];
  k_lincomb<<<grid_for(ctx, n, kBlock, 4), kBlock, 0, ctx->stream>>>(n, k, Z_dev, ldz, y, x_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_axpby(irk_ctx* ctx, int64_t n, double a, const double* x_dev, double b, double* y_dev) {
  IRK_REQUIRE(ctx && x_dev && y_dev, "irk_axpby: NULL argument");
  if (n == 0) return IRK_OK;
  k_axpby<<<grid_for(ctx, n), kBlock, 0, ctx->stream>>>(n, a, x_dev, b, y_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_scale_dev(irk_ctx* ctx, int64_t n, const double* num_dev, const double* den_dev,
                  const double* x_dev, double* y_dev) {
  IRK_REQUIRE(ctx && num_dev && den_dev && x_dev && y_dev, "irk_scale_dev: NULL argument");
  if (n == 0) return IRK_OK;
  k_scale_dev<<<grid_for(ctx, n), kBlock, 0, ctx->stream>>>(n, num_dev, den_dev, x_dev, y_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_norm2(irk_ctx* ctx, int64_t n, const double* x_dev, double* out_dev) {
  IRK_REQUIRE(ctx && x_dev && out_dev, "irk_norm2: NULL argument");
  int g = grid_for(ctx, n, kBlock, 4);
  IRK_TRY(ensure_red(ctx, (size_t)g));
  k_dot<true><<<g, kBlock, 0, ctx->stream>>>(n, x_dev, x_dev, ctx->red, ctx->counters + 2,
                                             out_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_dot(irk_ctx* ctx, int64_t n, const double* x_dev, const double* y_dev, double* out_dev) {
  IRK_REQUIRE(ctx && x_dev && y_dev && out_dev, "irk_dot: NULL argument");
  int g = grid_for(ctx, n, kBlock, 4);
  IRK_TRY(ensure_red(ctx, (size_t)g));
  k_dot<false><<<g, kBlock, 0, ctx->stream>>>(n, x_dev, y_dev, ctx->red, ctx->counters + 2,
                                              out_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_all_finite(irk_ctx* ctx, int64_t n, const double* x_dev, int* result_host) {
  IRK_REQUIRE(ctx && x_dev && result_host, "irk_all_finite: NULL argument");
  int* flag = (int*)(ctx->counters + (kNumCounters - 2));
  IRK_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  if (n) {
    k_nonfinite<<<grid_for(ctx, n), kBlock, 0, ctx->stream>>>(n, x_dev, flag);
    IRK_CHECK_LAUNCH(ctx);
  }
  int h = 0;
  IRK_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  *result_host = h ? 0 : 1;
  return IRK_OK;
}

}  // extern "C"
