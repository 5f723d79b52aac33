// Inner diagonal-block solvers (K4/K5): batched Jacobi-preconditioned CG on
// real SPD blocks, Jacobi-preconditioned COCG on complex-symmetric blocks
// (the 2x2 real-Schur pairs), and Jacobi-Chebyshev.
//
// These replace the SuperLU factorisation + triangular solves the reference
// uses for every stage block (BlockFactorization / factorize_block,
// /root/reference/pkg/src/implicitrk/sparsela.py:149-191; the preconditioner
// calls block_factors[i].solve at precond.py:116).
//
// Design: nb independent systems share one sparsity pattern and are stored
// interleaved (row r, system k at r*nb + k), so ONE pass over the pattern,
// the two value arrays and the vectors advances every system.  Loop control
// (convergence, breakdown, iteration cap) lives in device memory; each
// iteration is two kernels (SpMV + p-update fused; x/r/z update) and the
// host only polls a status block once per chunk of iterations.
#include <vector>

#include "irk_internal.cuh"

namespace irk {

// ----------------------------------------------------------- scalar algebra
struct cplx {
  double re, im;
};

__host__ __device__ __forceinline__ double s_zero(double) { return 0.0; }
__host__ __device__ __forceinline__ cplx s_zero(cplx) { return {0.0, 0.0}; }
__device__ __forceinline__ double s_mul(double a, double b) { return a * b; }
__device__ __forceinline__ cplx s_mul(cplx a, cplx b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__device__ __forceinline__ double s_add(double a, double b) { return a + b; }
__device__ __forceinline__ cplx s_add(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ double s_sub(double a, double b) { return a - b; }
__device__ __forceinline__ cplx s_sub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ double s_div(double a, double b) { return a / b; }
__device__ __forceinline__ cplx s_div(cplx a, cplx b) {
  double d = b.re * b.re + b.im * b.im;
  return {(a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d};
}
__device__ __forceinline__ double s_abs2(double a) { return a * a; }
__device__ __forceinline__ double s_abs2(cplx a) { return a.re * a.re + a.im * a.im; }
__device__ __forceinline__ bool s_finite(double a) { return isfinite(a); }
__device__ __forceinline__ bool s_finite(cplx a) { return isfinite(a.re) && isfinite(a.im); }
__device__ __forceinline__ bool s_isnull(double a) { return a == 0.0; }
__device__ __forceinline__ bool s_isnull(cplx a) { return a.re == 0.0 && a.im == 0.0; }
// alpha * a + beta * b for real matrix entries a, b
__device__ __forceinline__ double s_coef(double al, double be, double a, double b) {
  return al * a + be * b;
}
__device__ __forceinline__ cplx s_coef(cplx al, cplx be, double a, double b) {
  return {al.re * a + be.re * b, al.im * a + be.im * b};
}
__device__ __forceinline__ double s_from(double x) { return x; }
__device__ __forceinline__ cplx s_fromc(double x) { return {x, 0.0}; }
__device__ __forceinline__ double s_wsum(double v) { return warp_sum(v); }
__device__ __forceinline__ cplx s_wsum(cplx v) { return {warp_sum(v.re), warp_sum(v.im)}; }

template <typename T>
__device__ __forceinline__ T s_real(double x);
template <>
__device__ __forceinline__ double s_real<double>(double x) {
  return x;
}
template <>
__device__ __forceinline__ cplx s_real<cplx>(double x) {
  return {x, 0.0};
}

constexpr int kMaxSys = 8;

template <typename T>
struct SysParams {
  T alpha[kMaxSys];
  T beta[kMaxSys];
};

// Device-resident loop state (one block of memory, polled by the host).
template <typename T>
struct SysState {
  T rho[kMaxSys];    // r^T z
  T mu[kMaxSys];     // p^T A p
  T alpha[kMaxSys];  // step
  T beta[kMaxSys];   // direction update
  double rr[kMaxSys];
  double bb[kMaxSys];
  double tol2[kMaxSys];
  int active[kMaxSys];
  int its[kMaxSys];
  int code[kMaxSys];  // 0 running/converged, 1 maxit, 2 breakdown
  int done;
  int iter;
};

__device__ __forceinline__ bool last_block_inner(unsigned int* counter) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) *counter = 0u;
  return is_last;
}

// Deterministic reduction of per-block partials part[k*G + b] -> out[k].
template <typename T>
__device__ __forceinline__ void reduce_partials(const T* part, int nb, int G, T* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = warp; k < nb; k += kBlock / 32) {
    T s = s_zero(T{});
    for (int b = lane; b < G; b += 32) s = s_add(s, part[(int64_t)k * G + b]);
    s = s_wsum(s);
    if (lane == 0) out[k] = s;
  }
}

template <typename T, int NB>
__device__ __forceinline__ void block_reduce_store(T (&v)[NB], T* part, int G) {
  __shared__ T red[kBlock / 32][NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NB; ++k) v[k] = s_wsum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NB; ++k) red[warp][k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < NB) {
    T s = s_zero(T{});
    for (int w = 0; w < kBlock / 32; ++w) s = s_add(s, red[w][threadIdx.x]);
    part[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = s;
  }
}

template <int NB>
__device__ __forceinline__ void block_reduce_store_d(double (&v)[NB], double* part, int G) {
  __shared__ double redd[kBlock / 32][NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NB; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NB; ++k) redd[warp][k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < NB) {
    double s = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) s += redd[w][threadIdx.x];
    part[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = s;
  }
}

struct MatView {
  const int* slice_ptr;
  const int* sell_col;
  const int* diag_pos;
  const double* a;  // values of A
  const double* b;  // values of Bm (or nullptr)
};

// ------------------------------------------------------------------ init
// x = 0, r = b, z = D^-1 r, p_old = 0; rho = r^T z, bb = ||b||^2.
template <typename T, int NB, bool HASB, bool MASK>
__global__ void __launch_bounds__(kBlock)
    k_cg_init(int64_t m, MatView A, const SysParams<T> P, const double* __restrict__ shift,
              const uint8_t* __restrict__ mask, const T* __restrict__ rhs, int64_t ld_rhs,
              T* __restrict__ x, T* __restrict__ r, T* __restrict__ z, T* __restrict__ pold,
              T* __restrict__ dinv, double rtol2, double atol2, SysState<T>* st,
              double* __restrict__ part, unsigned int* counter) {
  T rho[NB];
  double bb[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    rho[k] = s_zero(T{});
    bb[k] = 0.0;
  }
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
    bool mr = MASK && mask[row];
    int dp = A.diag_pos[row];
    double da = dp >= 0 ? A.a[dp] : 0.0;
    double db = (HASB && dp >= 0) ? A.b[dp] : 0.0;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      T d;
      if (mr) {
        d = s_real<T>(1.0);
      } else {
        d = s_coef(P.alpha[k], P.beta[k], da, db);
        if (shift) d = s_add(d, s_real<T>(shift[row * NB + k]));
      }
      T di = s_div(s_real<T>(1.0), d);
      T b = rhs[row * ld_rhs + k];
      T zz = s_mul(di, b);
      int64_t q = row * NB + k;
      dinv[q] = di;
      x[q] = s_zero(T{});
      r[q] = b;
      z[q] = zz;
      pold[q] = s_zero(T{});
      rho[k] = s_add(rho[k], s_mul(b, zz));
      bb[k] += s_abs2(b);
    }
  }
  const int G = gridDim.x;
  T* pr = reinterpret_cast<T*>(part);
  double* pb = reinterpret_cast<double*>(pr + (int64_t)NB * G);
  block_reduce_store<T, NB>(rho, pr, G);
  block_reduce_store_d<NB>(bb, pb, G);
  if (last_block_inner(counter)) {
    __shared__ T srho[NB];
    __shared__ double sbb[NB];
    reduce_partials<T>(pr, NB, G, srho);
    reduce_partials<double>(pb, NB, G, sbb);
    __syncthreads();
    if (threadIdx.x == 0) {
      int any = 0;
      for (int k = 0; k < NB; ++k) {
        double tol2 = fmax(rtol2 * sbb[k], atol2);
        st->rho[k] = srho[k];
        st->bb[k] = sbb[k];
        st->rr[k] = sbb[k];
        st->tol2[k] = tol2;
        st->beta[k] = s_zero(T{});
        st->alpha[k] = s_zero(T{});
        st->its[k] = 0;
        st->code[k] = 0;
        int act = (sbb[k] > tol2) ? 1 : 0;
        if (act && (!s_finite(srho[k]) || s_isnull(srho[k]))) {
          act = 0;
          st->code[k] = 2;
        }
        st->active[k] = act;
        any |= act;
      }
      st->done = any ? 0 : 1;
      st->iter = 0;
    }
  }
}

// ------------------------------------------------- SpMV + direction update
// p_new = z + beta p_old (computed on the fly for every gathered column),
// q = B p_new, mu = p_new^T q;  alpha = rho / mu by the last block.
template <typename T, int NB, bool HASB, bool MASK>
__global__ void __launch_bounds__(kBlock)
    k_cg_spmv(int64_t m, MatView A, const SysParams<T> P, const double* __restrict__ shift,
              const uint8_t* __restrict__ mask, const T* __restrict__ z,
              const T* __restrict__ pold, T* __restrict__ pnew, T* __restrict__ q,
              SysState<T>* st, double* __restrict__ part, unsigned int* counter) {
  if (st->done) return;
  T beta[NB];
  bool act[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    beta[k] = st->beta[k];
    act[k] = st->active[k] != 0;
  }
  T mu[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) mu[k] = s_zero(T{});
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
    T pr[NB], acc[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      int64_t qi = row * NB + k;
      pr[k] = s_add(z[qi], s_mul(beta[k], pold[qi]));
      acc[k] = s_zero(T{});
    }
    if (MASK && mask[row]) {
#pragma unroll
      for (int k = 0; k < NB; ++k) acc[k] = pr[k];
    } else {
      int64_t sl = row / kSlice;
      int lane = (int)(row % kSlice);
      int base = __ldg(A.slice_ptr + sl), width = (__ldg(A.slice_ptr + sl + 1) - base) / kSlice;
      for (int kk = 0; kk < width; ++kk) {
        int pos = base + kk * kSlice + lane;
        int c = __ldg(A.sell_col + pos);
        if (MASK && __ldg(mask + c)) continue;
        double av = __ldg(A.a + pos);
        double bv = HASB ? __ldg(A.b + pos) : 0.0;
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          int64_t qc = (int64_t)c * NB + k;
          T pc = s_add(z[qc], s_mul(beta[k], pold[qc]));
          T cf = HASB ? s_coef(P.alpha[k], P.beta[k], av, bv) : s_coef(P.alpha[k], P.beta[k], av, 0.0);
          acc[k] = s_add(acc[k], s_mul(cf, pc));
        }
      }
      if (shift) {
#pragma unroll
        for (int k = 0; k < NB; ++k)
          acc[k] = s_add(acc[k], s_mul(s_real<T>(shift[row * NB + k]), pr[k]));
      }
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      if (!act[k]) continue;
      int64_t qi = row * NB + k;
      pnew[qi] = pr[k];
      q[qi] = acc[k];
      mu[k] = s_add(mu[k], s_mul(pr[k], acc[k]));
    }
  }
  const int G = gridDim.x;
  T* pp = reinterpret_cast<T*>(part);
  block_reduce_store<T, NB>(mu, pp, G);
  if (last_block_inner(counter)) {
    __shared__ T smu[NB];
    reduce_partials<T>(pp, NB, G, smu);
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 0; k < NB; ++k) {
        if (!st->active[k]) continue;
        T muk = smu[k];
        st->mu[k] = muk;
        if (!s_finite(muk) || s_isnull(muk)) {
          st->active[k] = 0;
          st->code[k] = 2;
          st->alpha[k] = s_zero(T{});
        } else {
          st->alpha[k] = s_div(st->rho[k], muk);
        }
      }
    }
  }
}

// x += alpha p, r -= alpha q, z = D^-1 r; rho' = r^T z, rr = ||r||^2;
// convergence / cap / beta by the last block.
template <typename T, int NB>
__global__ void __launch_bounds__(kBlock)
    k_cg_update(int64_t m, const T* __restrict__ p, const T* __restrict__ q,
                const T* __restrict__ dinv, T* __restrict__ x, T* __restrict__ r,
                T* __restrict__ z, int maxit, SysState<T>* st, double* __restrict__ part,
                unsigned int* counter) {
  if (st->done) return;
  T alpha[NB];
  bool act[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    alpha[k] = st->alpha[k];
    act[k] = st->active[k] != 0;
  }
  T rho[NB];
  double rr[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    rho[k] = s_zero(T{});
    rr[k] = 0.0;
  }
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      if (!act[k]) continue;
      int64_t qi = row * NB + k;
      T pk = p[qi];
      x[qi] = s_add(x[qi], s_mul(alpha[k], pk));
      T rk = s_sub(r[qi], s_mul(alpha[k], q[qi]));
      r[qi] = rk;
      T zk = s_mul(dinv[qi], rk);
      z[qi] = zk;
      rho[k] = s_add(rho[k], s_mul(rk, zk));
      rr[k] += s_abs2(rk);
    }
  }
  const int G = gridDim.x;
  T* pr = reinterpret_cast<T*>(part);
  double* pb = reinterpret_cast<double*>(pr + (int64_t)NB * G);
  block_reduce_store<T, NB>(rho, pr, G);
  block_reduce_store_d<NB>(rr, pb, G);
  if (last_block_inner(counter)) {
    __shared__ T srho[NB];
    __shared__ double srr[NB];
    reduce_partials<T>(pr, NB, G, srho);
    reduce_partials<double>(pb, NB, G, srr);
    __syncthreads();
    if (threadIdx.x == 0) {
      int any = 0;
      for (int k = 0; k < NB; ++k) {
        if (!st->active[k]) continue;
        st->its[k] += 1;
        st->rr[k] = srr[k];
        if (!(srr[k] > st->tol2[k])) {
          st->active[k] = 0;  // converged (or NaN residual: flagged below)
          if (!isfinite(srr[k])) st->code[k] = 2;
        } else if (st->its[k] >= maxit) {
          st->active[k] = 0;
          st->code[k] = 1;
        } else if (!s_finite(srho[k]) || s_isnull(srho[k])) {
          st->active[k] = 0;
          st->code[k] = 2;
        } else {
          st->beta[k] = s_div(srho[k], st->rho[k]);
          st->rho[k] = srho[k];
        }
        any |= st->active[k];
      }
      st->iter += 1;
      if (!any) st->done = 1;
    }
  }
}

template <typename T, int NB>
__global__ void k_cg_store(int64_t m, const T* __restrict__ x, T* __restrict__ out,
                           int64_t ld_out) {
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < NB; ++k) out[row * ld_out + k] = x[row * NB + k];
  }
}

// --------------------------------------------------------------- Chebyshev
// Jacobi-Chebyshev for SPD B_k with spectrum of D^-1 B_k in [lmin, lmax]:
//   x_{j+1} = x_j + y_j,  y_j = omega_j y_{j-1} + gamma_j D^-1 (b - B x_j)
// (three-term recurrence, no inner products).
struct ChebParams {
  double theta[kMaxSys], delta[kMaxSys];
};

template <int NB, bool HASB, bool MASK>
__global__ void __launch_bounds__(kBlock)
    k_cheb_step(int64_t m, MatView A, const SysParams<double> P, const double* __restrict__ shift,
                const uint8_t* __restrict__ mask, const double* __restrict__ rhs, int64_t ld_rhs,
                const double* __restrict__ xin, double* __restrict__ xout,
                const double* __restrict__ yin, double* __restrict__ yout, ChebParams cp,
                double rho_prev_by, int first, const double* __restrict__ rho_vec) {
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
    bool mr = MASK && mask[row];
    double acc[NB], diag[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) acc[k] = diag[k] = 0.0;
    if (mr) {
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        acc[k] = xin[row * NB + k];
        diag[k] = 1.0;
      }
    } else {
      int64_t sl = row / kSlice;
      int lane = (int)(row % kSlice);
      int base = __ldg(A.slice_ptr + sl), width = (__ldg(A.slice_ptr + sl + 1) - base) / kSlice;
      for (int kk = 0; kk < width; ++kk) {
        int pos = base + kk * kSlice + lane;
        int c = __ldg(A.sell_col + pos);
        if (MASK && __ldg(mask + c)) continue;
        double av = __ldg(A.a + pos);
        double bv = HASB ? __ldg(A.b + pos) : 0.0;
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          double cf = P.alpha[k] * av + P.beta[k] * bv;
          acc[k] += cf * xin[(int64_t)c * NB + k];
          if (c == row) diag[k] += cf;
        }
      }
      if (shift) {
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          acc[k] += shift[row * NB + k] * xin[row * NB + k];
          diag[k] += shift[row * NB + k];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      int64_t qi = row * NB + k;
      double res = rhs[row * ld_rhs + k] - acc[k];
      double zk = res / diag[k];
      double y;
      if (first) {
        y = zk / cp.theta[k];
      } else {
        double rk = rho_vec[k];        // rho_j
        double rkm = rho_vec[NB + k];  // rho_{j-1}
        y = rk * rkm * yin[qi] + 2.0 * rk / cp.delta[k] * zk;
      }
      yout[qi] = y;
      xout[qi] = xin[qi] + y;
    }
  }
}

}  // namespace irk

using namespace irk;

// ------------------------------------------------------------ host drivers
namespace {

template <typename T>
struct Workspace {
  SysState<T>* st;
  T *x, *r, *z, *p0, *p1, *q, *dinv;
};

template <typename T>
int carve(irk_ctx* ctx, int64_t m, int nb, Workspace<T>& w) {
  size_t vec = (size_t)m * nb * sizeof(T);
  vec = (vec + 255) & ~(size_t)255;
  size_t head = (sizeof(SysState<T>) + 255) & ~(size_t)255;
  IRK_TRY(ensure_work(ctx, head + 7 * vec));
  char* b = ctx->work;
  w.st = reinterpret_cast<SysState<T>*>(b);
  b += head;
  T** v[7] = {&w.x, &w.r, &w.z, &w.p0, &w.p1, &w.q, &w.dinv};
  for (int i = 0; i < 7; ++i) {
    *v[i] = reinterpret_cast<T*>(b);
    b += vec;
  }
  return IRK_OK;
}

template <typename T, int NB, bool HASB, bool MASK>
int run_cg(irk_ctx* ctx, int64_t m, const MatView& A, const SysParams<T>& P, const double* shift,
           const uint8_t* mask, const T* rhs, int64_t ld_rhs, T* xout, int64_t ld_x, double rtol,
           double atol, int maxit, int* its_host, double* relres_host) {
  Workspace<T> w;
  IRK_TRY(carve<T>(ctx, m, NB, w));
  int G = grid_for(ctx, m, kBlock, 4);
  IRK_TRY(ensure_red(ctx, (size_t)G * NB * 4 + 64));
  IRK_TRY(ensure_pinned(ctx, 2 * sizeof(SysState<T>) + 64));
  cudaStream_t s = ctx->stream;
  unsigned int* cnt = ctx->counters + 4;
  k_cg_init<T, NB, HASB, MASK><<<G, kBlock, 0, s>>>(m, A, P, shift, mask, rhs, ld_rhs, w.x, w.r,
                                                    w.z, w.p0, w.dinv, rtol * rtol, atol * atol,
                                                    w.st, ctx->red, cnt);
  IRK_CHECK_LAUNCH(ctx);
  SysState<T>* hst[2] = {reinterpret_cast<SysState<T>*>(ctx->pinned),
                         reinterpret_cast<SysState<T>*>(ctx->pinned) + 1};
  // Chunked issue with one chunk in flight ahead of the host check.
  int chunk = m < 65536 ? 8 : 16;
  int issued = 0, c = 0;
  bool finished = false;
  T* pbuf[2] = {w.p0, w.p1};
  while (!finished) {
    for (int t = 0; t < chunk && issued < maxit; ++t, ++issued) {
      T* pold = pbuf[issued & 1];
      T* pnew = pbuf[(issued + 1) & 1];
      k_cg_spmv<T, NB, HASB, MASK><<<G, kBlock, 0, s>>>(m, A, P, shift, mask, w.z, pold, pnew,
                                                       w.q, w.st, ctx->red, cnt);
      IRK_CHECK_LAUNCH(ctx);
      k_cg_update<T, NB><<<G, kBlock, 0, s>>>(m, pnew, w.q, w.dinv, w.x, w.r, w.z, maxit, w.st,
                                              ctx->red, cnt);
      IRK_CHECK_LAUNCH(ctx);
    }
    IRK_CUDA(cudaMemcpyAsync(hst[c & 1], w.st, sizeof(SysState<T>), cudaMemcpyDeviceToHost, s));
    IRK_CUDA(cudaEventRecord(ctx->ev[c & 1], s));
    if (issued >= maxit) {
      IRK_CUDA(cudaEventSynchronize(ctx->ev[c & 1]));
      finished = true;
      c++;
      break;
    }
    if (c > 0) {
      IRK_CUDA(cudaEventSynchronize(ctx->ev[(c - 1) & 1]));
      if (hst[(c - 1) & 1]->done) finished = true;
    }
    c++;
  }
  // final state (everything issued has completed once the last event fired)
  IRK_CUDA(cudaMemcpyAsync(hst[0], w.st, sizeof(SysState<T>), cudaMemcpyDeviceToHost, s));
  k_cg_store<T, NB><<<grid_for(ctx, m), kBlock, 0, s>>>(m, w.x, xout, ld_x);
  IRK_CHECK_LAUNCH(ctx);
  IRK_CUDA(cudaStreamSynchronize(s));
  const SysState<T>& fs = *hst[0];
  int status = IRK_OK;
  for (int k = 0; k < NB; ++k) {
    if (its_host) its_host[k] = fs.its[k];
    double rel = fs.bb[k] > 0 ? sqrt(fs.rr[k] / fs.bb[k]) : 0.0;
    if (relres_host) relres_host[k] = rel;
    if (fs.code[k] == 1 || fs.active[k]) status = IRK_ENOCONV;
    if (fs.code[k] == 2 && status == IRK_OK) {
      // breakdown is tolerated when the residual already met the target
      if (!(fs.rr[k] <= fs.tol2[k])) status = IRK_ESINGULAR;
    }
  }
  if (status == IRK_ENOCONV) set_error("pcg: iteration cap %d reached", maxit);
  if (status == IRK_ESINGULAR) set_error("pcg: breakdown (indefinite or singular block)");
  return status;
}

template <typename T, int NB>
int dispatch_flags(irk_ctx* ctx, int64_t m, const MatView& A, const SysParams<T>& P,
                   const double* shift, const uint8_t* mask, const T* rhs, int64_t ld_rhs, T* x,
                   int64_t ld_x, double rtol, double atol, int maxit, int* its, double* rel) {
  bool hb = A.b != nullptr, mk = mask != nullptr;
  if (hb && mk)
    return run_cg<T, NB, true, true>(ctx, m, A, P, shift, mask, rhs, ld_rhs, x, ld_x, rtol, atol,
                                     maxit, its, rel);
  if (hb)
    return run_cg<T, NB, true, false>(ctx, m, A, P, shift, mask, rhs, ld_rhs, x, ld_x, rtol, atol,
                                      maxit, its, rel);
  if (mk)
    return run_cg<T, NB, false, true>(ctx, m, A, P, shift, mask, rhs, ld_rhs, x, ld_x, rtol, atol,
                                      maxit, its, rel);
  return run_cg<T, NB, false, false>(ctx, m, A, P, shift, mask, rhs, ld_rhs, x, ld_x, rtol, atol,
                                     maxit, its, rel);
}

template <typename T>
int dispatch_nb(irk_ctx* ctx, int nb, int64_t m, const MatView& A, const SysParams<T>& P,
                const double* shift, const uint8_t* mask, const T* rhs, int64_t ld_rhs, T* x,
                int64_t ld_x, double rtol, double atol, int maxit, int* its, double* rel) {
  switch (nb) {
#define IRK_NB(K) \
  case K:         \
    return dispatch_flags<T, K>(ctx, m, A, P, shift, mask, rhs, ld_rhs, x, ld_x, rtol, atol, maxit, its, rel);
    IRK_NB(1)
    IRK_NB(2)
    IRK_NB(3)
    IRK_NB(4)
    IRK_NB(5)
    IRK_NB(6)
    IRK_NB(7)
    IRK_NB(8)
#undef IRK_NB
  }
  set_error("inner solver: 1 <= nb <= 8");
  return IRK_EINVAL;
}

}  // namespace

extern "C" {

int irk_pcg(irk_ctx* ctx, int nb, const double* alpha_host, const double* beta_host,
            const irk_mat* A, const irk_mat* Bm, const double* shift_dev,
            const uint8_t* rowmask_dev, const double* rhs_dev, int64_t ld_rhs, double* x_dev,
            int64_t ld_x, double rtol, double atol, int maxit, int* its_host,
            double* relres_host) {
  IRK_REQUIRE(ctx && A && rhs_dev && x_dev && alpha_host, "irk_pcg: NULL argument");
  IRK_REQUIRE(nb >= 1 && nb <= kMaxSys, "irk_pcg: 1 <= nb <= %d", kMaxSys);
  IRK_REQUIRE(!Bm || (beta_host && Bm->pat == A->pat), "irk_pcg: Bm must share A's pattern");
  IRK_REQUIRE(A->pat->nrows == A->pat->ncols, "irk_pcg: square blocks required");
  IRK_REQUIRE(ld_rhs >= nb && ld_x >= nb, "irk_pcg: leading dimensions must be >= nb");
  IRK_REQUIRE(maxit >= 0 && rtol >= 0 && atol >= 0, "irk_pcg: bad tolerances");
  int64_t m = A->pat->nrows;
  SysParams<double> P{};
  for (int k = 0; k < nb; ++k) {
    P.alpha[k] = alpha_host[k];
    P.beta[k] = Bm ? beta_host[k] : 0.0;
  }
  MatView V{A->pat->slice_ptr, A->pat->sell_col, A->pat->diag_pos, A->val, Bm ? Bm->val : nullptr};
  if (m == 0) return IRK_OK;
  return dispatch_nb<double>(ctx, nb, m, V, P, shift_dev, rowmask_dev, rhs_dev, ld_rhs, x_dev,
                             ld_x, rtol, atol, maxit, its_host, relres_host);
}

int irk_cocg(irk_ctx* ctx, int np, const double* alpha_re_host, const double* alpha_im_host,
             const double* beta_re_host, const double* beta_im_host, const irk_mat* A,
             const irk_mat* Bm, const uint8_t* rowmask_dev, const double* rhs_dev,
             int64_t ld_rhs, double* x_dev, int64_t ld_x, double rtol, double atol, int maxit,
             int* its_host, double* relres_host) {
  IRK_REQUIRE(ctx && A && rhs_dev && x_dev && alpha_re_host && alpha_im_host,
              "irk_cocg: NULL argument");
  IRK_REQUIRE(np >= 1 && np <= 4, "irk_cocg: 1 <= np <= 4");
  IRK_REQUIRE(!Bm || (beta_re_host && beta_im_host && Bm->pat == A->pat),
              "irk_cocg: Bm must share A's pattern");
  IRK_REQUIRE(ld_rhs >= 2 * np && ld_x >= 2 * np && ld_rhs % 2 == 0 && ld_x % 2 == 0,
              "irk_cocg: leading dimensions must be even and >= 2*np");
  IRK_REQUIRE(((uintptr_t)rhs_dev % 16) == 0 && ((uintptr_t)x_dev % 16) == 0,
              "irk_cocg: rhs/x must be 16-byte aligned");
  int64_t m = A->pat->nrows;
  SysParams<cplx> P{};
  for (int k = 0; k < np; ++k) {
    P.alpha[k] = {alpha_re_host[k], alpha_im_host[k]};
    P.beta[k] = Bm ? cplx{beta_re_host[k], beta_im_host[k]} : cplx{0.0, 0.0};
  }
  MatView V{A->pat->slice_ptr, A->pat->sell_col, A->pat->diag_pos, A->val, Bm ? Bm->val : nullptr};
  if (m == 0) return IRK_OK;
  return dispatch_nb<cplx>(ctx, np, m, V, P, nullptr, rowmask_dev,
                           reinterpret_cast<const cplx*>(rhs_dev), ld_rhs / 2,
                           reinterpret_cast<cplx*>(x_dev), ld_x / 2, rtol, atol, maxit, its_host,
                           relres_host);
}

int irk_chebyshev(irk_ctx* ctx, int nb, const double* alpha_host, const double* beta_host,
                  const irk_mat* A, const irk_mat* Bm, const double* shift_dev,
                  const uint8_t* rowmask_dev, const double* lmin_host, const double* lmax_host,
                  const double* rhs_dev, int64_t ld_rhs, double* x_dev, int64_t ld_x,
                  int iters) {
  IRK_REQUIRE(ctx && A && rhs_dev && x_dev && alpha_host && lmin_host && lmax_host,
              "irk_chebyshev: NULL argument");
  IRK_REQUIRE(nb >= 1 && nb <= 4, "irk_chebyshev: 1 <= nb <= 4");
  IRK_REQUIRE(!Bm || (beta_host && Bm->pat == A->pat), "irk_chebyshev: Bm must share A's pattern");
  IRK_REQUIRE(iters >= 1, "irk_chebyshev: iters >= 1");
  IRK_REQUIRE(ld_x == nb, "irk_chebyshev: ld_x must equal nb");
  int64_t m = A->pat->nrows;
  if (m == 0) return IRK_OK;
  SysParams<double> P{};
  ChebParams cp{};
  for (int k = 0; k < nb; ++k) {
    P.alpha[k] = alpha_host[k];
    P.beta[k] = Bm ? beta_host[k] : 0.0;
    IRK_REQUIRE(lmax_host[k] > lmin_host[k] && lmin_host[k] > 0,
                "irk_chebyshev: need 0 < lmin < lmax");
    cp.theta[k] = 0.5 * (lmax_host[k] + lmin_host[k]);
    cp.delta[k] = 0.5 * (lmax_host[k] - lmin_host[k]);
  }
  MatView V{A->pat->slice_ptr, A->pat->sell_col, A->pat->diag_pos, A->val, Bm ? Bm->val : nullptr};
  size_t vec = ((size_t)m * nb * sizeof(double) + 255) & ~(size_t)255;
  IRK_TRY(ensure_work(ctx, 4 * vec + 4096));
  double* xa = reinterpret_cast<double*>(ctx->work);
  double* xb = reinterpret_cast<double*>(ctx->work + vec);
  double* ya = reinterpret_cast<double*>(ctx->work + 2 * vec);
  double* yb = reinterpret_cast<double*>(ctx->work + 3 * vec);
  double* rho_dev = reinterpret_cast<double*>(ctx->work + 4 * vec);
  IRK_CUDA(cudaMemsetAsync(xa, 0, (size_t)m * nb * sizeof(double), ctx->stream));
  IRK_CUDA(cudaMemsetAsync(ya, 0, (size_t)m * nb * sizeof(double), ctx->stream));
  // rho_j recurrence (host-computed, per system): rho_0 = 1/sigma,
  // rho_j = 1 / (2 sigma - rho_{j-1}), sigma = theta/delta.
  double rho_prev[kMaxSys], rho_cur[kMaxSys];
  for (int k = 0; k < nb; ++k) rho_prev[k] = cp.delta[k] / cp.theta[k];
  int G = grid_for(ctx, m, kBlock, 4);
  double* xin = xa;
  double* xo = xb;
  double* yin = ya;
  double* yo = yb;
  std::vector<double> rv(2 * kMaxSys);
  for (int j = 0; j < iters; ++j) {
    for (int k = 0; k < nb; ++k) {
      double sigma = cp.theta[k] / cp.delta[k];
      rho_cur[k] = (j == 0) ? rho_prev[k] : 1.0 / (2.0 * sigma - rho_prev[k]);
      rv[k] = rho_cur[k];
      rv[nb + k] = rho_prev[k];
    }
    // stream-ordered upload of the two coefficient vectors
    double* rslot = rho_dev + (j & 1) * 2 * kMaxSys;
    IRK_CUDA(cudaMemcpyAsync(rslot, rv.data(), 2 * kMaxSys * sizeof(double),
                             cudaMemcpyHostToDevice, ctx->stream));
    bool hb = Bm != nullptr, mk = rowmask_dev != nullptr;
#define IRK_CHEB(NBV)                                                                          \
  if (nb == NBV) {                                                                             \
    if (hb && mk)                                                                              \
      k_cheb_step<NBV, true, true><<<G, kBlock, 0, ctx->stream>>>(                             \
          m, V, P, shift_dev, rowmask_dev, rhs_dev, ld_rhs, xin, xo, yin, yo, cp, 0.0, j == 0, \
          rslot);                                                                              \
    else if (hb)                                                                               \
      k_cheb_step<NBV, true, false><<<G, kBlock, 0, ctx->stream>>>(                            \
          m, V, P, shift_dev, rowmask_dev, rhs_dev, ld_rhs, xin, xo, yin, yo, cp, 0.0, j == 0, \
          rslot);                                                                              \
    else if (mk)                                                                               \
      k_cheb_step<NBV, false, true><<<G, kBlock, 0, ctx->stream>>>(                            \
          m, V, P, shift_dev, rowmask_dev, rhs_dev, ld_rhs, xin, xo, yin, yo, cp, 0.0, j == 0, \
          rslot);                                                                              \
    else                                                                                       \
      k_cheb_step<NBV, false, false><<<G, kBlock, 0, ctx->stream>>>(                           \
          m, V, P, shift_dev, rowmask_dev, rhs_dev, ld_rhs, xin, xo, yin, yo, cp, 0.0, j == 0, \
          rslot);                                                                              \
  }
    IRK_CHEB(1)
    IRK_CHEB(2)
    IRK_CHEB(3)
    IRK_CHEB(4)
#undef IRK_CHEB
    IRK_CHECK_LAUNCH(ctx);
    for (int k = 0; k < nb; ++k) rho_prev[k] = rho_cur[k];
    double* t = xin;
    xin = xo;
    xo = t;
    t = yin;
    yin = yo;
    yo = t;
  }
  k_cg_store<double, 1><<<grid_for(ctx, m * nb), kBlock, 0, ctx->stream>>>(m * nb, xin, x_dev, 1);
  IRK_CHECK_LAUNCH(ctx);
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  return IRK_OK;
}

}  // extern "C"
