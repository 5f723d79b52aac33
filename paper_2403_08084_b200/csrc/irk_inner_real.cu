// Real SPD diagonal blocks: batched Jacobi-PCG (irk_pcg) and
// Jacobi-Chebyshev (irk_chebyshev).  PCG kernels in irk_inner.cuh.

#include <algorithm>
#include <cstdlib>

#include "irk_inner.cuh"

namespace irk {

// --------------------------------------------------------------- Chebyshev
// Jacobi-Chebyshev for SPD B_k with spectrum of D^-1 B_k in [lmin, lmax]:
//   x_{j+1} = x_j + y_j,  y_0 = D^-1 r_0 / theta,
//   y_j = rho_j rho_{j-1} y_{j-1} + (2 rho_j / delta) D^-1 r_j
// (three-term recurrence, no inner products).
struct ChebParams {
  double theta[kMaxSys], delta[kMaxSys];
};

template <int NB, bool HASB>
__global__ void __launch_bounds__(kBlock)
    k_cheb_step(int64_t m, MatView A, const SysParams<double> P, const double* __restrict__ shift,
                const uint8_t* __restrict__ mask, const double* __restrict__ rhs, int64_t ld_rhs,
                const double* __restrict__ xin, double* __restrict__ xout,
                const double* __restrict__ yin, double* __restrict__ yout, ChebParams cp,
                int first, const double* __restrict__ rho_vec) {
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
    double acc[NB], diag[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) acc[k] = diag[k] = 0.0;
    if (mask && mask[row]) {
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        acc[k] = xin[row * NB + k];
        diag[k] = 1.0;
      }
    } else {
      const int64_t sl = row / kSlice;
      const int lane = (int)(row % kSlice);
      const int base = __ldg(A.slice_ptr + sl);
      const int width = (__ldg(A.slice_ptr + sl + 1) - base) / kSlice;
      const int q0 = base / kSlice;
      for (int kk = 0; kk < width; ++kk) {
        const int pos = base + kk * kSlice + lane;
        const int c = sell_col_at(A.colhdr, A.sell_col, q0 + kk, pos, row);
        const double av = sell_val_at(A.ua, A.a, q0 + kk, pos);
        const double bv = HASB ? sell_val_at(A.ub, A.b, q0 + kk, pos) : 0.0;
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          const double cf = P.alpha[k] * av + P.beta[k] * bv;
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
      const int64_t qi = row * NB + k;
      const double zk = (rhs[row * ld_rhs + k] - acc[k]) / diag[k];
      double y;
      if (first) {
        y = zk / cp.theta[k];
      } else {
        const double rk = rho_vec[k], rkm = rho_vec[NB + k];
        y = rk * rkm * yin[qi] + 2.0 * rk / cp.delta[k] * zk;
      }
      yout[qi] = y;
      xout[qi] = xin[qi] + y;
    }
  }
}

}  // namespace irk

using namespace irk;

namespace {

int dispatch_real(irk_ctx* ctx, int nb, int64_t m, int maxw, const MatView& A,
                  const SysParams<double>& P, const double* shift, const uint8_t* mask,
                  const double* rhs, int64_t ld_rhs, double* x, int64_t ld_x, double rtol,
                  double atol, int maxit, int* its, double* rel) {
  switch (nb) {
#define IRK_NB(K) \
  case K:         \
    return dispatch_flags<double, K>(ctx, m, maxw, A, P, shift, mask, rhs, ld_rhs, x, ld_x, rtol, atol, maxit, its, rel);
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
  set_error("irk_pcg: 1 <= nb <= 8");
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
  const int64_t m = A->pat->nrows;
  SysParams<double> P{};
  for (int k = 0; k < nb; ++k) {
    P.alpha[k] = alpha_host[k];
    P.beta[k] = Bm ? beta_host[k] : 0.0;
  }
  if (m == 0) return IRK_OK;
  const MatView V = make_view(A, Bm);
  return dispatch_real(ctx, nb, m, A->pat->maxw, V, P, shift_dev, rowmask_dev, rhs_dev, ld_rhs,
                       x_dev, ld_x, rtol, atol, maxit, its_host, relres_host);
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
  IRK_REQUIRE(ld_rhs >= nb && ld_x >= nb, "irk_chebyshev: leading dimensions must be >= nb");
  const int64_t m = A->pat->nrows;
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
  const MatView V = make_view(A, Bm);
  // three-term recurrence coefficients, precomputed on the host:
  // rho_0 = 1/sigma, rho_j = 1 / (2 sigma - rho_{j-1}), sigma = theta/delta
  double rho_prev[kMaxSys], rho_cur[kMaxSys];
  for (int k = 0; k < nb; ++k) rho_prev[k] = cp.delta[k] / cp.theta[k];
  std::vector<double> rv((size_t)iters * 2 * kMaxSys);
  for (int j = 0; j < iters; ++j) {
    double* rj = rv.data() + (size_t)j * 2 * kMaxSys;
    for (int k = 0; k < nb; ++k) {
      const double sigma = cp.theta[k] / cp.delta[k];
      rho_cur[k] = (j == 0) ? rho_prev[k] : 1.0 / (2.0 * sigma - rho_prev[k]);
      rj[k] = rho_cur[k];
      rj[nb + k] = rho_prev[k];
      rho_prev[k] = rho_cur[k];
    }
  }
  const size_t vec = ((size_t)m * nb * sizeof(double) + 255) & ~(size_t)255;
  IRK_TRY(ensure_work(ctx, 4 * vec + rv.size() * sizeof(double) + 256));
  double* xa = reinterpret_cast<double*>(ctx->work);
  double* xb = reinterpret_cast<double*>(ctx->work + vec);
  double* ya = reinterpret_cast<double*>(ctx->work + 2 * vec);
  double* yb = reinterpret_cast<double*>(ctx->work + 3 * vec);
  double* rho_dev = reinterpret_cast<double*>(ctx->work + 4 * vec);
  double *xin = xa, *xo = xb, *yin = ya, *yo = yb;
  IRK_CUDA(cudaMemsetAsync(xa, 0, (size_t)m * nb * sizeof(double), ctx->stream));
  IRK_CUDA(cudaMemsetAsync(ya, 0, (size_t)m * nb * sizeof(double), ctx->stream));
  IRK_CUDA(cudaMemcpyAsync(rho_dev, rv.data(), rv.size() * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
  const int G = grid_for(ctx, m, kBlock, 4);
  for (int j = 0; j < iters; ++j) {
    const double* rslot = rho_dev + (size_t)j * 2 * kMaxSys;
#define IRK_CHEB(NBV)                                                                         \
  if (nb == NBV) {                                                                            \
    if (Bm)                                                                                   \
      k_cheb_step<NBV, true><<<G, kBlock, 0, ctx->stream>>>(m, V, P, shift_dev, rowmask_dev,  \
                                                            rhs_dev, ld_rhs, xin, xo, yin, yo, \
                                                            cp, j == 0, rslot);               \
    else                                                                                      \
      k_cheb_step<NBV, false><<<G, kBlock, 0, ctx->stream>>>(m, V, P, shift_dev, rowmask_dev, \
                                                             rhs_dev, ld_rhs, xin, xo, yin,   \
                                                             yo, cp, j == 0, rslot);          \
  }
    IRK_CHEB(1)
    IRK_CHEB(2)
    IRK_CHEB(3)
    IRK_CHEB(4)
#undef IRK_CHEB
    IRK_CHECK_LAUNCH(ctx);
    std::swap(xin, xo);
    std::swap(yin, yo);
  }
  // strided store: row r of the nb systems goes to x_dev[r * ld_x + k]
  IRK_CUDA(cudaMemcpy2DAsync(x_dev, (size_t)ld_x * sizeof(double), xin, nb * sizeof(double),
                             nb * sizeof(double), (size_t)m, cudaMemcpyDeviceToDevice,
                             ctx->stream));
  return IRK_OK;
}

}  // extern "C"
