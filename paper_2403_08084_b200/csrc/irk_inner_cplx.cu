// Complex-symmetric diagonal blocks: batched Jacobi-COCG (irk_cocg) for the
// 2x2 real-Schur pairs of the transformed stage preconditioner.  Kernels in
// irk_inner.cuh instantiated with T = cplx.
#include "irk_inner.cuh"

using namespace irk;

namespace {

int dispatch_cplx(irk_ctx* ctx, int np, int64_t m, int maxw, const MatView& A,
                  const SysParams<cplx>& P, const uint8_t* mask, const cplx* rhs, int64_t ld_rhs,
                  cplx* x, int64_t ld_x, double rtol, double atol, int maxit, int* its,
                  double* rel) {
  switch (np) {
#define IRK_NP(K) \
  case K:         \
    return dispatch_flags<cplx, K>(ctx, m, maxw, A, P, nullptr, mask, rhs, ld_rhs, x, ld_x, rtol, atol, maxit, its, rel);
    IRK_NP(1)
    IRK_NP(2)
    IRK_NP(3)
    IRK_NP(4)
#undef IRK_NP
  }
  set_error("irk_cocg: 1 <= np <= 4");
  return IRK_EINVAL;
}

}  // namespace

extern "C" {

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
  const int64_t m = A->pat->nrows;
  SysParams<cplx> P{};
  for (int k = 0; k < np; ++k) {
    P.alpha[k] = {alpha_re_host[k], alpha_im_host[k]};
    P.beta[k] = Bm ? cplx{beta_re_host[k], beta_im_host[k]} : cplx{0.0, 0.0};
  }
  if (m == 0) return IRK_OK;
  return dispatch_cplx(ctx, np, m, A->pat->maxw, make_view(A, Bm), P, rowmask_dev,
                       reinterpret_cast<const cplx*>(rhs_dev), ld_rhs / 2,
                       reinterpret_cast<cplx*>(x_dev), ld_x / 2, rtol, atol, maxit, its_host,
                       relres_host);
}

}  // extern "C"
