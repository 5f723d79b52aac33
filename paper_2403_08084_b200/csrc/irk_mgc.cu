// Complex geometric multigrid for the complex-symmetric Schur-pair blocks
// alpha M + beta K (alpha, beta complex) of the transformed stage
// preconditioner, and the multigrid-preconditioned COCG that replaces the
// batched Jacobi-COCG for them (irk_cocg, precond.py SCHUR kind).
//
// The reference factorises every stage block with SuperLU (sparsela.py:
// 149-191); the Schur-pair blocks are complex, so this is the complex
// counterpart of irk_mg.cu's generic V-cycle:
//   levels      M_l, K_l re-assembled on N/2^l grids (nested P1), masked rows
//               identity, masked columns eliminated; the level operator
//               alpha M_l + beta K_l is formed on the fly from the two real
//               value streams (slot-uniform headers on stencil slices)
//   smoother    Chebyshev on D^-1 A with D = diag(alpha M + beta K) complex
//               and the real interval [lmax/4, lmax], lmax a Gershgorin
//               bound of |D^-1 A|: the spectrum of D^-1 A stays near the real
//               segment (mass- and stiffness-dominated modes have the phase
//               of their own diagonal), so real Chebyshev coefficients damp
//               the high-frequency error as in the real case
//   transfer    P1 interpolation / its transpose (as irk_mg.cu)
// COCG (r^T z, unconjugated) preconditioned by one V-cycle: 6-10 iterations
// per pair block at rtol 1e-6 instead of ~115 with Jacobi (3D 96^3,
// Gauss-Legendre 4, dt = 5e-3).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <vector>

#include "irk_inner.cuh"

namespace irk {
namespace {

struct GridC {
  int dim;
  int64_t n1;
};

__device__ __forceinline__ void unflat_c(const GridC& g, int64_t v, int64_t (&c)[3]) {
  c[0] = v % g.n1;
  c[1] = g.dim > 1 ? (v / g.n1) % g.n1 : 0;
  c[2] = g.dim > 2 ? v / (g.n1 * g.n1) : 0;
}
__device__ __forceinline__ int64_t flat_c(const GridC& g, const int64_t (&c)[3]) {
  return c[0] + g.n1 * (c[1] + g.n1 * c[2]);
}

// (alpha M + beta K) x at `row` through the SELL arrays
__device__ __forceinline__ cplx row_dot_c(const MatView& A, cplx al, cplx be, int64_t row,
                                          const cplx* __restrict__ x) {
  const int64_t sl = row / kSlice;
  const int lane = (int)(row % kSlice);
  int base, width;
  if (A.ellw) {
    base = (int)(sl * kSlice * A.ellw);
    width = A.ellw;
  } else {
    base = __ldg(A.slice_ptr + sl);
    width = (__ldg(A.slice_ptr + sl + 1) - base) / kSlice;
  }
  const int q0 = base / kSlice;
  cplx acc = {0.0, 0.0};
  for (int k = 0; k < width; ++k) {
    const int pos = base + k * kSlice + lane;
    const int c = sell_col_at(A.colhdr, A.sell_col, q0 + k, pos, row);
    const double a = sell_val_at(A.ua, A.a, q0 + k, pos);
    const double b = sell_val_at(A.ub, A.b, q0 + k, pos);
    acc = s_add(acc, s_mul(s_coef(al, be, a, b), ldv(x + c)));
  }
  return acc;
}

// stencil form (one warp per slice; x carries a readable halo): the W
// gathers are issued with the slot headers, one warp vote selects the
// uniform-stencil path
template <int W>
__device__ __forceinline__ cplx st_dot_c(const MatView& A, cplx al, cplx be, int64_t sl,
                                         int64_t row, bool valid, const cplx* __restrict__ x) {
  const int lane = threadIdx.x & 31;
  const int q0 = (int)(sl * W);
  const bool hl = lane < W;
  const int hd = hl ? __ldg(A.colhdr + q0 + lane) : 0;
  const double ha = hl ? __ldg(A.ua + q0 + lane) : 0.0;
  const double hb = hl ? __ldg(A.ub + q0 + lane) : 0.0;
  cplx ps[W];
#pragma unroll
  for (int k = 0; k < W; ++k) ps[k] = ldv(x + row + A.sd[k]);
  const bool ok = __all_sync(0xffffffffu, !hl || (hd == A.sd[hl ? lane : 0] && !isnan(ha) &&
                                                  !isnan(hb)));
  cplx acc = {0.0, 0.0};
  if (ok) {
#pragma unroll
    for (int k = 0; k < W; ++k)
      acc = s_add(acc, s_mul(s_coef(al, be, __shfl_sync(0xffffffffu, ha, k),
                                    __shfl_sync(0xffffffffu, hb, k)),
                             ps[k]));
  } else if (valid) {
    acc = row_dot_c(A, al, be, row, x);
  }
  return acc;
}

// One Chebyshev step: res = b - A x_in (x_in == nullptr: zero start),
// d = cd d + cr D^-1 res, x_out = x_in + d; masked rows x_out = b.
// W > 0: stencil form (x_in with halo), else SELL rows.
template <int W>
__global__ void __launch_bounds__(kBlock)
    k_mgc_cheb(int64_t m, MatView A, cplx al, cplx be, const uint8_t* __restrict__ mask,
               const cplx* __restrict__ dinv, const cplx* __restrict__ b,
               const cplx* __restrict__ xin, cplx* __restrict__ d, cplx* __restrict__ xout,
               double cd, double cr, const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (m + kSlice - 1) / kSlice;
  const int64_t ws = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; sl < nsl; sl += ws) {
    const int64_t i = sl * kSlice + lane;
    const bool valid = i < m;
    cplx ax = {0.0, 0.0};
    if (xin) {
      if (W > 0)
        ax = st_dot_c<(W > 0 ? W : 1)>(A, al, be, sl, i, valid, xin);
      else if (valid)
        ax = row_dot_c(A, al, be, i, xin);
    }
    if (!valid) continue;
    const cplx bi = b[i];
    if (mask && mask[i]) {
      d[i] = {0.0, 0.0};
      xout[i] = bi;
      continue;
    }
    const cplx res = s_sub(bi, ax);
    cplx dn = s_mul(s_real<cplx>(cr), s_mul(dinv[i], res));
    if (cd != 0.0) dn = s_add(dn, s_mul(s_real<cplx>(cd), d[i]));
    d[i] = dn;
    xout[i] = xin ? s_add(xin[i], dn) : dn;
  }
}

template <int W>
__global__ void __launch_bounds__(kBlock)
    k_mgc_residual(int64_t m, MatView A, cplx al, cplx be, const uint8_t* __restrict__ mask,
                   const cplx* __restrict__ b, const cplx* __restrict__ x,
                   cplx* __restrict__ r, const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (m + kSlice - 1) / kSlice;
  const int64_t ws = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; sl < nsl; sl += ws) {
    const int64_t i = sl * kSlice + lane;
    const bool valid = i < m;
    cplx ax;
    if (W > 0)
      ax = st_dot_c<(W > 0 ? W : 1)>(A, al, be, sl, i, valid, x);
    else
      ax = valid ? row_dot_c(A, al, be, i, x) : cplx{0.0, 0.0};
    if (valid) r[i] = (mask && mask[i]) ? cplx{0.0, 0.0} : s_sub(b[i], ax);
  }
}

// bc = P^T rf, zero at masked coarse nodes
__global__ void __launch_bounds__(kBlock)
    k_mgc_restrict(int64_t mc, GridC gc, GridC gf, const uint8_t* __restrict__ maskc,
                   const cplx* __restrict__ rf, cplx* __restrict__ bc, const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= mc) return;
  if (maskc && maskc[v]) {
    bc[v] = {0.0, 0.0};
    return;
  }
  int64_t c[3];
  unflat_c(gc, v, c);
  const int64_t f0[3] = {2 * c[0], 2 * c[1], 2 * c[2]};
  cplx acc = rf[flat_c(gf, f0)];
  const int np = (1 << gc.dim) - 1;
  for (int p = 1; p <= np; ++p) {
    const int pd[3] = {p & 1, (p >> 1) & 1, (p >> 2) & 1};
    bool up = true, dn = true;
    int64_t fu[3], fd[3];
    for (int k = 0; k < 3; ++k) {
      fu[k] = f0[k] + pd[k];
      fd[k] = f0[k] - pd[k];
      if (k < gc.dim) {
        up &= fu[k] < gf.n1;
        dn &= fd[k] >= 0;
      }
    }
    if (up) acc = s_add(acc, s_mul(s_real<cplx>(0.5), rf[flat_c(gf, fu)]));
    if (dn) acc = s_add(acc, s_mul(s_real<cplx>(0.5), rf[flat_c(gf, fd)]));
  }
  bc[v] = acc;
}

// xf += P ec
__global__ void __launch_bounds__(kBlock)
    k_mgc_prolong(int64_t mf, GridC gf, GridC gc, const cplx* __restrict__ ec,
                  cplx* __restrict__ xf, const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= mf) return;
  int64_t f[3];
  unflat_c(gf, v, f);
  int64_t c[3], c2[3];
  bool odd = false;
  for (int k = 0; k < 3; ++k) {
    const int64_t p = f[k] & 1;
    c[k] = f[k] >> 1;
    c2[k] = c[k] + p;
    odd |= p != 0;
  }
  const cplx e0 = ec[flat_c(gc, c)];
  const cplx e = odd ? s_mul(s_real<cplx>(0.5), s_add(e0, ec[flat_c(gc, c2)])) : e0;
  xf[v] = s_add(xf[v], e);
}

// dinv = 1 / (alpha m_ii + beta k_ii) (masked rows 1); block maxima of the
// Gershgorin bound sum_j |alpha m_ij + beta k_ij| / |alpha m_ii + beta k_ii|
__global__ void __launch_bounds__(kBlock)
    k_mgc_setup(int64_t m, MatView A, cplx al, cplx be, const uint8_t* __restrict__ mask,
                cplx* __restrict__ dinv, double* __restrict__ part) {
  double mx = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool fl = mask && mask[i];
    const int64_t sl = i / kSlice;
    const int lane = (int)(i % kSlice);
    int base, width;
    if (A.ellw) {
      base = (int)(sl * kSlice * A.ellw);
      width = A.ellw;
    } else {
      base = __ldg(A.slice_ptr + sl);
      width = (__ldg(A.slice_ptr + sl + 1) - base) / kSlice;
    }
    const int q0 = base / kSlice;
    double sabs = 0.0;
    cplx dg = {0.0, 0.0};
    for (int k = 0; k < width; ++k) {
      const int pos = base + k * kSlice + lane;
      const int c = sell_col_at(A.colhdr, A.sell_col, q0 + k, pos, i);
      const cplx a = s_coef(al, be, sell_val_at(A.ua, A.a, q0 + k, pos),
                            sell_val_at(A.ub, A.b, q0 + k, pos));
      sabs += sqrt(s_abs2(a));
      if (c == i) dg = s_add(dg, a);
    }
    dinv[i] = fl ? cplx{1.0, 0.0} : s_div(cplx{1.0, 0.0}, dg);
    if (!fl) mx = fmax(mx, sabs / sqrt(s_abs2(dg)));
  }
  __shared__ double red[kBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) t = fmax(t, red[w]);
    part[blockIdx.x] = t;
  }
}

struct McLevel {
  int64_t m = 0;
  GridC g{};
  MatView A{};
  const uint8_t* mask = nullptr;
  cplx* dinv = nullptr;
  cplx* b = nullptr;
  cplx* x[2] = {nullptr, nullptr};
  cplx* d = nullptr;
  cplx* r = nullptr;
  double lmax = 2.0;
  int st = 0;  // stencil width of the fast kernels (0: SELL rows)
};

std::atomic<uint64_t> g_mgc_uid{1ull << 40};

}  // namespace
}  // namespace irk

struct irk_mgc : public irk::CgPrec {
  int nu = 2, ncoarse = 4;
  int maxw = 0;  // widest row of the level-0 pattern (CG kernel dispatch)
  irk::cplx al{}, be{};
  std::vector<irk::McLevel> lev;
  void* mem = nullptr;

  static void cheb(double lo, double hi, int n, std::vector<double>& cd, std::vector<double>& cr) {
    const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
    cd.assign(n, 0.0);
    cr.assign(n, 0.0);
    double rho = 1.0 / sigma;
    cr[0] = 1.0 / theta;
    for (int k = 1; k < n; ++k) {
      const double rn = 1.0 / (2.0 * sigma - rho);
      cd[k] = rn * rho;
      cr[k] = 2.0 * rn / delta;
      rho = rn;
    }
  }

  int cheb_step(irk_ctx* ctx, cudaStream_t s, const irk::McLevel& L, const irk::cplx* b,
                const irk::cplx* xin, irk::cplx* xo, double cd, double cr, const int* stop) {
    using namespace irk;
    const int G = grid_for(ctx, L.m);
    cudaError_t e;
    if (xin && L.st == 15)
      e = launch(k_mgc_cheb<15>, G, kBlock, 0, s, L.m, L.A, al, be, L.mask, L.dinv, b, xin, L.d,
                 xo, cd, cr, stop);
    else if (xin && L.st == 7)
      e = launch(k_mgc_cheb<7>, G, kBlock, 0, s, L.m, L.A, al, be, L.mask, L.dinv, b, xin, L.d,
                 xo, cd, cr, stop);
    else if (xin && L.st == 3)
      e = launch(k_mgc_cheb<3>, G, kBlock, 0, s, L.m, L.A, al, be, L.mask, L.dinv, b, xin, L.d,
                 xo, cd, cr, stop);
    else
      e = launch(k_mgc_cheb<0>, G, kBlock, 0, s, L.m, L.A, al, be, L.mask, L.dinv, b, xin, L.d,
                 xo, cd, cr, stop);
    ctx->launches++;
    return e == cudaSuccess ? IRK_OK : IRK_ECUDA;
  }

  // n steps on level l from x[cur] (cur < 0: zero); the last writes `out`
  // when given; returns the buffer index holding the result (2 = out)
  int smooth(irk_ctx* ctx, cudaStream_t s, int l, const irk::cplx* b, int cur, int n,
             double lo_frac, irk::cplx* out, const int* stop, int* res) {
    irk::McLevel& L = lev[l];
    std::vector<double> cd, cr;
    cheb(lo_frac * L.lmax, L.lmax, n, cd, cr);
    for (int k = 0; k < n; ++k) {
      const int dst = cur == 0 ? 1 : 0;
      const irk::cplx* xin = cur < 0 ? nullptr : (cur == 2 ? out : L.x[cur]);
      irk::cplx* xo = (k == n - 1 && out) ? out : L.x[dst];
      IRK_TRY(cheb_step(ctx, s, L, b, xin, xo, cd[k], cr[k], stop));
      cur = xo == out ? 2 : dst;
    }
    *res = cur;
    return IRK_OK;
  }

  int vcycle(irk_ctx* ctx, cudaStream_t s, int l, const irk::cplx* b, irk::cplx* out,
             const int* stop, int* res) {
    using namespace irk;
    McLevel& L = lev[l];
    if (l == (int)lev.size() - 1) return smooth(ctx, s, l, b, -1, ncoarse, 0.05, out, stop, res);
    int c;
    IRK_TRY(smooth(ctx, s, l, b, -1, nu, 0.25, nullptr, stop, &c));
    const int G = grid_for(ctx, L.m);
    cudaError_t e;
    if (L.st == 15)
      e = launch(k_mgc_residual<15>, G, kBlock, 0, s, L.m, L.A, al, be, L.mask, b, L.x[c], L.r,
                 stop);
    else if (L.st == 7)
      e = launch(k_mgc_residual<7>, G, kBlock, 0, s, L.m, L.A, al, be, L.mask, b, L.x[c], L.r,
                 stop);
    else if (L.st == 3)
      e = launch(k_mgc_residual<3>, G, kBlock, 0, s, L.m, L.A, al, be, L.mask, b, L.x[c], L.r,
                 stop);
    else
      e = launch(k_mgc_residual<0>, G, kBlock, 0, s, L.m, L.A, al, be, L.mask, b, L.x[c], L.r,
                 stop);
    ctx->launches++;
    if (e != cudaSuccess) return IRK_ECUDA;
    McLevel& Cc = lev[l + 1];
    e = launch(k_mgc_restrict, (unsigned)((Cc.m + kBlock - 1) / kBlock), kBlock, 0, s, Cc.m, Cc.g,
               L.g, Cc.mask, (const cplx*)L.r, Cc.b, stop);
    ctx->launches++;
    if (e != cudaSuccess) return IRK_ECUDA;
    int cc;
    IRK_TRY(vcycle(ctx, s, l + 1, Cc.b, nullptr, stop, &cc));
    e = launch(k_mgc_prolong, (unsigned)((L.m + kBlock - 1) / kBlock), kBlock, 0, s, L.m, L.g,
               Cc.g, (const cplx*)Cc.x[cc], L.x[c], stop);
    ctx->launches++;
    if (e != cudaSuccess) return IRK_ECUDA;
    return smooth(ctx, s, l, b, c, nu, 0.25, out, stop, res);
  }

  int apply(irk_ctx* ctx, cudaStream_t s, const double* r, double* z, const int* stop) override {
    int c;
    const int e = vcycle(ctx, s, 0, reinterpret_cast<const irk::cplx*>(r),
                         reinterpret_cast<irk::cplx*>(z), stop, &c);
    if (e != IRK_OK || cudaGetLastError() != cudaSuccess) {
      irk::set_error("irk_mgc: V-cycle launch failed");
      return IRK_ECUDA;
    }
    return IRK_OK;
  }

  ~irk_mgc() override {
    if (mem) cudaFree(mem);
  }
};

using namespace irk;

extern "C" {

int irk_mgc_create(irk_ctx* ctx, int dim, int nlev, const int64_t* N_host,
                   const irk_mat* const* M_levels, const irk_mat* const* K_levels,
                   const uint8_t* const* masks, double alpha_re, double alpha_im, double beta_re,
                   double beta_im, int nu, int ncoarse, irk_mgc** out) {
  IRK_REQUIRE(ctx && N_host && M_levels && K_levels && out, "irk_mgc_create: NULL argument");
  IRK_REQUIRE(dim >= 1 && dim <= 3, "irk_mgc_create: dim must be 1, 2 or 3");
  IRK_REQUIRE(nlev >= 1 && nlev <= 16, "irk_mgc_create: 1 <= nlev <= 16");
  IRK_REQUIRE(nu >= 1 && nu <= 8 && ncoarse >= 1 && ncoarse <= 64,
              "irk_mgc_create: 1 <= nu <= 8, 1 <= ncoarse <= 64");
  irk_mgc* mg = new irk_mgc();
  mg->uid = g_mgc_uid.fetch_add(1);
  mg->nu = nu;
  mg->ncoarse = ncoarse;
  mg->al = {alpha_re, alpha_im};
  mg->maxw = M_levels[0] ? M_levels[0]->pat->maxw : 0;
  mg->be = {beta_re, beta_im};
  size_t total = 0;  // complex elements
  std::vector<int64_t> pads;
  for (int l = 0; l < nlev; ++l) {
    const int64_t n1 = N_host[l] + 1;
    int64_t m = n1;
    for (int k = 1; k < dim; ++k) m *= n1;
    const irk_mat* Ml = M_levels[l];
    const irk_mat* Kl = K_levels[l];
    if (!Ml || !Kl || Ml->pat != Kl->pat || Ml->pat->nrows != m || Ml->pat->ncols != m ||
        (l > 0 && N_host[l - 1] != 2 * N_host[l])) {
      delete mg;
      set_error("irk_mgc_create: level %d: need (N_l+1)^dim square M, K on one pattern, "
                "N_{l-1} = 2 N_l", l);
      return IRK_EINVAL;
    }
    McLevel L;
    L.m = m;
    L.g = GridC{dim, n1};
    L.A = make_view(Ml, Kl);
    L.mask = masks ? masks[l] : nullptr;
    int64_t pad = 0;
    if (L.A.sw == 3 || L.A.sw == 7 || L.A.sw == 15) {
      for (int k = 0; k < L.A.sw; ++k) pad = std::max<int64_t>(pad, std::abs(L.A.sd[k]));
      pad += 2 * kSlice;
      L.st = L.A.sw;
    }
    mg->lev.push_back(L);
    pads.push_back(pad);
    total += (size_t)(6 * m + 4 * pad + 32);
  }
  cudaError_t e = cudaMalloc(&mg->mem, total * sizeof(cplx));
  if (e != cudaSuccess) {
    delete mg;
    set_error("irk_mgc_create: %s", cudaGetErrorString(e));
    return IRK_ECUDA;
  }
  IRK_CUDA(cudaMemsetAsync(mg->mem, 0, total * sizeof(cplx), ctx->stream));
  cplx* p = reinterpret_cast<cplx*>(mg->mem);
  for (size_t l = 0; l < mg->lev.size(); ++l) {
    McLevel& L = mg->lev[l];
    cplx** v[6] = {&L.dinv, &L.b, &L.x[0], &L.x[1], &L.d, &L.r};
    for (int i = 0; i < 6; ++i) {
      const int64_t pd = (i == 2 || i == 3) ? pads[l] : 0;
      p += pd;
      *v[i] = p;
      p += L.m + pd;
    }
    p += 32;
  }
  for (size_t l = 0; l < mg->lev.size(); ++l) {
    McLevel& L = mg->lev[l];
    const int G = grid_for(ctx, L.m, kBlock, 4);
    IRK_TRY(ensure_red(ctx, (size_t)G + 64));
    k_mgc_setup<<<G, kBlock, 0, ctx->stream>>>(L.m, L.A, mg->al, mg->be, L.mask, L.dinv,
                                                ctx->red);
    IRK_CHECK_LAUNCH(ctx);
    std::vector<double> part(G);
    IRK_CUDA(cudaMemcpyAsync(part.data(), ctx->red, G * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    IRK_CUDA(cudaStreamSynchronize(ctx->stream));
    double mx = 0.0;
    for (double v : part) mx = std::fmax(mx, v);
    if (!(mx > 0.0) || !std::isfinite(mx)) {
      delete mg;
      set_error("irk_mgc_create: level %zu: bad diagonal / Gershgorin bound", l);
      return IRK_ESINGULAR;
    }
    L.lmax = mx;
  }
  *out = mg;
  return IRK_OK;
}

int irk_mgc_destroy(irk_mgc* mg) {
  delete mg;
  return IRK_OK;
}

int irk_mgc_cocg(irk_ctx* ctx, irk_mgc* mg, const double* rhs_dev, int64_t ld_rhs,
                 double* x_dev, int64_t ld_x, double rtol, double atol, int maxit,
                 int* its_host, double* relres_host) {
  IRK_REQUIRE(ctx && mg && rhs_dev && x_dev, "irk_mgc_cocg: NULL argument");
  IRK_REQUIRE(ld_rhs >= 2 && ld_x >= 2 && ld_rhs % 2 == 0 && ld_x % 2 == 0,
              "irk_mgc_cocg: leading dimensions must be even and >= 2");
  IRK_REQUIRE(((uintptr_t)rhs_dev % 16) == 0 && ((uintptr_t)x_dev % 16) == 0,
              "irk_mgc_cocg: rhs/x must be 16-byte aligned");
  IRK_REQUIRE(maxit >= 0 && rtol >= 0 && atol >= 0, "irk_mgc_cocg: bad tolerances");
  const McLevel& L0 = mg->lev[0];
  SysParams<cplx> P{};
  P.alpha[0] = mg->al;
  P.beta[0] = mg->be;
  const int mw = mg->maxw;
  const cplx* rhs = reinterpret_cast<const cplx*>(rhs_dev);
  cplx* x = reinterpret_cast<cplx*>(x_dev);
#define IRK_MGCRUN(W)                                                                        \
  return run_cg<cplx, 1, true, W>(ctx, L0.m, L0.A, P, nullptr, L0.mask, rhs, ld_rhs / 2, x, \
                                  ld_x / 2, rtol, atol, maxit, its_host, relres_host, mg)
  if (mw <= 8) IRK_MGCRUN(8);
  if (mw <= 16) IRK_MGCRUN(16);
  IRK_MGCRUN(0);
#undef IRK_MGCRUN
}

}  // extern "C"
