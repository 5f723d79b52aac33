// Geometric multigrid preconditioner for the P1 stage blocks
// alpha M + beta K (Dirichlet rows identity) on the structured grids, and
// the multigrid-preconditioned CG that replaces Jacobi-PCG for them.
//
// This is a B200-side replacement of the reference's exact SuperLU block
// solves (BlockFactorization / factorize_block, sparsela.py:149-191): the
// inner solve is an inexact preconditioner of the outer FGMRES, so any
// SPD preconditioner that reaches the inner tolerance is admissible; the
// multigrid one needs O(10) instead of O(sqrt(kappa)) = O(250) iterations.
//
// Hierarchy (built by the Python layer, sparsela.BlockFactorization): level
// l is the same operator re-assembled on the grid with N_l = N_0 / 2^l cells
// per direction (P1 on nested right triangles / Kuhn tetrahedra, so the
// re-discretised operator is the Galerkin one), coarse Dirichlet nodes where
// the coincident fine node is constrained.
//   prolongation: fine vertex f = 2c + p, p in {0,1}^d: p = 0 -> e[c];
//                 else the midpoint of the coarse edge (c, c+p) -> (e[c] + e[c+p]) / 2
//                 (every nonzero 0/1 direction is an edge of the triangulation)
//   restriction:  its transpose, then zero at constrained coarse nodes
//   smoother:     Chebyshev on D^-1 A over [lmax/4, lmax] (Gershgorin lmax),
//                 nu steps pre and post (symmetric cycle); constrained rows
//                 are solved exactly (identity rows)
//   coarsest:     `ncoarse` Chebyshev steps (the coarsest operator is
//                 mass-dominated: beta / (alpha H^2) small)
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "irk_inner.cuh"

namespace irk {

struct GridIdx {
  int dim;
  int64_t n1;  // vertices per direction
};

__device__ __forceinline__ void unflat(const GridIdx& g, int64_t v, int64_t (&c)[3]) {
  c[0] = v % g.n1;
  c[1] = g.dim > 1 ? (v / g.n1) % g.n1 : 0;
  c[2] = g.dim > 2 ? v / (g.n1 * g.n1) : 0;
}
__device__ __forceinline__ int64_t flat(const GridIdx& g, const int64_t (&c)[3]) {
  return c[0] + g.n1 * (c[1] + g.n1 * c[2]);
}

// row product (A x)_row through the SELL headers
__device__ __forceinline__ double row_dot(const MatView& A, int64_t row,
                                          const double* __restrict__ x) {
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
  double acc = 0.0;
  for (int k = 0; k < width; ++k) {
    const int pos = base + k * kSlice + lane;
    const int c = sell_col_at(A.colhdr, A.sell_col, q0 + k, pos, row);
    acc += sell_val_at(A.ua, A.a, q0 + k, pos) * __ldg(x + c);
  }
  return acc;
}

// One Chebyshev step: res = b - A x_in (x_in == nullptr: zero), then
// d = cd * d + cr * D^-1 res, x_out = x_in + d; constrained rows x_out = b.
__global__ void __launch_bounds__(kBlock)
    k_mg_cheb(int64_t m, MatView A, const uint8_t* __restrict__ mask,
              const double* __restrict__ dinv, const double* __restrict__ b,
              const double* __restrict__ xin, double* __restrict__ d, double* __restrict__ xout,
              double cd, double cr, const int* stop) {
  if (stop && *stop) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = b[i];
    if (mask && mask[i]) {
      d[i] = 0.0;
      xout[i] = bi;
      continue;
    }
    const double x0 = xin ? xin[i] : 0.0;
    const double res = xin ? bi - row_dot(A, i, xin) : bi;
    const double dn = (cd != 0.0 ? cd * d[i] : 0.0) + cr * dinv[i] * res;
    d[i] = dn;
    xout[i] = x0 + dn;
  }
}

// Stencil row product for stencil-aligned ELL patterns (A.sw == W): the
// W gathers at the stencil offsets are issued at once (x carries a readable
// halo of max|offset| + 32 elements on both sides), the slice's slot headers
// are loaded by lanes 0..W-1 and checked with one warp vote; slices that
// are not plain stencil slices take the generic path.  All 32 lanes of the
// warp must call it (one SELL slice per warp).
template <int W>
__device__ __forceinline__ double st_dot(const MatView& A, int64_t sl, int64_t row, bool valid,
                                         const double* __restrict__ x) {
  const int lane = threadIdx.x & 31;
  const int q0 = (int)(sl * W);
  const bool hl = lane < W;
  const int hd = hl ? __ldg(A.colhdr + q0 + lane) : 0;
  const double ha = hl ? __ldg(A.ua + q0 + lane) : 0.0;
  double ps[W];
#pragma unroll
  for (int k = 0; k < W; ++k) ps[k] = __ldg(x + row + A.sd[k]);
  const bool ok = __all_sync(0xffffffffu, !hl || (hd == A.sd[hl ? lane : 0] && !isnan(ha)));
  double acc = 0.0;
  if (ok) {
#pragma unroll
    for (int k = 0; k < W; ++k) acc += __shfl_sync(0xffffffffu, ha, k) * ps[k];
  } else if (valid) {
    acc = row_dot(A, row, x);
  }
  return acc;
}

template <int W>
__global__ void __launch_bounds__(kBlock)
    k_mg_cheb_st(int64_t m, MatView A, const uint8_t* __restrict__ mask,
                 const double* __restrict__ dinv, const double* __restrict__ b,
                 const double* __restrict__ xin, double* __restrict__ d,
                 double* __restrict__ xout, double cd, double cr, const int* stop) {
  if (stop && *stop) return;
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (m + kSlice - 1) / kSlice;
  const int64_t ws = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; sl < nsl; sl += ws) {
    const int64_t i = sl * kSlice + lane;
    const bool valid = i < m;
    const double ax = st_dot<W>(A, sl, i, valid, xin);
    if (!valid) continue;
    const double bi = b[i];
    if (mask && mask[i]) {
      d[i] = 0.0;
      xout[i] = bi;
      continue;
    }
    const double dn = (cd != 0.0 ? cd * d[i] : 0.0) + cr * dinv[i] * (bi - ax);
    d[i] = dn;
    xout[i] = xin[i] + dn;
  }
}

template <int W>
__global__ void __launch_bounds__(kBlock)
    k_mg_residual_st(int64_t m, MatView A, const uint8_t* __restrict__ mask,
                     const double* __restrict__ b, const double* __restrict__ x,
                     double* __restrict__ r, const int* stop) {
  if (stop && *stop) return;
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (m + kSlice - 1) / kSlice;
  const int64_t ws = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; sl < nsl; sl += ws) {
    const int64_t i = sl * kSlice + lane;
    const bool valid = i < m;
    const double ax = st_dot<W>(A, sl, i, valid, x);
    if (valid) r[i] = (mask && mask[i]) ? 0.0 : b[i] - ax;
  }
}

// r = b - A x (constrained rows: 0)
__global__ void __launch_bounds__(kBlock)
    k_mg_residual(int64_t m, MatView A, const uint8_t* __restrict__ mask,
                  const double* __restrict__ b, const double* __restrict__ x,
                  double* __restrict__ r, const int* stop) {
  if (stop && *stop) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    r[i] = (mask && mask[i]) ? 0.0 : b[i] - row_dot(A, i, x);
}

// bc = P^T rf, zero at constrained coarse nodes
__global__ void __launch_bounds__(kBlock)
    k_mg_restrict(int64_t mc, GridIdx gc, GridIdx gf, const uint8_t* __restrict__ maskc,
                  const double* __restrict__ rf, double* __restrict__ bc, const int* stop) {
  if (stop && *stop) return;
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= mc) return;
  if (maskc && maskc[v]) {
    bc[v] = 0.0;
    return;
  }
  int64_t c[3];
  unflat(gc, v, c);
  const int64_t f0[3] = {2 * c[0], 2 * c[1], 2 * c[2]};
  double acc = rf[flat(gf, f0)];
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
    if (up) acc += 0.5 * rf[flat(gf, fu)];
    if (dn) acc += 0.5 * rf[flat(gf, fd)];
  }
  bc[v] = acc;
}

// xf += P ec
__global__ void __launch_bounds__(kBlock)
    k_mg_prolong(int64_t mf, GridIdx gf, GridIdx gc, const double* __restrict__ ec,
                 double* __restrict__ xf, const int* stop) {
  if (stop && *stop) return;
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= mf) return;
  int64_t f[3];
  unflat(gf, v, f);
  int64_t c[3], c2[3];
  bool odd = false;
  for (int k = 0; k < 3; ++k) {
    const int64_t p = f[k] & 1;
    c[k] = f[k] >> 1;
    c2[k] = c[k] + p;
    odd |= p != 0;
  }
  const double e = odd ? 0.5 * (ec[flat(gc, c)] + ec[flat(gc, c2)]) : ec[flat(gc, c)];
  xf[v] += e;
}

// per row sum_j |a_ij| / |a_ii| (unconstrained rows), block maxima
__global__ void __launch_bounds__(kBlock)
    k_mg_gershgorin(int64_t m, MatView A, const uint8_t* __restrict__ mask,
                    double* __restrict__ dinv, double* __restrict__ part) {
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
    double sabs = 0.0, dg = 0.0;
    for (int k = 0; k < width; ++k) {
      const int pos = base + k * kSlice + lane;
      const int c = sell_col_at(A.colhdr, A.sell_col, q0 + k, pos, i);
      const double a = sell_val_at(A.ua, A.a, q0 + k, pos);
      sabs += fabs(a);
      if (c == i) dg += a;
    }
    dinv[i] = fl ? 1.0 : 1.0 / dg;
    if (!fl) mx = fmax(mx, sabs / fabs(dg));
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

struct MgLevel {
  int64_t m = 0;
  GridIdx g{};
  MatView A{};
  const uint8_t* mask = nullptr;
  double* dinv = nullptr;
  double* b = nullptr;  // rhs (coarse levels)
  double* x[2] = {nullptr, nullptr};
  double* d = nullptr;
  double* r = nullptr;
  double lmax = 2.0;
  int st = 0;  // stencil width of the fast kernels (0: generic row products)
};

static std::atomic<uint64_t> g_mg_uid{1};

}  // namespace irk

struct irk_mg : public irk::CgPrec {
  int dim = 0;
  int nu = 2, ncoarse = 8;
  std::vector<irk::MgLevel> lev;
  std::vector<const irk_mat*> mats;
  double* mem = nullptr;

  // Chebyshev coefficients (cd_k, cr_k) of steps k = 0..n-1 on [lo, hi]
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

  // n Chebyshev steps on level l starting from buffer x[cur] (cur < 0: zero
  // start); the last step writes `out` when given.  Returns the index of
  // the buffer holding the result (2 = out), or -1 on a launch error.
  int smooth(irk_ctx* ctx, cudaStream_t s, int l, const double* b, int cur, int n,
             double lo_frac, double* out, const int* stop) {
    using namespace irk;
    MgLevel& L = lev[l];
    std::vector<double> cd, cr;
    cheb(lo_frac * L.lmax, L.lmax, n, cd, cr);
    for (int k = 0; k < n; ++k) {
      const int dst = cur == 0 ? 1 : 0;
      const double* xin = cur < 0 ? nullptr : L.x[cur];
      double* xo = (k == n - 1 && out) ? out : L.x[dst];
      if (xin && L.st == 7)
        k_mg_cheb_st<7><<<grid_for(ctx, L.m), kBlock, 0, s>>>(L.m, L.A, L.mask, L.dinv, b, xin,
                                                             L.d, xo, cd[k], cr[k], stop);
      else if (xin && L.st == 15)
        k_mg_cheb_st<15><<<grid_for(ctx, L.m), kBlock, 0, s>>>(L.m, L.A, L.mask, L.dinv, b, xin,
                                                              L.d, xo, cd[k], cr[k], stop);
      else if (xin && L.st == 3)
        k_mg_cheb_st<3><<<grid_for(ctx, L.m), kBlock, 0, s>>>(L.m, L.A, L.mask, L.dinv, b, xin,
                                                             L.d, xo, cd[k], cr[k], stop);
      else
        k_mg_cheb<<<grid_for(ctx, L.m), kBlock, 0, s>>>(L.m, L.A, L.mask, L.dinv, b, xin, L.d,
                                                        xo, cd[k], cr[k], stop);
      if (cudaPeekAtLastError() != cudaSuccess) return -1;
      ctx->launches++;
      cur = xo == out ? 2 : dst;
    }
    return cur;
  }

  // x_l = V_l(b_l) from a zero start; the result lands in `out` (when
  // given) or in lev[l].x[returned index].
  int vcycle(irk_ctx* ctx, cudaStream_t s, int l, const double* b, double* out,
             const int* stop) {
    using namespace irk;
    MgLevel& L = lev[l];
    if (l == (int)lev.size() - 1) return smooth(ctx, s, l, b, -1, ncoarse, 0.05, out, stop);
    const int c = smooth(ctx, s, l, b, -1, nu, 0.25, nullptr, stop);
    if (c < 0) return -1;
    if (L.st == 7)
      k_mg_residual_st<7><<<grid_for(ctx, L.m), kBlock, 0, s>>>(L.m, L.A, L.mask, b, L.x[c],
                                                                 L.r, stop);
    else if (L.st == 15)
      k_mg_residual_st<15><<<grid_for(ctx, L.m), kBlock, 0, s>>>(L.m, L.A, L.mask, b, L.x[c],
                                                                  L.r, stop);
    else if (L.st == 3)
      k_mg_residual_st<3><<<grid_for(ctx, L.m), kBlock, 0, s>>>(L.m, L.A, L.mask, b, L.x[c],
                                                                 L.r, stop);
    else
      k_mg_residual<<<grid_for(ctx, L.m), kBlock, 0, s>>>(L.m, L.A, L.mask, b, L.x[c], L.r,
                                                          stop);
    ctx->launches++;
    MgLevel& Cc = lev[l + 1];
    k_mg_restrict<<<(unsigned)((Cc.m + kBlock - 1) / kBlock), kBlock, 0, s>>>(
        Cc.m, Cc.g, L.g, Cc.mask, L.r, Cc.b, stop);
    ctx->launches++;
    const int cc = vcycle(ctx, s, l + 1, Cc.b, nullptr, stop);
    if (cc < 0) return -1;
    k_mg_prolong<<<(unsigned)((L.m + kBlock - 1) / kBlock), kBlock, 0, s>>>(
        L.m, L.g, Cc.g, Cc.x[cc], L.x[c], stop);
    ctx->launches++;
    return smooth(ctx, s, l, b, c, nu, 0.25, out, stop);
  }

  int apply(irk_ctx* ctx, cudaStream_t s, const double* r, double* z,
            const int* stop) override {
    const int c = vcycle(ctx, s, 0, r, z, stop);
    if (c < 0 || cudaGetLastError() != cudaSuccess) {
      irk::set_error("irk_mg: V-cycle launch failed");
      return IRK_ECUDA;
    }
    return IRK_OK;
  }

  ~irk_mg() override {
    if (mem) cudaFree(mem);
  }
};

using namespace irk;

extern "C" {

int irk_mg_create(irk_ctx* ctx, int dim, int nlev, const int64_t* N_host,
                  const irk_mat* const* A_levels, const uint8_t* const* masks, int nu,
                  int ncoarse, irk_mg** out) {
  IRK_REQUIRE(ctx && N_host && A_levels && out, "irk_mg_create: NULL argument");
  IRK_REQUIRE(dim >= 1 && dim <= 3, "irk_mg_create: dim must be 1, 2 or 3");
  IRK_REQUIRE(nlev >= 1 && nlev <= 16, "irk_mg_create: 1 <= nlev <= 16");
  IRK_REQUIRE(nu >= 1 && nu <= 8 && ncoarse >= 1 && ncoarse <= 64,
              "irk_mg_create: 1 <= nu <= 8, 1 <= ncoarse <= 64");
  irk_mg* mg = new irk_mg();
  mg->uid = g_mg_uid.fetch_add(1);
  mg->dim = dim;
  mg->nu = nu;
  mg->ncoarse = ncoarse;
  size_t total = 0;
  std::vector<int64_t> pads;
  for (int l = 0; l < nlev; ++l) {
    const int64_t n1 = N_host[l] + 1;
    int64_t m = n1;
    for (int k = 1; k < dim; ++k) m *= n1;
    if (!A_levels[l] || A_levels[l]->pat->nrows != m || A_levels[l]->pat->ncols != m ||
        (l > 0 && N_host[l - 1] != 2 * N_host[l])) {
      delete mg;
      set_error("irk_mg_create: level %d: need an (N_l+1)^dim square matrix, N_{l-1} = 2 N_l", l);
      return IRK_EINVAL;
    }
    MgLevel L;
    L.m = m;
    L.g = GridIdx{dim, n1};
    L.A = make_view(A_levels[l], nullptr);
    L.mask = masks ? masks[l] : nullptr;
    mg->lev.push_back(L);
    // the iterate buffers carry a halo for the speculative stencil gathers
    int64_t pad = 0;
    if (L.A.sw == 3 || L.A.sw == 7 || L.A.sw == 15) {
      for (int k = 0; k < L.A.sw; ++k) pad = std::max<int64_t>(pad, std::abs(L.A.sd[k]));
      pad += 2 * kSlice;
      L.st = L.A.sw;
    }
    mg->lev.back().st = L.st;
    pads.push_back(pad);
    total += (size_t)(6 * m + 4 * pad + 64);
  }
  cudaError_t e = cudaMalloc(&mg->mem, total * sizeof(double));
  if (e != cudaSuccess) {
    delete mg;
    set_error("irk_mg_create: %s", cudaGetErrorString(e));
    return IRK_ECUDA;
  }
  IRK_CUDA(cudaMemsetAsync(mg->mem, 0, total * sizeof(double), ctx->stream));
  double* p = mg->mem;
  for (size_t l = 0; l < mg->lev.size(); ++l) {
    MgLevel& L = mg->lev[l];
    double** v[6] = {&L.dinv, &L.b, &L.x[0], &L.x[1], &L.d, &L.r};
    for (int i = 0; i < 6; ++i) {
      const int64_t pd = (i == 2 || i == 3) ? pads[l] : 0;
      p += pd;
      *v[i] = p;
      p += L.m + pd;
    }
    p += 64;
  }
  for (size_t l = 0; l < mg->lev.size(); ++l) {
    MgLevel& L = mg->lev[l];
    const int G = grid_for(ctx, L.m, kBlock, 4);
    IRK_TRY(ensure_red(ctx, (size_t)G + 64));
    k_mg_gershgorin<<<G, kBlock, 0, ctx->stream>>>(L.m, L.A, L.mask, L.dinv, ctx->red);
    IRK_CHECK_LAUNCH(ctx);
    std::vector<double> part(G);
    IRK_CUDA(cudaMemcpyAsync(part.data(), ctx->red, G * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    IRK_CUDA(cudaStreamSynchronize(ctx->stream));
    double mx = 0.0;
    for (double v : part) mx = std::fmax(mx, v);
    if (!(mx > 0.0) || !std::isfinite(mx)) {
      delete mg;
      set_error("irk_mg_create: level %zu: bad diagonal / Gershgorin bound", l);
      return IRK_ESINGULAR;
    }
    L.lmax = mx;
  }
  for (int l = 0; l < nlev; ++l) mg->mats.push_back(A_levels[l]);
  *out = mg;
  return IRK_OK;
}

int irk_mg_destroy(irk_mg* mg) {
  delete mg;
  return IRK_OK;
}

int irk_mg_vcycle(irk_ctx* ctx, irk_mg* mg, const double* r_dev, double* z_dev) {
  IRK_REQUIRE(ctx && mg && r_dev && z_dev, "irk_mg_vcycle: NULL argument");
  IRK_REQUIRE(r_dev != z_dev, "irk_mg_vcycle: r and z must differ");
  return mg->apply(ctx, ctx->stream, r_dev, z_dev, nullptr);
}

int irk_mg_pcg(irk_ctx* ctx, irk_mg* mg, const double* rhs_dev, int64_t ld_rhs, double* x_dev,
               int64_t ld_x, double rtol, double atol, int maxit, int* its_host,
               double* relres_host) {
  IRK_REQUIRE(ctx && mg && rhs_dev && x_dev, "irk_mg_pcg: NULL argument");
  IRK_REQUIRE(ld_rhs >= 1 && ld_x >= 1, "irk_mg_pcg: leading dimensions must be >= 1");
  IRK_REQUIRE(maxit >= 0 && rtol >= 0 && atol >= 0, "irk_mg_pcg: bad tolerances");
  const MgLevel& L0 = mg->lev[0];
  SysParams<double> P{};
  P.alpha[0] = 1.0;
  const int mw = mg->mats[0]->pat->maxw;
  CgPrec* prec = mg;
#define IRK_MGRUN(W)                                                                           \
  return run_cg<double, 1, false, W>(ctx, L0.m, L0.A, P, nullptr, L0.mask, rhs_dev, ld_rhs,   \
                                     x_dev, ld_x, rtol, atol, maxit, its_host, relres_host, prec)
  if (mw <= 8) IRK_MGRUN(8);
  if (mw <= 16) IRK_MGRUN(16);
  IRK_MGRUN(0);
#undef IRK_MGRUN
}

}  // extern "C"
