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
#include "irk_dst3.cuh"

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

// ---------------------------------------------------------------------------
// Structured 3D path (P1 Kuhn-tetrahedra grid levels with the full-boundary
// Dirichlet set, nu = 2): every level operator alpha M_l + beta K_l is ONE
// 3x3x3 stencil (15 nonzero slots) on the interior, extracted from the
// assembled level matrices and verified against every row at setup.  A
// level is three matrix-free tile kernels with shared-memory halos (as the
// 2D path of irk_mg.cu): pre (two Chebyshev steps from zero), residual +
// restriction, prolongation + two post steps.  Tiles cover every grid point
// (boundary points included: x = b there); the coarsest level stays on the
// generic kernels.
struct Sten3 {
  cplx c[27];  // c[(dz+1)*9 + (dy+1)*3 + dx+1]
  cplx dinv;
  unsigned nz;  // bit k: c[k] != 0
};

__device__ __forceinline__ bool interior3(int x, int y, int z, int N) {
  return x >= 1 && x < N && y >= 1 && y < N && z >= 1 && z < N;
}

// The 15 slots of the Kuhn-split P1 stencil: the centre and +-p for the
// seven 0/1 directions p (every one an edge of the triangulation)
constexpr unsigned kuhn_mask() {
  unsigned m = 0;
  for (int k = 0; k < 27; ++k) {
    const int dx = k % 3 - 1, dy = (k / 3) % 3 - 1, dz = k / 9 - 1;
    const bool pos = dx >= 0 && dy >= 0 && dz >= 0, neg = dx <= 0 && dy <= 0 && dz <= 0;
    if (pos || neg) m |= 1u << k;
  }
  return m;
}
constexpr unsigned kKuhnNZ = kuhn_mask();

// sum_k c_k s[i + off_k] over the nonzero slots (region row width W, plane
// WH); KUHN: the slot set is kKuhnNZ, resolved at compile time
template <bool KUHN>
__device__ __forceinline__ cplx sten3_apply(const Sten3& S, const cplx* s, int i, int W, int WH) {
  cplx acc = {0.0, 0.0};
#pragma unroll
  for (int k = 0; k < 27; ++k) {
    if (KUHN ? !((kKuhnNZ >> k) & 1u) : !((S.nz >> k) & 1u)) continue;
    const int dx = k % 3 - 1, dy = (k / 3) % 3 - 1, dz = k / 9 - 1;
    acc = s_add(acc, s_mul(S.c[k], s[i + dz * WH + dy * W + dx]));
  }
  return acc;
}

// region [ox, ox+W) x [oy, oy+H) x [oz, oz+D) of a grid vector into shared
// memory, zero outside the interior
__device__ __forceinline__ void load3(cplx* dst, const cplx* __restrict__ src, int n1, int ox,
                                      int oy, int oz, int W, int H, int D) {
  const int N = n1 - 1;
  for (int k = threadIdx.x; k < W * H * D; k += blockDim.x) {
    const int x = ox + k % W, y = oy + (k / W) % H, z = oz + k / (W * H);
    dst[k] = interior3(x, y, z, N) ? ldv(src + ((int64_t)z * n1 + y) * n1 + x) : cplx{0.0, 0.0};
  }
}

struct Cheb2c {
  double cr0, cd1, cr1;
};

// x2 = two Chebyshev steps from zero (boundary points: x2 = b)
template <int TX, int TY, int TZ, bool KUHN>
__global__ void __launch_bounds__(kBlock)
    k_mg3_pre(int n1, Sten3 S, Cheb2c C, const cplx* __restrict__ b, cplx* __restrict__ x2,
              const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  constexpr int W = TX + 2, H = TY + 2, D = TZ + 2;
  extern __shared__ cplx dyn3[];
  cplx* sb = dyn3;  // W * H * D
  const int N = n1 - 1;
  const int x0 = TX * blockIdx.x, y0 = TY * blockIdx.y, z0 = TZ * blockIdx.z;
  load3(sb, b, n1, x0 - 1, y0 - 1, z0 - 1, W, H, D);
  __syncthreads();
  const cplx s0 = s_mul(s_real<cplx>(C.cr0), S.dinv);
  const cplx k1 = s_mul(s_real<cplx>(1.0 + C.cd1), s0);
  const cplx k2 = s_mul(s_real<cplx>(C.cr1), S.dinv);
  for (int k = threadIdx.x; k < TX * TY * TZ; k += blockDim.x) {
    const int lx = k % TX, ly = (k / TX) % TY, lz = k / (TX * TY);
    const int x = x0 + lx, y = y0 + ly, z = z0 + lz;
    if (x > N || y > N || z > N) continue;
    const int64_t g = ((int64_t)z * n1 + y) * n1 + x;
    if (!interior3(x, y, z, N)) {
      x2[g] = ldv(b + g);
      continue;
    }
    const int i = ((lz + 1) * H + ly + 1) * W + lx + 1;
    const cplx bi = sb[i];
    const cplx ax1 = s_mul(s0, sten3_apply<KUHN>(S, sb, i, W, W * H));
    x2[g] = s_add(s_mul(k1, bi), s_mul(k2, s_sub(bi, ax1)));
  }
}

// b_c = P^T (b - A x2) on the coarse tile (fine boundary: r = 0; coarse
// boundary rows 0); P^T weights 1 at 2c and 1/2 at 2c +- p for the seven
// Kuhn edge directions p in {0,1}^3 \ 0
template <int CX, int CY, int CZ, bool KUHN>
__global__ void __launch_bounds__(kBlock)
    k_mg3_restrict(int n1f, int n1c, Sten3 S, const cplx* __restrict__ bf,
                   const cplx* __restrict__ x2, cplx* __restrict__ bc, const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  constexpr int RW = 2 * CX + 1, RH = 2 * CY + 1, RD = 2 * CZ + 1;
  constexpr int XW = RW + 2, XH = RH + 2, XD = RD + 2;
  extern __shared__ cplx dyn3[];
  cplx* sx = dyn3;                // XW * XH * XD
  cplx* sr = dyn3 + XW * XH * XD;  // RW * RH * RD
  const int Nf = n1f - 1, Nc = n1c - 1;
  const int cx0 = CX * blockIdx.x, cy0 = CY * blockIdx.y, cz0 = CZ * blockIdx.z;
  const int rx0 = 2 * cx0 - 1, ry0 = 2 * cy0 - 1, rz0 = 2 * cz0 - 1;
  load3(sx, x2, n1f, rx0 - 1, ry0 - 1, rz0 - 1, XW, XH, XD);
  __syncthreads();
  for (int k = threadIdx.x; k < RW * RH * RD; k += blockDim.x) {
    const int lx = k % RW, ly = (k / RW) % RH, lz = k / (RW * RH);
    const int x = rx0 + lx, y = ry0 + ly, z = rz0 + lz;
    cplx r = {0.0, 0.0};
    if (interior3(x, y, z, Nf)) {
      const int64_t g = ((int64_t)z * n1f + y) * n1f + x;
      r = s_sub(ldv(bf + g),
                sten3_apply<KUHN>(S, sx, ((lz + 1) * XH + ly + 1) * XW + lx + 1, XW, XW * XH));
    }
    sr[k] = r;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < CX * CY * CZ; k += blockDim.x) {
    const int cx = cx0 + k % CX, cy = cy0 + (k / CX) % CY, cz = cz0 + k / (CX * CY);
    if (cx > Nc || cy > Nc || cz > Nc) continue;
    cplx v = {0.0, 0.0};
    if (interior3(cx, cy, cz, Nc)) {
      const int i = ((2 * cz - rz0) * RH + (2 * cy - ry0)) * RW + (2 * cx - rx0);
      v = sr[i];
      cplx h = {0.0, 0.0};
#pragma unroll
      for (int p = 1; p < 8; ++p) {
        const int o = (p >> 2) * RW * RH + ((p >> 1) & 1) * RW + (p & 1);
        h = s_add(h, s_add(sr[i + o], sr[i - o]));
      }
      v = s_add(v, s_mul(s_real<cplx>(0.5), h));
    }
    bc[((int64_t)cz * n1c + cy) * n1c + cx] = v;
  }
}

// z = two Chebyshev steps from x_p = x2 + P e_c (boundary points z = b):
// x_p on the tile + halo 2, x_a on halo 1
template <int TX, int TY, int TZ, bool KUHN>
__global__ void __launch_bounds__(kBlock)
    k_mg3_post(int n1, int n1c, Sten3 S, Cheb2c C, const cplx* __restrict__ b,
               const cplx* __restrict__ x2, const cplx* __restrict__ ec,
               cplx* __restrict__ z, const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  constexpr int PW = TX + 4, PH = TY + 4, PD = TZ + 4;
  constexpr int AW = TX + 2, AH = TY + 2, AD = TZ + 2;
  extern __shared__ cplx dyn3[];
  cplx* sp = dyn3;                             // PW * PH * PD
  cplx* sa = sp + PW * PH * PD;                // AW * AH * AD
  cplx* sb = sa + AW * AH * AD;                // AW * AH * AD
  const int N = n1 - 1;
  const int x0 = TX * blockIdx.x, y0 = TY * blockIdx.y, z0 = TZ * blockIdx.z;
  const int px = x0 - 2, py = y0 - 2, pz = z0 - 2;
  for (int k = threadIdx.x; k < PW * PH * PD; k += blockDim.x) {
    const int x = px + k % PW, y = py + (k / PW) % PH, zz = pz + k / (PW * PH);
    cplx v = {0.0, 0.0};
    if (interior3(x, y, zz, N)) {
      const int64_t c = ((int64_t)(zz >> 1) * n1c + (y >> 1)) * n1c + (x >> 1);
      const cplx e0 = ldv(ec + c);
      const int odd = (x & 1) | (y & 1) | (zz & 1);
      cplx e = e0;
      if (odd) {
        const int64_t c2 = c + ((int64_t)(zz & 1) * n1c + (y & 1)) * n1c + (x & 1);
        e = s_mul(s_real<cplx>(0.5), s_add(e0, ldv(ec + c2)));
      }
      v = s_add(ldv(x2 + ((int64_t)zz * n1 + y) * n1 + x), e);
    }
    sp[k] = v;
  }
  load3(sb, b, n1, x0 - 1, y0 - 1, z0 - 1, AW, AH, AD);
  __syncthreads();
  const cplx s0 = s_mul(s_real<cplx>(C.cr0), S.dinv);
  for (int k = threadIdx.x; k < AW * AH * AD; k += blockDim.x) {
    const int lx = k % AW, ly = (k / AW) % AH, lz = k / (AW * AH);
    const int x = x0 - 1 + lx, y = y0 - 1 + ly, zz = z0 - 1 + lz;
    cplx v = {0.0, 0.0};
    if (interior3(x, y, zz, N)) {
      const int i = ((lz + 1) * PH + ly + 1) * PW + lx + 1;
      v = s_add(sp[i], s_mul(s0, s_sub(sb[k], sten3_apply<KUHN>(S, sp, i, PW, PW * PH))));
    }
    sa[k] = v;
  }
  __syncthreads();
  const cplx cd1 = s_real<cplx>(C.cd1), k2 = s_mul(s_real<cplx>(C.cr1), S.dinv);
  for (int k = threadIdx.x; k < TX * TY * TZ; k += blockDim.x) {
    const int lx = k % TX, ly = (k / TX) % TY, lz = k / (TX * TY);
    const int x = x0 + lx, y = y0 + ly, zz = z0 + lz;
    if (x > N || y > N || zz > N) continue;
    const int64_t g = ((int64_t)zz * n1 + y) * n1 + x;
    if (!interior3(x, y, zz, N)) {
      z[g] = ldv(b + g);
      continue;
    }
    const int ia = ((lz + 1) * AH + ly + 1) * AW + lx + 1;
    const int ip = ((lz + 2) * PH + ly + 2) * PW + lx + 2;
    const cplx xa = sa[ia];
    z[g] = s_add(s_add(xa, s_mul(cd1, s_sub(xa, sp[ip]))),
                 s_mul(k2, s_sub(sb[ia], sten3_apply<KUHN>(S, sa, ia, AW, AW * AH))));
  }
}

// 3x3x3 stencil of `row` of a real matrix (out[27]); err = 1 for entries
// outside the box
__global__ void k_mg3_row_stencil(MatView A, bool useb, int64_t row, int n1, double* out,
                                  int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int k = 0; k < 27; ++k) out[k] = 0.0;
  const int64_t sl = row / kSlice;
  const int lane = (int)(row % kSlice);
  int base, width;
  if (A.ellw) {
    base = (int)(sl * kSlice * A.ellw);
    width = A.ellw;
  } else {
    base = A.slice_ptr[sl];
    width = (A.slice_ptr[sl + 1] - base) / kSlice;
  }
  const int q0 = base / kSlice;
  for (int k = 0; k < width; ++k) {
    const int pos = base + k * kSlice + lane;
    const int c = sell_col_at(A.colhdr, A.sell_col, q0 + k, pos, row);
    const double v = useb ? sell_val_at(A.ub, A.b, q0 + k, pos) : sell_val_at(A.ua, A.a, q0 + k, pos);
    const int64_t d = (int64_t)c - row;
    int hit = -1;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx)
          if (d == dx + (int64_t)n1 * (dy + (int64_t)n1 * dz)) hit = (dz + 1) * 9 + (dy + 1) * 3 + dx + 1;
    if (hit >= 0)
      out[hit] += v;
    else if (v != 0.0)
      err[0] = 1;
  }
}

// max over rows of |(A v) - (S v)| and |A v| for v_i = sin(0.37 i + 0.11)
// (A = M or K by useb; S the real stencil cs; masked rows identity)
__global__ void __launch_bounds__(kBlock)
    k_mg3_verify(MatView A, bool useb, int n1, const double* __restrict__ cs,
                 const uint8_t* __restrict__ mask, double* part) {
  const int N = n1 - 1;
  const int64_t m = (int64_t)n1 * n1 * n1;
  double emax = 0.0, amax = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % n1), y = (int)((i / n1) % n1), z = (int)(i / ((int64_t)n1 * n1));
    const bool in = interior3(x, y, z, N);
    if (in == (mask[i] != 0)) {
      emax = INFINITY;
      continue;
    }
    if (!in) continue;  // masked rows: identity in the kernels, zero in M, K
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
    double av = 0.0;
    for (int k = 0; k < width; ++k) {
      const int pos = base + k * kSlice + lane;
      const int c = sell_col_at(A.colhdr, A.sell_col, q0 + k, pos, i);
      const double a = useb ? sell_val_at(A.ub, A.b, q0 + k, pos) : sell_val_at(A.ua, A.a, q0 + k, pos);
      av += a * sin(0.37 * c + 0.11);
    }
    double sv = 0.0;
    for (int k = 0; k < 27; ++k) {
      const int dx = k % 3 - 1, dy = (k / 3) % 3 - 1, dz = k / 9 - 1;
      if (interior3(x + dx, y + dy, z + dz, N))
        sv += cs[k] * sin(0.37 * (((int64_t)(z + dz) * n1 + y + dy) * n1 + x + dx) + 0.11);
    }
    emax = fmax(emax, fabs(av - sv));
    amax = fmax(amax, fabs(av));
  }
  __shared__ double re[kBlock / 32], ra[kBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  }
  if (lane == 0) {
    re[warp] = emax;
    ra[warp] = amax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double e = 0.0, a = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) {
      e = fmax(e, re[w]);
      a = fmax(a, ra[w]);
    }
    part[2 * blockIdx.x] = e;
    part[2 * blockIdx.x + 1] = a;
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
  int dim = 0;
  irk::cplx al{}, be{};
  std::vector<irk::McLevel> lev;
  void* mem = nullptr;
  // structured 3D path (k_mg3_*): levels 0..nlev-2 as stencil tile kernels
  bool s3_on = false, s3_ok = false;
  std::vector<irk::Sten3> s3;
  std::vector<irk::Cheb2c> c3;
  // fast sine-transform preconditioner of the level-0 block (irk_dst3.cu):
  // available / in use instead of the V-cycle
  bool dst_ok = false, dst_on = false;
  irk::Dst3Plan dstP{};
  void* dst_mem = nullptr;

  // Set up the sine-transform preconditioner on the verified level-0 stencil
  // (structured path available): the stencil averaged over the reflections
  // of every offset, its eigenvalues bounded away from zero on all modes.
  int setup_dst3(irk_ctx* ctx) {
    using namespace irk;
    dst_ok = false;
    if (!s3_ok || dim != 3) return IRK_OK;
    const int N = (int)lev[0].g.n1 - 1;
    if (!dst3_supported(N)) return IRK_OK;
    Dst3Coef C{};
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const cplx c = s3[0].c[(dz + 1) * 9 + (dy + 1) * 3 + dx + 1];
          const int a = dx != 0, b = dy != 0, e = dz != 0;
          const double w = 1.0 / (double)(1 << (a + b + e));
          C.s[a + 2 * b + 4 * e].x += w * c.re;
          C.s[a + 2 * b + 4 * e].y += w * c.im;
        }
    C.sc = 8.0 / ((double)N * (double)N * (double)N);
    std::vector<double> ck(N + 1);
    for (int k = 0; k <= N; ++k) ck[k] = std::cos(M_PI * (double)k / N);
    double lo = INFINITY, hi = 0.0;
    for (int kz = 1; kz < N; ++kz)
      for (int ky = 1; ky < N; ++ky) {
        const double tz = 2 * ck[kz], ty = 2 * ck[ky];
        double pr[2], qr[2];
        for (int c = 0; c < 2; ++c) {
          auto S = [&](int i) { return c == 0 ? C.s[i].x : C.s[i].y; };
          pr[c] = S(0) + S(2) * ty + S(4) * tz + S(6) * ty * tz;
          qr[c] = S(1) + S(3) * ty + S(5) * tz + S(7) * ty * tz;
        }
        for (int kx = 1; kx < N; ++kx) {
          const double tx = 2 * ck[kx];
          const double re = pr[0] + qr[0] * tx, im = pr[1] + qr[1] * tx;
          const double a2 = re * re + im * im;
          lo = std::fmin(lo, a2);
          hi = std::fmax(hi, a2);
        }
      }
    if (!(lo > 1e-24 * hi) || !std::isfinite(hi)) return IRK_OK;
    const int L = 2 * N;
    const size_t n1 = (size_t)N + 1;
    const size_t bytes = (n1 * n1 * n1 + (size_t)L) * sizeof(double2) + (n1 + 8) * sizeof(double);
    if (!dst_mem) IRK_CUDA(cudaMalloc(&dst_mem, bytes));
    double2* T = reinterpret_cast<double2*>(dst_mem);
    double2* tw = T + n1 * n1 * n1;
    double* cosk = reinterpret_cast<double*>(tw + L);
    std::vector<double> host(2 * (size_t)L + n1);
    for (int q = 0; q < L; ++q) {
      const double a = -2.0 * M_PI * (double)q / (double)L;
      host[2 * q] = std::cos(a);
      host[2 * q + 1] = std::sin(a);
    }
    for (int k = 0; k <= N; ++k) host[2 * (size_t)L + k] = ck[k];
    IRK_CUDA(cudaMemcpyAsync(tw, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    IRK_CUDA(cudaStreamSynchronize(ctx->stream));
    IRK_TRY(dst3_prepare(N));
    dstP.N = N;
    dstP.C = C;
    dstP.T = T;
    dstP.tw = tw;
    dstP.cosk = cosk;
    dst_ok = true;
    return IRK_OK;
  }

  int setup_s3(irk_ctx* ctx) {
    using namespace irk;
    static const bool off = getenv("IRK_MG_GENERIC") != nullptr;
    s3_on = false;
    const int nl = (int)lev.size();
    if (off || dim != 3 || nu != 2 || nl < 2) return IRK_OK;
    for (const McLevel& L : lev)
      if (!L.mask || L.g.n1 - 1 < 4 || L.g.n1 > 1290) return IRK_OK;
    const int G = ctx->num_sms * 4;
    IRK_TRY(ensure_red(ctx, 2 * (size_t)G + 64));
    s3.assign(nl, Sten3{});
    c3.assign(nl, Cheb2c{});
    double* dst = nullptr;
    IRK_CUDA(cudaMalloc(&dst, 2 * 27 * sizeof(double)));
    int* err = (int*)ctx->counters + (kNumCounters - 2);
    int rc = IRK_OK;
    for (int l = 0; l + 1 < nl && rc == IRK_OK; ++l) {
      const McLevel& L = lev[l];
      const int n1 = (int)L.g.n1, N = n1 - 1;
      const int64_t row = ((int64_t)(N / 2) * n1 + N / 2) * n1 + N / 2;
      double cs[2][27];
      bool ok = true;
      for (int which = 0; which < 2 && ok; ++which) {
        cudaMemsetAsync(err, 0, sizeof(int), ctx->stream);
        k_mg3_row_stencil<<<1, 32, 0, ctx->stream>>>(L.A, which == 1, row, n1, dst + 27 * which,
                                                      err);
        int herr = 0;
        cudaMemcpyAsync(cs[which], dst + 27 * which, 27 * sizeof(double), cudaMemcpyDeviceToHost,
                        ctx->stream);
        cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess || herr) {
          ok = false;
          break;
        }
        k_mg3_verify<<<G, kBlock, 0, ctx->stream>>>(L.A, which == 1, n1, dst + 27 * which,
                                                     L.mask, ctx->red);
        std::vector<double> part(2 * G);
        cudaMemcpyAsync(part.data(), ctx->red, part.size() * sizeof(double),
                        cudaMemcpyDeviceToHost, ctx->stream);
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
          ok = false;
          break;
        }
        double e = 0.0, a = 0.0;
        for (int b = 0; b < G; ++b) {
          e = std::fmax(e, part[2 * b]);
          a = std::fmax(a, part[2 * b + 1]);
        }
        if (!(e <= 1e-12 * a)) ok = false;
      }
      if (!ok) {
        rc = -1;
        break;
      }
      Sten3& S = s3[l];
      S.nz = 0;
      for (int k = 0; k < 27; ++k) {
        S.c[k] = {al.re * cs[0][k] + be.re * cs[1][k], al.im * cs[0][k] + be.im * cs[1][k]};
        if (S.c[k].re != 0.0 || S.c[k].im != 0.0) S.nz |= 1u << k;
      }
      if (S.c[13].re == 0.0 && S.c[13].im == 0.0) {
        rc = -1;
        break;
      }
      const double dd = S.c[13].re * S.c[13].re + S.c[13].im * S.c[13].im;
      S.dinv = {S.c[13].re / dd, -S.c[13].im / dd};
      std::vector<double> cd, cr;
      cheb(0.25 * L.lmax, L.lmax, 2, cd, cr);
      c3[l] = Cheb2c{cr[0], cd[1], cr[1]};
    }
    cudaFree(dst);
    cudaGetLastError();
    s3_ok = s3_on = rc == IRK_OK && set_smem_attrs() == IRK_OK;
    cudaGetLastError();
    return IRK_OK;
  }

  // 3D tiles: pre/post TX x TY x TZ fine points, restriction CX x CY x CZ
  // coarse points (dynamic shared memory; sizes below)
  static constexpr int TX3 = 16, TY3 = 4, TZ3 = 4, CX3 = 8, CY3 = 4, CZ3 = 4;  // 16x8x8, 16x8x4: no better
  static constexpr size_t kPreSmem = (size_t)(TX3 + 2) * (TY3 + 2) * (TZ3 + 2) * 16;
  static constexpr size_t kResSmem =
      ((size_t)(2 * CX3 + 3) * (2 * CY3 + 3) * (2 * CZ3 + 3) +
       (size_t)(2 * CX3 + 1) * (2 * CY3 + 1) * (2 * CZ3 + 1)) * 16;
  static constexpr size_t kPostSmem =
      ((size_t)(TX3 + 4) * (TY3 + 4) * (TZ3 + 4) + 2 * (size_t)(TX3 + 2) * (TY3 + 2) * (TZ3 + 2)) *
      16;

  static int set_smem_attrs() {
    using namespace irk;
    for (const void* fn : {(const void*)k_mg3_pre<TX3, TY3, TZ3, true>,
                           (const void*)k_mg3_pre<TX3, TY3, TZ3, false>})
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPreSmem))
        return IRK_ECUDA;
    for (const void* fn : {(const void*)k_mg3_restrict<CX3, CY3, CZ3, true>,
                           (const void*)k_mg3_restrict<CX3, CY3, CZ3, false>})
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kResSmem))
        return IRK_ECUDA;
    for (const void* fn : {(const void*)k_mg3_post<TX3, TY3, TZ3, true>,
                           (const void*)k_mg3_post<TX3, TY3, TZ3, false>})
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPostSmem))
        return IRK_ECUDA;
    return IRK_OK;
  }

  // structured 3D V-cycle on level l (l < nlev-1); the result lands in out
  int vcycle3(irk_ctx* ctx, cudaStream_t s, int l, const irk::cplx* b, irk::cplx* out,
              const int* stop) {
    using namespace irk;
    McLevel& L = lev[l];
    McLevel& Cc = lev[l + 1];
    const int n1 = (int)L.g.n1, n1c = (int)Cc.g.n1;
    const dim3 gt((n1 + TX3 - 1) / TX3, (n1 + TY3 - 1) / TY3, (n1 + TZ3 - 1) / TZ3);
    const dim3 gr((n1c + CX3 - 1) / CX3, (n1c + CY3 - 1) / CY3, (n1c + CZ3 - 1) / CZ3);
    const bool kuhn = s3[l].nz == kKuhnNZ;
    if (kuhn) {
      launch(k_mg3_pre<TX3, TY3, TZ3, true>, gt, kBlock, kPreSmem, s, n1, s3[l], c3[l], b,
             L.x[0], stop);
      launch(k_mg3_restrict<CX3, CY3, CZ3, true>, gr, kBlock, kResSmem, s, n1, n1c, s3[l], b,
             (const cplx*)L.x[0], Cc.b, stop);
    } else {
      launch(k_mg3_pre<TX3, TY3, TZ3, false>, gt, kBlock, kPreSmem, s, n1, s3[l], c3[l], b,
             L.x[0], stop);
      launch(k_mg3_restrict<CX3, CY3, CZ3, false>, gr, kBlock, kResSmem, s, n1, n1c, s3[l], b,
             (const cplx*)L.x[0], Cc.b, stop);
    }
    ctx->launches += 2;
    if (cudaPeekAtLastError() != cudaSuccess) return IRK_ECUDA;
    cplx* ec;
    if (l + 2 == (int)lev.size()) {
      int res;
      IRK_TRY(smooth(ctx, s, l + 1, Cc.b, -1, ncoarse, 0.05, Cc.r, stop, &res));
      ec = Cc.r;
    } else {
      IRK_TRY(vcycle3(ctx, s, l + 1, Cc.b, Cc.x[1], stop));
      ec = Cc.x[1];
    }
    if (kuhn)
      launch(k_mg3_post<TX3, TY3, TZ3, true>, gt, kBlock, kPostSmem, s, n1, n1c, s3[l], c3[l],
             b, (const cplx*)L.x[0], (const cplx*)ec, out, stop);
    else
      launch(k_mg3_post<TX3, TY3, TZ3, false>, gt, kBlock, kPostSmem, s, n1, n1c, s3[l], c3[l],
             b, (const cplx*)L.x[0], (const cplx*)ec, out, stop);
    ctx->launches++;
    return cudaPeekAtLastError() == cudaSuccess ? IRK_OK : IRK_ECUDA;
  }

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

  // sine-transform-preconditioned COCG: ~2.7 iterations to 1e-6
  int prefix_iters() override { return dst_on ? 2 : -1; }

  int apply(irk_ctx* ctx, cudaStream_t s, const double* r, double* z, const int* stop) override {
    if (dst_on) {
      const int e = irk::dst3_apply(ctx, s, dstP, reinterpret_cast<const double2*>(r),
                                    reinterpret_cast<double2*>(z), stop);
      if (e != IRK_OK || cudaGetLastError() != cudaSuccess) {
        irk::set_error("irk_mgc: sine-transform preconditioner launch failed");
        return IRK_ECUDA;
      }
      return IRK_OK;
    }
    if (s3_on) {
      const int e = vcycle3(ctx, s, 0, reinterpret_cast<const irk::cplx*>(r),
                            reinterpret_cast<irk::cplx*>(z), stop);
      if (e != IRK_OK || cudaGetLastError() != cudaSuccess) {
        irk::set_error("irk_mgc: structured V-cycle launch failed");
        return IRK_ECUDA;
      }
      return IRK_OK;
    }
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
    if (dst_mem) cudaFree(dst_mem);
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
  mg->dim = dim;
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
  IRK_TRY(mg->setup_s3(ctx));
  {
    const int ed = mg->setup_dst3(ctx);
    if (ed != IRK_OK) {
      delete mg;
      return ed;
    }
  }
  *out = mg;
  return IRK_OK;
}

int irk_mgc_set_dst(irk_mgc* mg, int on) {
  IRK_REQUIRE(mg, "irk_mgc_set_dst: NULL argument");
  IRK_REQUIRE(!on || mg->dst_ok,
              "irk_mgc_set_dst: no sine-transform preconditioner for this block (needs a verified "
              "3D grid stencil with the full-boundary Dirichlet set and 2N = 2^a or 3 * 2^a in "
              "[24, 384])");
  if ((on != 0) != mg->dst_on) {
    mg->dst_on = on != 0;
    mg->uid = g_mgc_uid.fetch_add(1);  // cached graphs hold the other kernel sequence
  }
  return IRK_OK;
}

int irk_mgc_dst_info(const irk_mgc* mg, int* available, int* on) {
  IRK_REQUIRE(mg, "irk_mgc_dst_info: NULL argument");
  if (available) *available = mg->dst_ok ? 1 : 0;
  if (on) *on = mg->dst_on ? 1 : 0;
  return IRK_OK;
}

int irk_mgc_set_structured(irk_mgc* mg, int on) {
  IRK_REQUIRE(mg, "irk_mgc_set_structured: NULL argument");
  IRK_REQUIRE(!on || mg->s3_ok,
              "irk_mgc_set_structured: no structured path for this hierarchy (needs 3D levels "
              "with the full-boundary Dirichlet set and nu = 2)");
  if ((on != 0) != mg->s3_on) {
    mg->s3_on = on != 0;
    mg->uid = g_mgc_uid.fetch_add(1);  // cached graphs hold the other kernel sequence
  }
  return IRK_OK;
}

int irk_mgc_info(const irk_mgc* mg, int* nlev, int* structured) {
  IRK_REQUIRE(mg, "irk_mgc_info: NULL argument");
  if (nlev) *nlev = (int)mg->lev.size();
  if (structured) *structured = mg->s3_on ? 1 : 0;
  return IRK_OK;
}

int irk_mgc_vcycle(irk_ctx* ctx, irk_mgc* mg, const double* r_dev, double* z_dev) {
  IRK_REQUIRE(ctx && mg && r_dev && z_dev, "irk_mgc_vcycle: NULL argument");
  IRK_REQUIRE(r_dev != z_dev, "irk_mgc_vcycle: r and z must differ");
  IRK_REQUIRE(((uintptr_t)r_dev % 16) == 0 && ((uintptr_t)z_dev % 16) == 0,
              "irk_mgc_vcycle: r/z must be 16-byte aligned");
  return mg->apply(ctx, ctx->stream, r_dev, z_dev, nullptr);
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

int irk_mgc_cocg_multi(irk_ctx* ctx, int n, irk_mgc* const* mgs, const double* rhs_dev,
                       int64_t ld_rhs, int64_t rhs_step, double* x_dev, int64_t ld_x,
                       int64_t x_step, double rtol, double atol, int maxit, int* its_host,
                       double* relres_host) {
  IRK_REQUIRE(ctx && mgs && n >= 0, "irk_mgc_cocg_multi: NULL argument");
  IRK_REQUIRE(rhs_step % 2 == 0 && x_step % 2 == 0, "irk_mgc_cocg_multi: odd system step");
  const bool deferred = !its_host && !relres_host && ctx->log_on;
  return run_forked(ctx, n, deferred, [&](int k, irk_ctx* c) {
    return irk_mgc_cocg(c, mgs[k], rhs_dev + k * rhs_step, ld_rhs, x_dev + k * x_step, ld_x, rtol,
                        atol, maxit, its_host ? its_host + k : nullptr,
                        relres_host ? relres_host + k : nullptr);
  });
}

}  // extern "C"
