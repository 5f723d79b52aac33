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
#include <string>
#include <vector>

#include "irk_inner.cuh"
#define IRK_DST_2D
#include "irk_dst.cuh"

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
  IRK_PDL_ENTER();
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
  IRK_PDL_ENTER();
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
  IRK_PDL_ENTER();
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
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    r[i] = (mask && mask[i]) ? 0.0 : b[i] - row_dot(A, i, x);
}

// bc = P^T rf, zero at constrained coarse nodes
__global__ void __launch_bounds__(kBlock)
    k_mg_restrict(int64_t mc, GridIdx gc, GridIdx gf, const uint8_t* __restrict__ maskc,
                  const double* __restrict__ rf, double* __restrict__ bc, const int* stop) {
  IRK_PDL_ENTER();
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
  IRK_PDL_ENTER();
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

// ---------------------------------------------------------------------------
// Structured 2D path (P1/Q1 grid blocks with the full-boundary Dirichlet
// set, nu = 2): every level operator is ONE 3x3 stencil on the interior
// (boundary rows identity, boundary columns eliminated), read from the
// assembled level matrix and verified against it at setup.  A V-cycle level
// is then three matrix-free tile kernels with shared-memory halos instead of
// seven gather kernels:
//   k_mg2_pre      x2 = two Chebyshev steps from zero      (reads b,     writes x2)
//   k_mg2_restrict b_c = P^T (b - A x2)                     (reads b, x2, writes b_c)
//   k_mg2_post     z = two Chebyshev steps from x2 + P e_c  (reads b, x2, e_c, writes z)
// (16-24 B per fine point each instead of ~244 B over the seven kernels),
// and the coarsest level is one single-CTA kernel holding the grid in
// shared memory.  Same arithmetic as the generic path up to summation order.
// tile of the structured pre/post kernels on levels with N >= 512 (64 x 16
// measured best on B200 against 64 x 8, 32 x 16 and 128 x 8)
constexpr int kBTX = 64, kBTY = 16;

struct Sten2 {
  double c[3][3];  // c[dy + 1][dx + 1]: coefficient of the neighbour (x+dx, y+dy)
  double dinv;     // 1 / c[1][1]
};

// Chebyshev smoother of nu <= kMaxNu steps: d_k = cd_k d_{k-1} + cr_k D^-1 r_k
// (cd_0 = 0), i.e. x_{k+1} = x_k + cd_k (x_k - x_{k-1}) + cr_k D^-1 (b - A x_k)
constexpr int kMaxNu = 4;
struct ChebS {
  double cd[kMaxNu], cr[kMaxNu];
};

constexpr int kMaxCoarse = 64;
struct ChebN {
  int n;
  double cd[kMaxCoarse], cr[kMaxCoarse];
};

// sum_{dx,dy} c[dy][dx] s[i + dy*W + dx] (zero coefficients skipped at
// compile time for the P1 diagonal-edge layout: (1,-1) and (-1,1) are 0)
template <bool F9>
__device__ __forceinline__ double sten_apply(const Sten2& S, const double* s, int i, int W) {
  double acc = S.c[1][1] * s[i];
  acc += S.c[1][0] * s[i - 1] + S.c[1][2] * s[i + 1];
  acc += S.c[0][1] * s[i - W] + S.c[2][1] * s[i + W];
  acc += S.c[0][0] * s[i - W - 1] + S.c[2][2] * s[i + W + 1];
  if (F9) acc += S.c[0][2] * s[i - W + 1] + S.c[2][0] * s[i + W - 1];
  return acc;
}

__device__ __forceinline__ bool interior2(int gx, int gy, int N) {
  return gx >= 1 && gx < N && gy >= 1 && gy < N;
}

// region [gx0, gx0 + W) x [gy0, gy0 + H) of a grid vector, zero outside the
// interior (eliminated boundary columns / outside the grid): element
// k = threadIdx.x + j * kBlock into v[j].  All loads are issued before any
// use (memory-level parallelism: one round trip per region, not per element).
template <int W, int H>
struct Region {
  static constexpr int kN = W * H;
  static constexpr int kPer = (kN + kBlock - 1) / kBlock;
  __device__ __forceinline__ static void load(double (&v)[kPer], const double* __restrict__ src,
                                              int n1, int gx0, int gy0) {
    const int N = n1 - 1;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int k = threadIdx.x + j * kBlock;
      const int gx = gx0 + k % W, gy = gy0 + k / W;
      v[j] = (k < kN && interior2(gx, gy, N)) ? src[(int64_t)gy * n1 + gx] : 0.0;
    }
  }
  __device__ __forceinline__ static void store(double* dst, const double (&v)[kPer]) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int k = threadIdx.x + j * kBlock;
      if (k < kN) dst[k] = v[j];
    }
  }
};

// Tiles cover the interior-anchored ranges [1 + T t, 1 + T (t+1)) in each
// direction (clipped to [0, N]); the boundary lines x = 0 / y = 0 are written
// by the first tile row/column.  f(gx, gy, lx, ly) for each owned grid point
// (lx, ly: position in the tile, -1 on the boundary lines x = 0 / y = 0).
template <int TX, int TY, typename F>
__device__ __forceinline__ void for_tile_points(int N, F&& f) {
  static_assert((TX * TY) % kBlock == 0, "tile must be a multiple of the block");
  const int x0 = 1 + TX * blockIdx.x, y0 = 1 + TY * blockIdx.y;
#pragma unroll
  for (int j = 0; j < TX * TY / kBlock; ++j) {
    const int k = threadIdx.x + j * kBlock;
    const int lx = k % TX, ly = k / TX;
    const int gx = x0 + lx, gy = y0 + ly;
    if (gx <= N && gy <= N) f(gx, gy, lx, ly);
  }
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < TY; j += kBlock)
      if (y0 + j <= N) f(0, y0 + j, -1, j);
  if (blockIdx.y == 0)
    for (int i = threadIdx.x; i < TX; i += kBlock)
      if (x0 + i <= N) f(x0 + i, 0, i, -1);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) f(0, 0, -1, -1);
}

// The boundary lines x = 0 / y = 0 next to the first tile column / row
// (outside the interior-anchored tiles): f(gx, gy).
template <int TX, int TY, typename F>
__device__ __forceinline__ void boundary_lines(int N, F&& f) {
  const int x0 = 1 + TX * blockIdx.x, y0 = 1 + TY * blockIdx.y;
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < TY; j += kBlock)
      if (y0 + j <= N) f(0, y0 + j);
  if (blockIdx.y == 0)
    for (int i = threadIdx.x; i < TX; i += kBlock)
      if (x0 + i <= N) f(x0 + i, 0);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) f(0, 0);
}

// One Chebyshev step on halo h of a tile (shared buffers of halo HX, row
// width WL), register-blocked: thread t owns column t % w (w = TX + 2h) over
// a segment of rows and slides a 3x3 window of x_k down it, so each point
// costs 3 shared loads of x_k (the new row) + b + x_{k-1} instead of 9.
// sink(local index, gx, gy, value) receives x_{k+1} at every point of the
// region (zero-extended outside the interior is the caller's job).
template <int TX, int TY, int HX, bool F9, typename Sink>
__device__ __forceinline__ void cheb_rows(int h, const Sten2& S, const double* __restrict__ xk,
                                          const double* __restrict__ xm, bool first,
                                          const double* __restrict__ sb, double cd, double cr,
                                          int ox, int oy, int N, Sink&& sink) {
  constexpr int WL = TX + 2 * HX;
  const int w = TX + 2 * h, hgt = TY + 2 * h;
  const int nseg = kBlock / w;
  const int rs = (hgt + nseg - 1) / nseg;
  const int c = threadIdx.x % w, sg = threadIdx.x / w;
  if (sg >= nseg) return;
  const int i = HX - h + c;
  const int j0 = HX - h + sg * rs, j1 = min(HX - h + hgt, j0 + rs);
  if (j0 >= j1) return;
  const double* col = xk + i;
  // window rows j-1 (s), j (c), j+1 (n) of columns i-1 (w), i, i+1 (e)
  double ws = col[(j0 - 1) * WL - 1], cs = col[(j0 - 1) * WL], es = col[(j0 - 1) * WL + 1];
  double wc = col[j0 * WL - 1], cc = col[j0 * WL], ec = col[j0 * WL + 1];
  const int gx = ox + i;
  for (int j = j0; j < j1; ++j) {
    const double* r = col + (j + 1) * WL;
    const double wn = r[-1], cn = r[0], en = r[1];
    const int gy = oy + j;
    const int li = j * WL + i;
    double v = 0.0;
    if (interior2(gx, gy, N)) {
      double ax = S.c[1][1] * cc;
      ax += S.c[1][0] * wc + S.c[1][2] * ec;
      ax += S.c[0][1] * cs + S.c[2][1] * cn;
      ax += S.c[0][0] * ws + S.c[2][2] * en;
      if (F9) ax += S.c[0][2] * es + S.c[2][0] * wn;
      const double xmv = first ? 0.0 : xm[li];
      v = cc + cd * (cc - xmv) + cr * (sb[li] - ax);
    }
    sink(li, gx, gy, v);
    ws = wc, cs = cc, es = ec;
    wc = wn, cc = cn, ec = en;
  }
}

// x = NU Chebyshev steps from zero on b (boundary rows: x = b), temporally
// blocked: b and x_1 = cr_0 D^-1 b on the tile + halo NU-1, step k on halo
// NU-1-k; the iterates ping-pong between two shared buffers (x_{k+1}
// overwrites x_{k-1} point by point), only x_NU goes to global memory.
template <int TX, int TY, int NU, bool F9>
__global__ void __launch_bounds__(kBlock)
    k_mg2_pre(int n1, Sten2 S, ChebS C, const double* __restrict__ b, double* __restrict__ x2,
              const int* stop, SkipCtl sk) {
  IRK_PDL_ENTER();
  if (sk.st) {
    // fused CG: the skip decision of k_cg_skip, taken by every CTA from the
    // update kernel's partials (same order) and published for the rest of
    // the V-cycle
    __shared__ double srr[1];
    reduce_partials<double, 1>(sk.rr, sk.G, srr);
    const bool skip = cg_skip_pred<double>(sk.st, srr[0], sk.maxit);
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) sk.st->skip = skip ? 1 : 0;
    if (skip) return;
  } else if (stop && *stop) {
    return;
  }
  constexpr int HX = NU - 1, WL = TX + 2 * HX, HL = TY + 2 * HX;
  using R = Region<WL, HL>;
  __shared__ double sb[WL * HL], sx[2][WL * HL];
  const int N = n1 - 1;
  const int ox = 1 + TX * blockIdx.x - HX, oy = 1 + TY * blockIdx.y - HX;
  {
    double v[R::kPer];
    R::load(v, b, n1, ox, oy);
    const double c0 = C.cr[0] * S.dinv;
#pragma unroll
    for (int j = 0; j < R::kPer; ++j) {
      const int k = threadIdx.x + j * kBlock;
      if (k < R::kN) {
        sb[k] = v[j];
        sx[0][k] = c0 * v[j];  // x_1 (zero outside the interior)
      }
    }
  }
  __syncthreads();
  int cur = 0;  // sx[cur] = x_k
#pragma unroll
  for (int k = 1; k < NU - 1; ++k) {
    const double* xk = sx[cur];
    double* xo = sx[cur ^ 1];  // x_{k-1} in, x_{k+1} out
    cheb_rows<TX, TY, HX, F9>(NU - 1 - k, S, xk, xo, k == 1, sb, C.cd[k], C.cr[k] * S.dinv, ox,
                              oy, N, [&](int li, int, int, double v) { xo[li] = v; });
    __syncthreads();
    cur ^= 1;
  }
  cheb_rows<TX, TY, HX, F9>(0, S, sx[cur], sx[cur ^ 1], NU == 2, sb, C.cd[NU - 1],
                            C.cr[NU - 1] * S.dinv, ox, oy, N,
                            [&](int, int gx, int gy, double v) {
                              if (gx > N || gy > N) return;
                              const int64_t g = (int64_t)gy * n1 + gx;
                              x2[g] = interior2(gx, gy, N) ? v : b[g];
                            });
  boundary_lines<TX, TY>(N, [&](int gx, int gy) {
    const int64_t g = (int64_t)gy * n1 + gx;
    x2[g] = b[g];
  });
}

// b_c = P^T r on the coarse tile, r = b - A x2 on the fine interior (0 on the
// boundary); coarse boundary rows 0.  Fine point f = 2c + p: P^T weights 1
// (p = 0) and 1/2 for the six P1 edge neighbours 2c +- (1,0), (0,1), (1,1).
template <int CX, int CY, bool F9>
__global__ void __launch_bounds__(kBlock)
    k_mg2_restrict(int n1f, int n1c, Sten2 S, const double* __restrict__ bf,
                   const double* __restrict__ x2, double* __restrict__ bc, const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  constexpr int RW = 2 * CX + 1, RH = 2 * CY + 1;  // residual region
  constexpr int XW = RW + 2, XH = RH + 2;          // x2 region (halo 1)
  using RX = Region<XW, XH>;
  using RB = Region<RW, RH>;
  __shared__ double sx[XW * XH];
  __shared__ double sr[RW * RH];
  const int Nc = n1c - 1;
  const int cx0 = 1 + CX * blockIdx.x, cy0 = 1 + CY * blockIdx.y;
  const int rx0 = 2 * cx0 - 1, ry0 = 2 * cy0 - 1;
  double vb[RB::kPer];
  {
    double vx[RX::kPer];
    RX::load(vx, x2, n1f, rx0 - 1, ry0 - 1);
    RB::load(vb, bf, n1f, rx0, ry0);  // zero on the boundary: r = 0 there
    RX::store(sx, vx);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < RB::kPer; ++j) {
    const int k = threadIdx.x + j * kBlock;
    if (k < RB::kN) {
      const int lx = k % RW, ly = k / RW;
      const bool in = interior2(rx0 + lx, ry0 + ly, n1f - 1);
      sr[k] = in ? vb[j] - sten_apply<F9>(S, sx, (ly + 1) * XW + lx + 1, XW) : 0.0;
    }
  }
  __syncthreads();
  for_tile_points<CX, CY>(Nc, [&](int gx, int gy, int, int) {
    double v = 0.0;
    if (interior2(gx, gy, Nc)) {
      const int i = (2 * gy - ry0) * RW + (2 * gx - rx0);
      v = sr[i] + 0.5 * (sr[i - 1] + sr[i + 1] + sr[i - RW] + sr[i + RW] + sr[i - RW - 1] +
                         sr[i + RW + 1]);
    }
    bc[(int64_t)gy * n1c + gx] = v;
  });
}

// z = NU Chebyshev steps from x_p = x2 + P e_c (boundary rows z = b),
// temporally blocked like k_mg2_pre: x_p and b on the tile + halo NU, step k
// on halo NU-1-k, only z goes to global memory.
template <int TX, int TY, int NU, bool F9>
__global__ void __launch_bounds__(kBlock, 4)
    k_mg2_post(int n1, int n1c, Sten2 S, ChebS C, const double* __restrict__ b,
               const double* __restrict__ x2, const double* __restrict__ ec,
               double* __restrict__ z, const int* stop, double* __restrict__ rz_part) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  constexpr int HX = NU, WL = TX + 2 * HX, HL = TY + 2 * HX;
  using R = Region<WL, HL>;
  __shared__ double sb[WL * HL], sx[2][WL * HL];
  const int N = n1 - 1;
  const int ox = 1 + TX * blockIdx.x - HX, oy = 1 + TY * blockIdx.y - HX;
  {
    double vb[R::kPer];
    R::load(vb, b, n1, ox, oy);
    R::store(sb, vb);
  }
  {
    double vx[R::kPer], e0[R::kPer], e1[R::kPer];
#pragma unroll
    for (int j = 0; j < R::kPer; ++j) {
      const int k = threadIdx.x + j * kBlock;
      const int gx = ox + k % WL, gy = oy + k / WL;
      vx[j] = e0[j] = e1[j] = 0.0;
      if (k < R::kN && interior2(gx, gy, N)) {
        const int64_t c = (int64_t)(gy >> 1) * n1c + (gx >> 1);
        vx[j] = x2[(int64_t)gy * n1 + gx];
        e0[j] = ec[c];
        e1[j] = ec[c + (int64_t)(gy & 1) * n1c + (gx & 1)];
      }
    }
#pragma unroll
    for (int j = 0; j < R::kPer; ++j) {
      const int k = threadIdx.x + j * kBlock;
      const int gx = ox + k % WL, gy = oy + k / WL;
      const bool odd = ((gx | gy) & 1) != 0;
      if (k < R::kN) sx[0][k] = vx[j] + (odd ? 0.5 * (e0[j] + e1[j]) : e0[j]);
    }
  }
  __syncthreads();
  int cur = 0;  // sx[cur] = x_k
#pragma unroll
  for (int k = 0; k < NU - 1; ++k) {
    const double* xk = sx[cur];
    double* xo = sx[cur ^ 1];
    cheb_rows<TX, TY, HX, F9>(NU - 1 - k, S, xk, xo, k == 0, sb, C.cd[k], C.cr[k] * S.dinv, ox,
                              oy, N, [&](int li, int, int, double v) { xo[li] = v; });
    __syncthreads();
    cur ^= 1;
  }
  double rz = 0.0;  // r.z of the written points (fused CG: rz_part)
  cheb_rows<TX, TY, HX, F9>(0, S, sx[cur], sx[cur ^ 1], false, sb, C.cd[NU - 1],
                            C.cr[NU - 1] * S.dinv, ox, oy, N,
                            [&](int li, int gx, int gy, double v) {
                              if (gx > N || gy > N) return;
                              const int64_t g = (int64_t)gy * n1 + gx;
                              const bool in = interior2(gx, gy, N);
                              const double bi = in ? sb[li] : b[g];
                              const double zi = in ? v : bi;
                              z[g] = zi;
                              rz += bi * zi;
                            });
  boundary_lines<TX, TY>(N, [&](int gx, int gy) {
    const int64_t g = (int64_t)gy * n1 + gx;
    const double bi = b[g];
    z[g] = bi;
    rz += bi * bi;
  });
  if (rz_part) {
    double v[1] = {rz};
    __shared__ double red[kBlock / 32][1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v[0] = warp_sum(v[0]);
    if (lane == 0) red[warp][0] = v[0];
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kBlock / 32; ++w) t += red[w][0];
      rz_part[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
  }
}

// Restriction of level l fused with the pre-smoothing of level l+1 (one
// kernel per descent step instead of two): the CTA owns a coarse tile,
// forms the fine residual r = b - A x2 over the fine region under the
// coarse tile + halo NU-1 (fine x2 with one more halo), restricts it to
// b_c on that coarse region, then runs the NU pre-smoothing steps of level
// l+1 in shared memory.  Writes b_c and x2_c of the tile (both are read
// again by the level's post-smoother and the next descent step).  The
// coarse buffers alias the fine x2 buffer once the residual is formed.
template <int CX, int CY, int NU, bool F9>
__global__ void __launch_bounds__(kBlock)
    k_mg2_rp(int n1f, int n1c, Sten2 Sf, Sten2 Sc, ChebS C, const double* __restrict__ bf,
             const double* __restrict__ x2f, double* __restrict__ bc, double* __restrict__ x2c,
             const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  constexpr int HX = NU - 1, WL = CX + 2 * HX, HL = CY + 2 * HX;  // coarse region
  constexpr int RW = 2 * WL + 1, RH = 2 * HL + 1;                  // fine residual region
  constexpr int XW = RW + 2, XH = RH + 2;                          // fine x2 region
  static_assert(3 * WL * HL <= XW * XH, "coarse buffers alias the fine x2 buffer");
  using RX = Region<XW, XH>;
  using RB = Region<RW, RH>;
  __shared__ double sxf[XW * XH];
  __shared__ double srf[RW * RH];
  double* sb = sxf;
  double* sx[2] = {sxf + WL * HL, sxf + 2 * WL * HL};
  const int Nf = n1f - 1, Nc = n1c - 1;
  const int ox = 1 + CX * blockIdx.x - HX, oy = 1 + CY * blockIdx.y - HX;
  const int rx0 = 2 * ox - 1, ry0 = 2 * oy - 1;
  {
    double vb[RB::kPer];
    {
      double vx[RX::kPer];
      RX::load(vx, x2f, n1f, rx0 - 1, ry0 - 1);
      RB::load(vb, bf, n1f, rx0, ry0);
      RX::store(sxf, vx);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RB::kPer; ++j) {
      const int k = threadIdx.x + j * kBlock;
      if (k < RB::kN) {
        const int lx = k % RW, ly = k / RW;
        srf[k] = interior2(rx0 + lx, ry0 + ly, Nf)
                     ? vb[j] - sten_apply<F9>(Sf, sxf, (ly + 1) * XW + lx + 1, XW)
                     : 0.0;
      }
    }
  }
  __syncthreads();  // sxf is free from here on
  const double c0 = C.cr[0] * Sc.dinv;
  for (int k = threadIdx.x; k < WL * HL; k += kBlock) {
    const int cx = ox + k % WL, cy = oy + k / WL;
    double v = 0.0;
    if (interior2(cx, cy, Nc)) {
      const int i = (2 * cy - ry0) * RW + (2 * cx - rx0);
      v = srf[i] + 0.5 * (srf[i - 1] + srf[i + 1] + srf[i - RW] + srf[i + RW] +
                          srf[i - RW - 1] + srf[i + RW + 1]);
    }
    sb[k] = v;
    sx[0][k] = c0 * v;  // x_1
  }
  __syncthreads();
  int cur = 0;
#pragma unroll
  for (int k = 1; k < NU - 1; ++k) {
    const double* xk = sx[cur];
    double* xo = sx[cur ^ 1];
    cheb_rows<CX, CY, HX, F9>(NU - 1 - k, Sc, xk, xo, k == 1, sb, C.cd[k], C.cr[k] * Sc.dinv, ox,
                              oy, Nc, [&](int li, int, int, double v) { xo[li] = v; });
    __syncthreads();
    cur ^= 1;
  }
  cheb_rows<CX, CY, HX, F9>(0, Sc, sx[cur], sx[cur ^ 1], NU == 2, sb, C.cd[NU - 1],
                            C.cr[NU - 1] * Sc.dinv, ox, oy, Nc,
                            [&](int li, int gx, int gy, double v) {
                              if (gx > Nc || gy > Nc) return;
                              const int64_t g = (int64_t)gy * n1c + gx;
                              const bool in = interior2(gx, gy, Nc);
                              bc[g] = in ? sb[li] : 0.0;
                              x2c[g] = in ? v : 0.0;
                            });
  boundary_lines<CX, CY>(Nc, [&](int gx, int gy) {
    const int64_t g = (int64_t)gy * n1c + gx;
    bc[g] = 0.0;
    x2c[g] = 0.0;
  });
}

// Restriction of level L-2 fused with the coarsest solve (one CTA): the
// whole fine level (x2 zero-extended, then the residual in place of it) and
// the coarse iterate live in shared memory; b_c of the owned coarse points
// goes to registers, then C.n Chebyshev steps as in k_mg2_coarse.
template <int PPT, bool F9>
__global__ void __launch_bounds__(1024, 1)
    k_mg2_rc(int n1f, int n1, Sten2 Sf, Sten2 S, ChebN C, const double* __restrict__ bf,
             const double* __restrict__ x2f, double* __restrict__ z, const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  extern __shared__ double sm[];
  const int Nf = n1f - 1, mf = n1f * n1f;
  const int N = n1 - 1, m = n1 * n1;
  double* fx = sm;       // fine x2 (zero outside the interior)
  double* fr = sm + mf;  // fine residual
  double* buf[2] = {sm + 2 * mf, sm + 2 * mf + m};
  // row-wise mapping (warp = row, lane = column): no runtime div/mod per point
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int gy = warp; gy < n1f; gy += 32)
    for (int gx = lane; gx < n1f; gx += 32) {
      const int g = gy * n1f + gx;
      const bool in = interior2(gx, gy, Nf);
      fx[g] = in ? x2f[g] : 0.0;
      fr[g] = in ? bf[g] : 0.0;
    }
  for (int g = threadIdx.x; g < 2 * m; g += 1024) buf[0][g] = 0.0;
  __syncthreads();
  for (int gy = 1 + warp; gy < Nf; gy += 32)
    for (int gx = 1 + lane; gx < Nf; gx += 32) {
      const int g = gy * n1f + gx;
      fr[g] -= sten_apply<F9>(Sf, fx, g, n1f);
    }
  __syncthreads();
  // the coarse points of this thread, once: index, or -1 off the interior
  double bi[PPT], xi[PPT], di[PPT];
  int gi[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int g = threadIdx.x + p * 1024;
    double v = 0.0;
    gi[p] = -1;
    if (g < m) {
      const int cx = g % n1, cy = g / n1;
      if (interior2(cx, cy, N)) {
        gi[p] = g;
        const int i = 2 * cy * n1f + 2 * cx;
        v = fr[i] + 0.5 * (fr[i - 1] + fr[i + 1] + fr[i - n1f] + fr[i + n1f] + fr[i - n1f - 1] +
                           fr[i + n1f + 1]);
      }
    }
    bi[p] = v;
    xi[p] = 0.0;
    di[p] = 0.0;
  }
  int cur = 0;
  for (int k = 0; k < C.n; ++k) {
    const double* xs = buf[cur];
    double* xo = buf[cur ^ 1];
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
      const int g = gi[p];
      if (g < 0) continue;  // b_c = 0 there: x stays 0
      const double res = bi[p] - (k ? sten_apply<F9>(S, xs, g, n1) : 0.0);
      const double dn = (k ? C.cd[k] * di[p] : 0.0) + C.cr[k] * S.dinv * res;
      di[p] = dn;
      xi[p] += dn;
      xo[g] = xi[p];
    }
    __syncthreads();
    cur ^= 1;
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int g = threadIdx.x + p * 1024;
    if (g < m) z[g] = xi[p];
  }
}

// Coarsest level: C.n Chebyshev steps from zero in ONE CTA (1024 threads,
// up to PPT grid points per thread); the iterate lives in shared memory
// (two zero-bordered n1 x n1 buffers), b / x / d of the owned points in
// registers.
template <int PPT, bool F9>
__global__ void __launch_bounds__(1024, 1)
    k_mg2_coarse(int n1, Sten2 S, ChebN C, const double* __restrict__ b, double* __restrict__ z,
                 const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  extern __shared__ double sm[];
  const int N = n1 - 1, m = n1 * n1;
  double* buf[2] = {sm, sm + m};
  double bi[PPT], xi[PPT], di[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int g = threadIdx.x + p * 1024;
    bi[p] = g < m ? b[g] : 0.0;
    xi[p] = 0.0;
    di[p] = 0.0;
  }
  for (int g = threadIdx.x; g < 2 * m; g += 1024) sm[g] = 0.0;
  bool inp[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int g = threadIdx.x + p * 1024;
    inp[p] = g < m && interior2(g % n1, g / n1, N);
  }
  __syncthreads();
  int cur = 0;
  for (int k = 0; k < C.n; ++k) {
    const double* xs = buf[cur];
    double* xo = buf[cur ^ 1];
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
      const int g = threadIdx.x + p * 1024;
      if (g >= m) continue;
      if (!inp[p]) {
        xi[p] = bi[p];
        continue;  // stays 0 in the shared iterate (eliminated column)
      }
      const double res = bi[p] - (k ? sten_apply<F9>(S, xs, g, n1) : 0.0);
      const double dn = (k ? C.cd[k] * di[p] : 0.0) + C.cr[k] * S.dinv * res;
      di[p] = dn;
      xi[p] += dn;
      xo[g] = xi[p];
    }
    __syncthreads();
    cur ^= 1;
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int g = threadIdx.x + p * 1024;
    if (g < m) z[g] = xi[p];
  }
}

// Stencil of an interior row of a level matrix: out[(dy+1)*3 + dx+1] for the
// entries of `row` at columns row + dx + n1 dy (|dx|, |dy| <= 1); err[0] = 1
// when the row has any other column.
__global__ void k_mg2_row_stencil(MatView A, int64_t row, int n1, double* out, int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int k = 0; k < 9; ++k) out[k] = 0.0;
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
    const double v = sell_val_at(A.ua, A.a, q0 + k, pos);
    const int64_t d = (int64_t)c - row;
    int hit = -1;
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx)
        if (d == dx + (int64_t)dy * n1) hit = (dy + 1) * 3 + dx + 1;
    if (hit >= 0)
      out[hit] += v;
    else if (v != 0.0)
      err[0] = 1;
  }
}

// max_i |(A v)_i - (S v)_i| and max_i |(A v)_i| over all rows for the
// pseudo-random v_i = sin(0.37 i + 0.11) (block maxima into part[2 * block])
__global__ void __launch_bounds__(kBlock)
    k_mg2_verify(MatView A, int n1, Sten2 S, const uint8_t* __restrict__ mask, double* part) {
  const int N = n1 - 1;
  const int64_t m = (int64_t)n1 * n1;
  double emax = 0.0, amax = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int gx = (int)(i % n1), gy = (int)(i / n1);
    const bool in = interior2(gx, gy, N);
    if (in == (mask[i] != 0)) {  // the mask must be exactly the boundary
      emax = INFINITY;
      continue;
    }
    // A v through the SELL arrays
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
      av += sell_val_at(A.ua, A.a, q0 + k, pos) * sin(0.37 * c + 0.11);
    }
    double sv;
    if (!in) {
      sv = sin(0.37 * i + 0.11);  // identity row
    } else {
      sv = 0.0;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int x = gx + dx, y = gy + dy;
          if (interior2(x, y, N)) sv += S.c[dy + 1][dx + 1] * sin(0.37 * ((int64_t)y * n1 + x) + 0.11);
        }
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
  // structured 2D path (see k_mg2_*): available / in use
  bool s2_ok = false, s2_on = false;
  std::vector<irk::Sten2> sten;
  std::vector<bool> f9;
  std::vector<irk::ChebS> c2;  // per level (lmax differs)
  irk::ChebN cn{};
  // fast sine-transform preconditioner of the level-0 block (irk_dst.cuh):
  // available / in use instead of the V-cycle
  bool dst_ok = false, dst_on = false;
  int dst_N = 0;
  irk::DstStencil dstS{};
  double* dst_mem = nullptr;
  double* dst_T = nullptr;      // N x N spectral work array
  double* dst_cos = nullptr;    // cos(pi k / N), k = 0..N
  double2* dst_tw = nullptr;    // e^{-2 pi i q / (2N)}, q < 2N

  // Set up the sine-transform preconditioner on a verified level-0 stencil
  // (structured path available): N a power of two in [32, 2048], the
  // symmetrised stencil's eigenvalues positive (bilinear in cos(pi k/N),
  // cos(pi l/N): the extremes are at the corners).
  int setup_dst(irk_ctx* ctx) {
    using namespace irk;
    dst_ok = false;
    if (!s2_ok || dim != 2) return IRK_OK;
    const int N = (int)lev[0].g.n1 - 1;
    if (N < 32 || N > 2048 || (N & (N - 1)) != 0) return IRK_OK;
    const Sten2& C = sten[0];
    DstStencil S;
    S.s00 = C.c[1][1];
    S.s10 = 0.5 * (C.c[1][0] + C.c[1][2]);
    S.s01 = 0.5 * (C.c[0][1] + C.c[2][1]);
    S.s11 = 0.25 * (C.c[0][0] + C.c[0][2] + C.c[2][0] + C.c[2][2]);
    const double ce[2] = {std::cos(M_PI / N), -std::cos(M_PI / N)};
    for (double a : ce)
      for (double b : ce) {
        const double lam = S.s00 + 2 * S.s10 * a + 2 * S.s01 * b + 4 * S.s11 * a * b;
        if (!(lam > 0.0) || !std::isfinite(lam)) return IRK_OK;
      }
    const int L = 2 * N;
    const size_t doubles = (size_t)N * N + (N + 1) + 2 * (size_t)L + 8;
    if (!dst_mem) IRK_CUDA(cudaMalloc(&dst_mem, doubles * sizeof(double)));
    dst_T = dst_mem;
    dst_tw = reinterpret_cast<double2*>(dst_mem + (size_t)N * N);  // 16-byte aligned (N even)
    dst_cos = dst_mem + (size_t)N * N + 2 * (size_t)L;
    std::vector<double> host(2 * (size_t)L + N + 1);
    for (int q = 0; q < L; ++q) {
      // exact at the multiples of pi/4 (the cos/sin of the reduced angle)
      const double a = -2.0 * M_PI * (double)q / (double)L;
      host[2 * q] = std::cos(a);
      host[2 * q + 1] = std::sin(a);
    }
    for (int k = 0; k <= N; ++k) host[2 * (size_t)L + k] = std::cos(M_PI * (double)k / N);
    IRK_CUDA(cudaMemcpyAsync(dst_tw, host.data(), host.size() * sizeof(double),
                             cudaMemcpyHostToDevice, ctx->stream));
    IRK_CUDA(cudaStreamSynchronize(ctx->stream));
    IRK_TRY(dst_attrs(L));
    dstS = S;
    dst_N = N;
    dst_ok = true;
    return IRK_OK;
  }

  template <int L>
  static int dst_attrs_l() {
    IRK_CUDA(cudaFuncSetAttribute(irk::k_dst_rows<L, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  irk::fpad_len(L) * 16));
    IRK_CUDA(cudaFuncSetAttribute(irk::k_dst_rows<L, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  irk::fpad_len(L) * 16));
    IRK_CUDA(cudaFuncSetAttribute(irk::k_dst_cols<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  2 * irk::fpad_len(L) * 16));
    return IRK_OK;
  }
  // half-length transforms (irk_dst.cuh dsth_transform): N >= 256;
  // env IRK_DST_FULL keeps the length-2N odd-extension kernels (A/B)
  static bool dst_half(int N) {
    static const bool full = getenv("IRK_DST_FULL") != nullptr;
    return !full && N >= 256;
  }
  template <int N>
  static int dsth_attrs_n() {
    const int one = irk::fpad_len(N) * 16;
    IRK_CUDA(cudaFuncSetAttribute(irk::k_dsth_rows<N, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, one));
    IRK_CUDA(cudaFuncSetAttribute(irk::k_dsth_rows<N, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, one));
    IRK_CUDA(cudaFuncSetAttribute(irk::k_dsth_cols<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  2 * one));
    return IRK_OK;
  }
  static int dst_attrs(int L) {
    if (dst_half(L / 2)) {
      switch (L / 2) {
        case 256: return dsth_attrs_n<256>();
        case 512: return dsth_attrs_n<512>();
        case 1024: return dsth_attrs_n<1024>();
        case 2048: return dsth_attrs_n<2048>();
      }
    }
    switch (L) {
      case 64: return dst_attrs_l<64>();
      case 128: return dst_attrs_l<128>();
      case 256: return dst_attrs_l<256>();
      case 512: return dst_attrs_l<512>();
      case 1024: return dst_attrs_l<1024>();
      case 2048: return dst_attrs_l<2048>();
      case 4096: return dst_attrs_l<4096>();
    }
    return IRK_EINVAL;
  }

  template <int L>
  int apply_dst_l(irk_ctx* ctx, cudaStream_t s, const double* r, double* z, const int* stop,
                  const irk::SkipCtl& sk, double* rz_part) {
    using namespace irk;
    const int N = dst_N;
    // fused CG: the forward row kernel decides the skip (sk) and publishes
    // it in sk.st->skip for the other two; the inverse one writes rz_part
    constexpr size_t kBuf = (size_t)fpad_len(L) * 16;  // one padded FFT buffer
    launch(k_dst_rows<L, false>, N / 2, L / 8, kBuf, s, N, r, dst_T, r, dst_tw, stop, sk,
           (double*)nullptr);
    launch(k_dst_cols<L>, N / 4, L / 4, 2 * kBuf, s, N, dst_T, dstS, dst_cos, dst_tw, stop);
    launch(k_dst_rows<L, true>, N / 2, L / 8, kBuf, s, N, dst_T, z, r, dst_tw, stop, SkipCtl{},
           rz_part);
    ctx->launches += 3;
    return cudaPeekAtLastError() == cudaSuccess ? IRK_OK : IRK_ECUDA;
  }
  template <int N>
  int apply_dsth_n(irk_ctx* ctx, cudaStream_t s, const double* r, double* z, const int* stop,
                   const irk::SkipCtl& sk, double* rz_part) {
    using namespace irk;
    constexpr size_t kBuf = (size_t)fpad_len(N) * 16;
    launch(k_dsth_rows<N, false>, N / 2, N / 8, kBuf, s, r, dst_T, r, dst_cos, dst_tw, stop, sk,
           (double*)nullptr);
    launch(k_dsth_cols<N>, N / 4, N / 4, 2 * kBuf, s, dst_T, dstS, dst_cos, dst_tw, stop);
    launch(k_dsth_rows<N, true>, N / 2, N / 8, kBuf, s, (const double*)dst_T, z, r, dst_cos,
           dst_tw, stop, SkipCtl{}, rz_part);
    ctx->launches += 3;
    return cudaPeekAtLastError() == cudaSuccess ? IRK_OK : IRK_ECUDA;
  }
  // z = B_s^-1 r (r != z)
  int apply_dst(irk_ctx* ctx, cudaStream_t s, const double* r, double* z, const int* stop,
                const irk::SkipCtl& sk = irk::SkipCtl{}, double* rz_part = nullptr) {
    if (dst_half(dst_N)) {
      switch (dst_N) {
        case 256: return apply_dsth_n<256>(ctx, s, r, z, stop, sk, rz_part);
        case 512: return apply_dsth_n<512>(ctx, s, r, z, stop, sk, rz_part);
        case 1024: return apply_dsth_n<1024>(ctx, s, r, z, stop, sk, rz_part);
        case 2048: return apply_dsth_n<2048>(ctx, s, r, z, stop, sk, rz_part);
      }
    }
    switch (2 * dst_N) {
      case 64: return apply_dst_l<64>(ctx, s, r, z, stop, sk, rz_part);
      case 128: return apply_dst_l<128>(ctx, s, r, z, stop, sk, rz_part);
      case 256: return apply_dst_l<256>(ctx, s, r, z, stop, sk, rz_part);
      case 512: return apply_dst_l<512>(ctx, s, r, z, stop, sk, rz_part);
      case 1024: return apply_dst_l<1024>(ctx, s, r, z, stop, sk, rz_part);
      case 2048: return apply_dst_l<2048>(ctx, s, r, z, stop, sk, rz_part);
      case 4096: return apply_dst_l<4096>(ctx, s, r, z, stop, sk, rz_part);
    }
    irk::set_error("irk_mg: no sine-transform plan");
    return IRK_EINVAL;
  }

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
        launch(k_mg_cheb_st<7>, grid_for(ctx, L.m), kBlock, 0, s, L.m, L.A, L.mask, L.dinv, b, xin,
                                                             L.d, xo, cd[k], cr[k], stop);
      else if (xin && L.st == 15)
        launch(k_mg_cheb_st<15>, grid_for(ctx, L.m), kBlock, 0, s, L.m, L.A, L.mask, L.dinv, b, xin,
                                                              L.d, xo, cd[k], cr[k], stop);
      else if (xin && L.st == 3)
        launch(k_mg_cheb_st<3>, grid_for(ctx, L.m), kBlock, 0, s, L.m, L.A, L.mask, L.dinv, b, xin,
                                                             L.d, xo, cd[k], cr[k], stop);
      else
        launch(k_mg_cheb, grid_for(ctx, L.m), kBlock, 0, s, L.m, L.A, L.mask, L.dinv, b, xin, L.d,
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
      launch(k_mg_residual_st<7>, grid_for(ctx, L.m), kBlock, 0, s, L.m, L.A, L.mask, b, L.x[c],
                                                                 L.r, stop);
    else if (L.st == 15)
      launch(k_mg_residual_st<15>, grid_for(ctx, L.m), kBlock, 0, s, L.m, L.A, L.mask, b, L.x[c],
                                                                  L.r, stop);
    else if (L.st == 3)
      launch(k_mg_residual_st<3>, grid_for(ctx, L.m), kBlock, 0, s, L.m, L.A, L.mask, b, L.x[c],
                                                                 L.r, stop);
    else
      launch(k_mg_residual, grid_for(ctx, L.m), kBlock, 0, s, L.m, L.A, L.mask, b, L.x[c], L.r,
                                                          stop);
    ctx->launches++;
    MgLevel& Cc = lev[l + 1];
    launch(k_mg_restrict, (unsigned)((Cc.m + kBlock - 1) / kBlock), kBlock, 0, s, 
        Cc.m, Cc.g, L.g, Cc.mask, L.r, Cc.b, stop);
    ctx->launches++;
    const int cc = vcycle(ctx, s, l + 1, Cc.b, nullptr, stop);
    if (cc < 0) return -1;
    launch(k_mg_prolong, (unsigned)((L.m + kBlock - 1) / kBlock), kBlock, 0, s, 
        L.m, L.g, Cc.g, Cc.x[cc], L.x[c], stop);
    ctx->launches++;
    return smooth(ctx, s, l, b, c, nu, 0.25, out, stop);
  }

  // structured 2D V-cycle: z_l = V_l(b_l) (see the k_mg2_* kernels).  The
  // descent fuses each restriction with the next level's pre-smoothing
  // (k_mg2_rp) and the last one with the coarsest solve (k_mg2_rc): 11
  // kernels instead of 16 on 6 levels.  Env IRK_MG_NOFUSE: separate kernels.
  int coarse2(irk_ctx* ctx, cudaStream_t s, const double* b, double* out, const int* stop) {
    using namespace irk;
    const int l = (int)lev.size() - 1;
    const MgLevel& L = lev[l];
    const int n1 = (int)L.g.n1;
    const Sten2& S = sten[l];
    const bool F = f9[l];
    const int ppt = (int)((L.m + 1023) / 1024);
    const size_t sh = 2 * (size_t)L.m * sizeof(double);
#define IRK_CO(P)                                                                           \
  (F ? launch(k_mg2_coarse<P, true>, 1, 1024, sh, s, n1, S, cn, b, out, stop)                  \
     : launch(k_mg2_coarse<P, false>, 1, 1024, sh, s, n1, S, cn, b, out, stop))
    if (ppt <= 1) IRK_CO(1);
    else if (ppt <= 2) IRK_CO(2);
    else if (ppt <= 4) IRK_CO(4);
    else IRK_CO(8);
#undef IRK_CO
    ctx->launches++;
    return cudaPeekAtLastError() == cudaSuccess ? IRK_OK : IRK_ECUDA;
  }

  bool fuse_ok() const {
    static const bool off = getenv("IRK_MG_NOFUSE") != nullptr;
    return !off && nu <= 4;
  }
  // k_mg2_rc: the fine level and the coarsest fit one CTA's shared memory
  bool rc_ok() const {
    const int64_t mf = lev[lev.size() - 2].m, mc = lev.back().m;
    return fuse_ok() && mc <= 2048 && (2 * mf + 2 * mc) * (int64_t)sizeof(double) <= kRcSmem;
  }
  static constexpr int kRcSmem = 200 * 1024;

  // sk / rz_part (fused CG, top level only): the top pre-smoother takes the
  // skip decision, the top post-smoother writes the r.z partials
  int vcycle2(irk_ctx* ctx, cudaStream_t s, int l, const double* b, double* out,
              const int* stop, const irk::SkipCtl& sk = irk::SkipCtl{},
              double* rz_part = nullptr) {
    using namespace irk;
    if (l == (int)lev.size() - 1) return coarse2(ctx, s, b, out, stop);
    const MgLevel& L = lev[l];
    const int n1 = (int)L.g.n1, N = n1 - 1;
    const Sten2& S = sten[l];
    const ChebS C2 = c2[l];
    const bool F = f9[l];
    double* x2 = L.x[0];
#define IRK_MG2(N_, KER, NU, ...)                                                          \
  do {                                                                                     \
    if ((N_) >= 512) {                                                                     \
      const dim3 g_(((N_) + kBTX - 1) / kBTX, ((N_) + kBTY - 1) / kBTY);                   \
      if (F) launch(KER<kBTX, kBTY, NU, true>, g_, kBlock, 0, s, __VA_ARGS__);             \
      else launch(KER<kBTX, kBTY, NU, false>, g_, kBlock, 0, s, __VA_ARGS__);              \
    } else {                                                                               \
      const dim3 g_(((N_) + 31) / 32, ((N_) + 7) / 8);                                     \
      if (F) launch(KER<32, 8, NU, true>, g_, kBlock, 0, s, __VA_ARGS__);                  \
      else launch(KER<32, 8, NU, false>, g_, kBlock, 0, s, __VA_ARGS__);                   \
    }                                                                                      \
    ctx->launches++;                                                                       \
  } while (0)
#define IRK_NU(N_, KER, ...)                            \
  do {                                                  \
    if (nu == 2) IRK_MG2(N_, KER, 2, __VA_ARGS__);      \
    else if (nu == 3) IRK_MG2(N_, KER, 3, __VA_ARGS__); \
    else IRK_MG2(N_, KER, 4, __VA_ARGS__);              \
  } while (0)
    if (l == 0) IRK_NU(N, k_mg2_pre, n1, S, C2, b, x2, sk.st ? nullptr : stop, sk);  // top pre
    const MgLevel& Cc = lev[l + 1];
    const int n1c = (int)Cc.g.n1, Nc = n1c - 1;
    const bool last = l + 2 == (int)lev.size();
    const dim3 gr((Nc + 31) / 32, (Nc + 7) / 8);
    if (last && rc_ok()) {
      const int ppt = (int)((Cc.m + 1023) / 1024);
      const size_t sh = (2 * (size_t)L.m + 2 * (size_t)Cc.m) * sizeof(double);
      if (ppt <= 1) {
        if (F) launch(k_mg2_rc<1, true>, 1, 1024, sh, s, n1, n1c, S, sten[l + 1], cn, b, x2, Cc.x[1], stop);
        else launch(k_mg2_rc<1, false>, 1, 1024, sh, s, n1, n1c, S, sten[l + 1], cn, b, x2, Cc.x[1], stop);
      } else {
        if (F) launch(k_mg2_rc<2, true>, 1, 1024, sh, s, n1, n1c, S, sten[l + 1], cn, b, x2, Cc.x[1], stop);
        else launch(k_mg2_rc<2, false>, 1, 1024, sh, s, n1, n1c, S, sten[l + 1], cn, b, x2, Cc.x[1], stop);
      }
      ctx->launches++;
    } else if (!last && fuse_ok()) {
      // restriction + the next level's pre-smoothing (32 x 8 coarse tiles)
      const ChebS Cn = c2[l + 1];
      const bool F1 = F || f9[l + 1];
#define IRK_RP(NU)                                                                              \
  (F1 ? launch(k_mg2_rp<32, 8, NU, true>, gr, kBlock, 0, s, n1, n1c, S, sten[l + 1], Cn, b, x2, \
               Cc.b, Cc.x[0], stop)                                                              \
      : launch(k_mg2_rp<32, 8, NU, false>, gr, kBlock, 0, s, n1, n1c, S, sten[l + 1], Cn, b, x2, \
               Cc.b, Cc.x[0], stop))
      if (nu == 2) IRK_RP(2);
      else if (nu == 3) IRK_RP(3);
      else IRK_RP(4);
#undef IRK_RP
      ctx->launches++;
    } else {
      if (F) launch(k_mg2_restrict<32, 8, true>, gr, kBlock, 0, s, n1, n1c, S, b, x2, Cc.b, stop);
      else launch(k_mg2_restrict<32, 8, false>, gr, kBlock, 0, s, n1, n1c, S, b, x2, Cc.b, stop);
      ctx->launches++;
      if (last) {
        IRK_TRY(coarse2(ctx, s, Cc.b, Cc.x[1], stop));
      } else {
        const ChebS Cn = c2[l + 1];
        const bool Fs = F;
        {
          const bool F = Fs || f9[l + 1];
          const Sten2& S1 = sten[l + 1];
          IRK_NU(Nc, k_mg2_pre, n1c, S1, Cn, Cc.b, Cc.x[0], stop, SkipCtl{});
        }
      }
    }
    if (cudaPeekAtLastError() != cudaSuccess) return IRK_ECUDA;
    if (!last) IRK_TRY(vcycle2(ctx, s, l + 1, Cc.b, Cc.x[1], stop));
    const double* ec = Cc.x[1];
    IRK_NU(N, k_mg2_post, n1, n1c, S, C2, b, x2, ec, out, stop, l == 0 ? rz_part : nullptr);
#undef IRK_NU
#undef IRK_MG2
    return cudaPeekAtLastError() == cudaSuccess ? IRK_OK : IRK_ECUDA;
  }

  // Enable the structured path when every level is a verified 2D stencil
  // operator with the full-boundary Dirichlet set (else keep the generic one).
  int setup_s2(irk_ctx* ctx) {
    using namespace irk;
    s2_ok = false;
    const int nl = (int)lev.size();
    if (dim != 2 || nu < 2 || nu > kMaxNu || ncoarse > kMaxCoarse) return IRK_OK;
    if (lev.back().m > 8 * 1024) return IRK_OK;
    for (const MgLevel& L : lev)
      if (!L.mask || L.g.n1 - 1 < 4 || L.g.n1 > 46341) return IRK_OK;
    IRK_TRY(ensure_red(ctx, 2 * (size_t)ctx->num_sms * 4 + 64));
    sten.assign(nl, Sten2{});
    f9.assign(nl, false);
    for (int l = 0; l < nl; ++l) {
      const MgLevel& L = lev[l];
      const int n1 = (int)L.g.n1, N = n1 - 1;
      int* err = (int*)ctx->counters + (kNumCounters - 2);
      IRK_CUDA(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
      k_mg2_row_stencil<<<1, 32, 0, ctx->stream>>>(L.A, (int64_t)(N / 2) * n1 + N / 2, n1,
                                                    ctx->red, err);
      IRK_CHECK_LAUNCH(ctx);
      double c[9];
      int herr = 0;
      IRK_CUDA(cudaMemcpyAsync(c, ctx->red, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
      IRK_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      IRK_CUDA(cudaStreamSynchronize(ctx->stream));
      if (herr || !(c[4] != 0.0) || !std::isfinite(c[4])) return IRK_OK;
      Sten2& S = sten[l];
      for (int k = 0; k < 9; ++k) S.c[k / 3][k % 3] = c[k];
      S.dinv = 1.0 / c[4];
      f9[l] = c[2] != 0.0 || c[6] != 0.0;
      const int G = ctx->num_sms * 4;
      k_mg2_verify<<<G, kBlock, 0, ctx->stream>>>(L.A, n1, S, L.mask, ctx->red);
      IRK_CHECK_LAUNCH(ctx);
      std::vector<double> part(2 * G);
      IRK_CUDA(cudaMemcpyAsync(part.data(), ctx->red, part.size() * sizeof(double),
                               cudaMemcpyDeviceToHost, ctx->stream));
      IRK_CUDA(cudaStreamSynchronize(ctx->stream));
      double e = 0.0, a = 0.0;
      for (int b = 0; b < G; ++b) {
        e = std::fmax(e, part[2 * b]);
        a = std::fmax(a, part[2 * b + 1]);
      }
      if (!(e <= 1e-12 * a)) return IRK_OK;
    }
    // Chebyshev coefficients, as smooth(): [lmax/4, lmax] on the fine
    // levels, [0.05 lmax, lmax] with ncoarse steps on the coarsest
    c2.assign(nl, ChebS{});
    std::vector<double> cd, cr;
    for (int l = 0; l + 1 < nl; ++l) {
      cheb(0.25 * lev[l].lmax, lev[l].lmax, nu, cd, cr);
      for (int k = 0; k < nu; ++k) {
        c2[l].cd[k] = cd[k];
        c2[l].cr[k] = cr[k];
      }
    }
    cheb(0.05 * lev.back().lmax, lev.back().lmax, ncoarse, cd, cr);
    cn.n = ncoarse;
    for (int k = 0; k < ncoarse; ++k) {
      cn.cd[k] = cd[k];
      cn.cr[k] = cr[k];
    }
    s2_ok = true;
    return IRK_OK;
  }

  // fused CG support (structured path with at least two levels): the
  // top-level post-smoother's CTAs write the r.z partials
  int fused_rz_count() override {
    static const bool off = getenv("IRK_MG_NOFUSE") || getenv("IRK_CG_NOFUSE");
    // sine-transform preconditioner: one partial per CTA of the inverse row
    // kernel (row-kernel blocks of at least kBlock threads: N >= 1024)
    if (dst_on) {
      // the row kernels' block: N / 8 threads (half-length) or N / 4
      const int nt = dst_half(dst_N) ? dst_N / 8 : dst_N / 4;
      const bool ok = dst_half(dst_N) ? (nt >= irk::kBlock || 2 * nt == irk::kBlock)
                                      : nt >= irk::kBlock;
      return (!off && ok) ? dst_N / 2 : 0;
    }
    if (off || !s2_on || lev.size() < 2) return 0;
    const int N = (int)lev[0].g.n1 - 1;
    return N >= 512 ? ((N + irk::kBTX - 1) / irk::kBTX) * ((N + irk::kBTY - 1) / irk::kBTY)
                    : ((N + 31) / 32) * ((N + 7) / 8);
  }

  // the sine-transform-preconditioned CG reaches 1e-6 in 2 iterations (3-4
  // at 1e-12): issue 2 with the init sequence, the rest from the loop
  int prefix_iters() override { return dst_on ? 2 : -1; }

  int apply_fused(irk_ctx* ctx, cudaStream_t s, const double* r, double* z,
                  const irk::SkipCtl& sk, double* rz_part) override {
    const int* stop = sk.st ? &sk.st->skip : nullptr;
    if (dst_on) {
      const int e = apply_dst(ctx, s, r, z, stop, sk, rz_part);
      if (e != IRK_OK || cudaGetLastError() != cudaSuccess) {
        irk::set_error("irk_mg: fused sine-transform preconditioner launch failed");
        return IRK_ECUDA;
      }
      return IRK_OK;
    }
    const int e = vcycle2(ctx, s, 0, r, z, stop, sk, rz_part);
    if (e != IRK_OK || cudaGetLastError() != cudaSuccess) {
      irk::set_error("irk_mg: fused structured V-cycle launch failed");
      return IRK_ECUDA;
    }
    return IRK_OK;
  }

  int apply(irk_ctx* ctx, cudaStream_t s, const double* r, double* z,
            const int* stop) override {
    if (dst_on) {
      const int e = apply_dst(ctx, s, r, z, stop);
      if (e != IRK_OK || cudaGetLastError() != cudaSuccess) {
        irk::set_error("irk_mg: sine-transform preconditioner launch failed");
        return IRK_ECUDA;
      }
      return IRK_OK;
    }
    if (s2_on) {
      const int e = vcycle2(ctx, s, 0, r, z, stop);
      if (e != IRK_OK || cudaGetLastError() != cudaSuccess) {
        irk::set_error("irk_mg: structured V-cycle launch failed");
        return IRK_ECUDA;
      }
      return IRK_OK;
    }
    const int c = vcycle(ctx, s, 0, r, z, stop);
    if (c < 0 || cudaGetLastError() != cudaSuccess) {
      irk::set_error("irk_mg: V-cycle launch failed");
      return IRK_ECUDA;
    }
    return IRK_OK;
  }

  ~irk_mg() override {
    if (mem) cudaFree(mem);
    if (dst_mem) cudaFree(dst_mem);
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
  IRK_REQUIRE(nu >= 0 && nu <= 8 && ncoarse >= 1 && ncoarse <= 64,
              "irk_mg_create: 0 <= nu <= 8 (0: automatic), 1 <= ncoarse <= 64");
  irk_mg* mg = new irk_mg();
  mg->uid = g_mg_uid.fetch_add(1);
  mg->dim = dim;
  // nu = 0 (automatic): 2.  Measured on B200 (config 2): nu = 3 / 4 cut the
  // CG iterations of a block solve from 6 to 5 / 4 and the solve time by
  // 6 / 11 %, but the outer FGMRES then needs 9.0 instead of 8.1 iterations
  // per step (the inexact blocks change), so the step is slower.
  const bool nu_auto = nu == 0;
  mg->nu = nu_auto ? 2 : nu;
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
  {
    const int e = mg->setup_s2(ctx);
    if (e != IRK_OK) {
      delete mg;
      return e;
    }
    static const bool generic = getenv("IRK_MG_GENERIC") != nullptr;
    mg->s2_on = mg->s2_ok && !generic;
    const int ed = mg->setup_dst(ctx);
    if (ed != IRK_OK) {
      delete mg;
      return ed;
    }
    if (mg->s2_ok) {
      // dynamic shared memory of the single-CTA coarsest kernel (2 buffers)
      const int sh4 = 2 * 4 * 1024 * (int)sizeof(double);
      const int sh8 = 2 * 8 * 1024 * (int)sizeof(double);
      IRK_CUDA(cudaFuncSetAttribute(k_mg2_coarse<4, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, sh4));
      IRK_CUDA(cudaFuncSetAttribute(k_mg2_coarse<4, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, sh4));
      IRK_CUDA(cudaFuncSetAttribute(k_mg2_coarse<8, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, sh8));
      IRK_CUDA(cudaFuncSetAttribute(k_mg2_coarse<8, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, sh8));
      for (const void* fn : {(const void*)k_mg2_rc<1, false>, (const void*)k_mg2_rc<1, true>,
                             (const void*)k_mg2_rc<2, false>, (const void*)k_mg2_rc<2, true>})
        IRK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      irk_mg::kRcSmem));
    }
  }
  *out = mg;
  return IRK_OK;
}

int irk_mg_set_structured(irk_mg* mg, int on) {
  IRK_REQUIRE(mg, "irk_mg_set_structured: NULL argument");
  IRK_REQUIRE(!on || mg->s2_ok,
              "irk_mg_set_structured: no structured path for this hierarchy (needs 2D levels "
              "with the full-boundary Dirichlet set, nu = 2, a coarsest level <= 8192 points)");
  if ((on != 0) != mg->s2_on) {
    mg->s2_on = on != 0;
    mg->uid = g_mg_uid.fetch_add(1);  // cached graphs hold the other kernel sequence
  }
  return IRK_OK;
}

int irk_mg_set_dst(irk_mg* mg, int on) {
  IRK_REQUIRE(mg, "irk_mg_set_dst: NULL argument");
  IRK_REQUIRE(!on || mg->dst_ok,
              "irk_mg_set_dst: no sine-transform preconditioner for this block (needs a verified "
              "2D grid stencil with the full-boundary Dirichlet set, N a power of two in "
              "[32, 2048], positive symmetrised eigenvalues)");
  if ((on != 0) != mg->dst_on) {
    mg->dst_on = on != 0;
    mg->uid = g_mg_uid.fetch_add(1);  // cached graphs hold the other kernel sequence
  }
  return IRK_OK;
}

int irk_mg_dst_info(const irk_mg* mg, int* available, int* on) {
  IRK_REQUIRE(mg, "irk_mg_dst_info: NULL argument");
  if (available) *available = mg->dst_ok ? 1 : 0;
  if (on) *on = mg->dst_on ? 1 : 0;
  return IRK_OK;
}

int irk_mg_info(const irk_mg* mg, int* nlev, int* structured) {
  IRK_REQUIRE(mg, "irk_mg_info: NULL argument");
  if (nlev) *nlev = (int)mg->lev.size();
  if (structured) *structured = mg->s2_on ? 1 : 0;
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

int irk_mg_pcg_multi(irk_ctx* ctx, int n, irk_mg* const* mgs, const double* rhs_dev,
                     int64_t ld_rhs, int64_t rhs_step, double* x_dev, int64_t ld_x,
                     int64_t x_step, double rtol, double atol, int maxit, int* its_host,
                     double* relres_host) {
  IRK_REQUIRE(ctx && mgs && n >= 0, "irk_mg_pcg_multi: NULL argument");
  const bool deferred = !its_host && !relres_host && ctx->log_on;
  return run_forked(ctx, n, deferred, [&](int k, irk_ctx* c) {
    return irk_mg_pcg(c, mgs[k], rhs_dev + k * rhs_step, ld_rhs, x_dev + k * x_step, ld_x, rtol,
                      atol, maxit, its_host ? its_host + k : nullptr,
                      relres_host ? relres_host + k : nullptr);
  });
}

}  // extern "C"
