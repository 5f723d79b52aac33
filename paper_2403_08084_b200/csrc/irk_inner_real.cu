// Real SPD diagonal blocks: batched Jacobi-PCG (irk_pcg) and
// Jacobi-Chebyshev (irk_chebyshev).  Kernels in irk_inner.cuh, plus the
// persistent single-block PCG below.
#include <cooperative_groups.h>

#include <cstdlib>

#include "irk_inner.cuh"

namespace cg = cooperative_groups;

namespace irk {

// ------------------------------------------------- persistent Jacobi-PCG
// One cooperative launch runs the WHOLE solve of one pre-combined block
// (nb = 1, identity rows baked in): one CTA of 1024 threads per SM, rows
// statically partitioned by SELL slices (block b owns a contiguous slice
// range; warp w of the block owns slices w, w+32, ... of it, lane = row in
// slice).  p, r and D^-1 of the block's rows live in shared memory, q = B p
// in registers, x accumulates in the (L2-resident) output; p is also
// published to global memory once per iteration for the SpMV gathers of the
// other blocks.  Three grid barriers per iteration (p
// visible; p.q; r.z and r.r), each reduction summed in block order by every
// block so all blocks take identical, deterministic decisions.
constexpr int kPersistThreads = 1024;

// The block's slot headers (colhdr / uval of its slice range) are staged in
// shared memory at kernel start, so the per-entry decode is a shared-memory
// read; p is gathered with L1-cached loads (the grid barrier's gpu-scope
// fence invalidates L1, so every iteration sees the freshly published p).
template <int RMAX, int MAXW>
__global__ void __launch_bounds__(kPersistThreads, 1)
    k_pcg_persist(int64_t m, int64_t nslices, int64_t slices_per_block, MatView A,
                  const double* __restrict__ rhs, int64_t ld_rhs, double* __restrict__ xout,
                  int64_t ld_x, double* pg, double* __restrict__ part, double rtol2,
                  double atol2, int maxit, SysState<double>* st) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double smem[];
  __shared__ double wred[kPersistThreads / 32][2];
  __shared__ double bcast[2];
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s0 = (int64_t)blockIdx.x * slices_per_block;
  const int64_t s1 = min(nslices, s0 + slices_per_block);
  const int cap = (int)(slices_per_block * kSlice);
  const int hcap = (int)(slices_per_block * MAXW);
  double* sp = smem;  // p of the block's rows
  double* sr = smem + cap;
  double* sd = smem + 2 * cap;
  double* hv = smem + 3 * cap;
  int* hc = reinterpret_cast<int*>(smem + 3 * cap + hcap);
  // stage the block's slot headers
  const int qb = s0 < s1 ? __ldg(A.slice_ptr + s0) / kSlice : 0;
  const int qe = s0 < s1 ? __ldg(A.slice_ptr + s1) / kSlice : 0;
  for (int t = threadIdx.x; t < qe - qb; t += blockDim.x) {
    hv[t] = __ldg(A.ua + qb + t);
    hc[t] = __ldg(A.colhdr + qb + t);
  }
  __syncthreads();

  // block reduction of (a, b) -> part[slot*2*G + {0,1}*G + block], then
  // after the grid barrier every block sums all partials in block order.
  auto reduce2 = [&](double a, double b, int slot, double& ra, double& rb) {
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
      wred[warp][0] = a;
      wred[warp][1] = b;
    }
    __syncthreads();
    if (warp == 0) {
      double ta = wred[lane][0], tb = wred[lane][1];
      ta = warp_sum(ta);
      tb = warp_sum(tb);
      if (lane == 0) {
        part[(int64_t)slot * 2 * G + blockIdx.x] = ta;
        part[(int64_t)slot * 2 * G + G + blockIdx.x] = tb;
      }
    }
    grid.sync();
    if (warp == 0) {
      double ta = 0.0, tb = 0.0;
      for (int q = lane; q < G; q += 32) {
        ta += __ldcg(part + (int64_t)slot * 2 * G + q);
        tb += __ldcg(part + (int64_t)slot * 2 * G + G + q);
      }
      ta = warp_sum(ta);
      tb = warp_sum(tb);
      if (lane == 0) {
        bcast[0] = ta;
        bcast[1] = tb;
      }
    }
    __syncthreads();
    ra = bcast[0];
    rb = bcast[1];
    __syncthreads();
  };

  // ---- init: x = 0, r = b, D^-1, rho = r.z, bb = b.b
  double rho_p = 0.0, bb_p = 0.0;
  double q[RMAX];
#pragma unroll
  for (int j = 0; j < RMAX; ++j) {
    q[j] = 0.0;
    const int64_t sl = s0 + warp + 32 * j;
    if (sl < s1) {
      const int64_t row = sl * kSlice + lane;
      const int lr = (int)((sl - s0) * kSlice + lane);
      if (row < m) {
        const int dp = A.diag_pos[row];
        const double d = dp >= 0 ? A.a[dp] : 0.0;
        const double di = 1.0 / d;
        const double b = rhs[row * ld_rhs];
        xout[row * ld_x] = 0.0;
        sp[lr] = 0.0;
        sr[lr] = b;
        sd[lr] = di;
        rho_p += b * (di * b);
        bb_p += b * b;
      }
    }
  }
  double rho, bb;
  reduce2(rho_p, bb_p, 0, rho, bb);
  const double tol2 = fmax(rtol2 * bb, atol2);
  int its = 0, code = 0;
  double rr = bb, beta = 0.0;
  bool done = !(bb > tol2);
  if (!done && (!isfinite(rho) || rho == 0.0)) {
    done = true;
    code = 2;
  }
  while (!done) {
    // ---- A: p = z + beta p  (z = D^-1 r), publish p
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
      const int64_t sl = s0 + warp + 32 * j;
      if (sl < s1) {
        const int64_t row = sl * kSlice + lane;
        const int lr = (int)((sl - s0) * kSlice + lane);
        if (row < m) {
          const double pj = sd[lr] * sr[lr] + beta * sp[lr];
          sp[lr] = pj;
          pg[row] = pj;
        }
      }
    }
    grid.sync();
    // ---- B: q = B p, mu = p.q
    double mu_p = 0.0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
      const int64_t sl = s0 + warp + 32 * j;
      if (sl < s1) {
        const int64_t row = sl * kSlice + lane;
        const int base = __ldg(A.slice_ptr + sl);
        const int width = (__ldg(A.slice_ptr + sl + 1) - base) / kSlice;
        const int ql = base / kSlice - qb;
        int cc[MAXW];
        double av[MAXW];
#pragma unroll
        for (int kk = 0; kk < MAXW; ++kk) {
          if (kk < width) {
            const int pos = base + kk * kSlice + lane;
            const int h = hc[ql + kk];
            const double u = hv[ql + kk];
            cc[kk] = h != kNonUniform ? (int)(row + h) : __ldg(A.sell_col + pos);
            av[kk] = isnan(u) ? __ldg(A.a + pos) : u;
          }
        }
        double acc = 0.0;
#pragma unroll
        for (int kk = 0; kk < MAXW; ++kk)
          if (kk < width) acc += av[kk] * __ldca(pg + cc[kk]);
        q[j] = acc;
        if (row < m) mu_p += sp[(sl - s0) * kSlice + lane] * acc;
      }
    }
    double mu, unused;
    reduce2(mu_p, 0.0, 1, mu, unused);
    if (!isfinite(mu) || mu == 0.0) {
      code = 2;
      break;
    }
    const double alpha = rho / mu;
    // ---- C: x += alpha p, r -= alpha q, z = D^-1 r; rz, rr
    double rz_p = 0.0, rr_p = 0.0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
      const int64_t sl = s0 + warp + 32 * j;
      if (sl < s1) {
        const int64_t row = sl * kSlice + lane;
        const int lr = (int)((sl - s0) * kSlice + lane);
        if (row < m) {
          xout[row * ld_x] += alpha * sp[lr];
          const double r = sr[lr] - alpha * q[j];
          sr[lr] = r;
          rz_p += r * (sd[lr] * r);
          rr_p += r * r;
        }
      }
    }
    double rz;
    reduce2(rz_p, rr_p, 0, rz, rr);
    ++its;
    if (!(rr > tol2)) {
      if (!isfinite(rr)) code = 2;
      break;
    }
    if (its >= maxit) {
      code = 1;
      break;
    }
    if (!isfinite(rz) || rz == 0.0) {
      code = 2;
      break;
    }
    beta = rz / rho;
    rho = rz;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->its[0] = its;
    st->rr[0] = rr;
    st->bb[0] = bb;
    st->tol2[0] = tol2;
    st->code[0] = code;
    st->active[0] = 0;
    st->done = 1;
    st->iter = its;
  }
}

// Launch the persistent solver when the block's rows fit; returns 1 when
// handled, 0 when the caller should use the two-kernel path.
template <int RMAX, int MAXW>
static int try_persist_rmax(irk_ctx* ctx, int64_t m, int64_t nslices, const MatView& A,
                            const double* rhs, int64_t ld_rhs, double* x, int64_t ld_x,
                            double rtol, double atol, int maxit, int* its_host, double* rel_host,
                            int* status) {
  const int G = ctx->num_sms;
  const int64_t spb = (nslices + G - 1) / G;
  if ((spb + 31) / 32 > RMAX) return 0;
  const size_t smem = (size_t)spb * kSlice * 3 * sizeof(double) +
                      (size_t)spb * MAXW * (sizeof(double) + sizeof(int)) + 64;
  static int configured_smem[64] = {0};  // per device, per instantiation
  int dev = ctx->device;
  if (smem > 200 * 1024) return 0;
  if ((size_t)configured_smem[dev & 63] < smem) {
    if (cudaFuncSetAttribute(k_pcg_persist<RMAX, MAXW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    configured_smem[dev & 63] = (int)smem;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_persist<RMAX, MAXW>, kPersistThreads,
                                                    smem) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  if (ensure_red(ctx, 4 * (size_t)G + 64) != IRK_OK) return 0;
  if (ensure_work(ctx, 1024 + ((m * sizeof(double) + 255) & ~(size_t)255)) != IRK_OK) return 0;
  if (ensure_pinned(ctx, sizeof(SysState<double>) + 64) != IRK_OK) return 0;
  static_assert(sizeof(SysState<double>) <= 1024, "state header");
  SysState<double>* st = reinterpret_cast<SysState<double>*>(ctx->work);
  double* pg = reinterpret_cast<double*>(ctx->work + 1024);
  double* part = ctx->red;
  double rtol2 = rtol * rtol, atol2 = atol * atol;
  int64_t mm = m, ns = nslices, sp = spb, lr = ld_rhs, lx = ld_x;
  int mi = maxit;
  MatView Av = A;
  const double* rh = rhs;
  double* xo = x;
  void* args[] = {&mm, &ns, &sp, &Av, &rh, &lr, &xo, &lx, &pg, &part, &rtol2, &atol2, &mi, &st};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k_pcg_persist<RMAX, MAXW>, dim3(G),
                                              dim3(kPersistThreads), args, smem, ctx->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  ctx->launches++;
  SysState<double>* h = reinterpret_cast<SysState<double>*>(ctx->pinned);
  if (cudaMemcpyAsync(h, st, sizeof(SysState<double>), cudaMemcpyDeviceToHost, ctx->stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    set_error("persistent pcg: %s", cudaGetErrorString(cudaGetLastError()));
    *status = IRK_ECUDA;
    return 1;
  }
  if (its_host) its_host[0] = h->its[0];
  if (rel_host) rel_host[0] = h->bb[0] > 0 ? sqrt(h->rr[0] / h->bb[0]) : 0.0;
  *status = IRK_OK;
  if (h->code[0] == 1) {
    set_error("pcg: iteration cap %d reached", maxit);
    *status = IRK_ENOCONV;
  } else if (h->code[0] == 2 && !(h->rr[0] <= h->tol2[0])) {
    set_error("pcg: breakdown (indefinite or singular block)");
    *status = IRK_ESINGULAR;
  }
  return 1;
}

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
  // single pre-combined block: one persistent cooperative launch per solve
  const bool persist_off = getenv("IRK_NO_PERSIST") != nullptr;
  if (nb == 1 && !Bm && !shift_dev && !rowmask_dev && alpha_host[0] == 1.0 && !persist_off) {
    int status = IRK_OK;
    const int mw = A->pat->maxw;
    if (mw <= 8 && try_persist_rmax<8, 8>(ctx, m, A->pat->nslices, V, rhs_dev, ld_rhs, x_dev,
                                          ld_x, rtol, atol, maxit, its_host, relres_host, &status))
      return status;
    if (mw > 8 && mw <= 16 &&
        try_persist_rmax<8, 16>(ctx, m, A->pat->nslices, V, rhs_dev, ld_rhs, x_dev, ld_x, rtol,
                                atol, maxit, its_host, relres_host, &status))
      return status;
  }
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
  IRK_REQUIRE(ld_x == nb, "irk_chebyshev: ld_x must equal nb");
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
  const size_t vec = ((size_t)m * nb * sizeof(double) + 255) & ~(size_t)255;
  IRK_TRY(ensure_work(ctx, 4 * vec + 4096));
  double* xa = reinterpret_cast<double*>(ctx->work);
  double* xb = reinterpret_cast<double*>(ctx->work + vec);
  double* ya = reinterpret_cast<double*>(ctx->work + 2 * vec);
  double* yb = reinterpret_cast<double*>(ctx->work + 3 * vec);
  double* rho_dev = reinterpret_cast<double*>(ctx->work + 4 * vec);
  IRK_CUDA(cudaMemsetAsync(xa, 0, (size_t)m * nb * sizeof(double), ctx->stream));
  IRK_CUDA(cudaMemsetAsync(ya, 0, (size_t)m * nb * sizeof(double), ctx->stream));
  // rho_0 = 1/sigma, rho_j = 1 / (2 sigma - rho_{j-1}), sigma = theta/delta
  double rho_prev[kMaxSys], rho_cur[kMaxSys];
  for (int k = 0; k < nb; ++k) rho_prev[k] = cp.delta[k] / cp.theta[k];
  const int G = grid_for(ctx, m, kBlock, 4);
  double *xin = xa, *xo = xb, *yin = ya, *yo = yb;
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
  IRK_TRY(ensure_work(ctx, 4 * vec + rv.size() * sizeof(double) + 256));
  xa = reinterpret_cast<double*>(ctx->work);
  xb = reinterpret_cast<double*>(ctx->work + vec);
  ya = reinterpret_cast<double*>(ctx->work + 2 * vec);
  yb = reinterpret_cast<double*>(ctx->work + 3 * vec);
  rho_dev = reinterpret_cast<double*>(ctx->work + 4 * vec);
  xin = xa, xo = xb, yin = ya, yo = yb;
  IRK_CUDA(cudaMemsetAsync(xa, 0, (size_t)m * nb * sizeof(double), ctx->stream));
  IRK_CUDA(cudaMemsetAsync(ya, 0, (size_t)m * nb * sizeof(double), ctx->stream));
  IRK_CUDA(cudaMemcpyAsync(rho_dev, rv.data(), rv.size() * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
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
  IRK_CUDA(cudaMemcpyAsync(x_dev, xin, (size_t)m * nb * sizeof(double), cudaMemcpyDeviceToDevice,
                           ctx->stream));
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  return IRK_OK;
}

}  // extern "C"
