// Real SPD diagonal blocks: batched Jacobi-PCG (irk_pcg) and
// Jacobi-Chebyshev (irk_chebyshev).  Kernels in irk_inner.cuh, plus the
// persistent single-block PCG below.
#include <cooperative_groups.h>

#include <algorithm>
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
constexpr int kPersistThreads = 768;  // 24 warps: 85 registers/thread at 1 CTA/SM
constexpr int kPersistWarps = kPersistThreads / 32;
constexpr int kMaxPersistBlocks = 256;
constexpr int kExplicitBase = INT_MIN + 1;  // hc value of explicit slot 0 (smem only)

struct WinLo {
  int lo[kMaxPersistBlocks];  // first column of each block's p window
};

// Per block: the p window [wlo, whi] covering every column its rows touch
// (own rows + halo), the residual r, D^-1 and the slot headers all live in
// shared memory; x and q = B p live in registers.  After the first barrier
// of an iteration each block copies only its halo of the freshly published
// p into the window, so the SpMV gathers are shared-memory reads.
// Debug bounds check (TRACE builds only): records the first violation.
#define PCHK(cond, cd)                                                        \
  do {                                                                        \
    if (TRACE && !(cond)) {                                                   \
      if (atomicCAS(&st->code[7], 0, (cd)) == 0) {                           \
        st->its[7] = blockIdx.x;                                              \
        st->its[6] = threadIdx.x;                                             \
      }                                                                       \
    }                                                                         \
  } while (0)

template <int RMAX, int MAXW, bool TRACE>
__global__ void __launch_bounds__(kPersistThreads, 1)
    k_pcg_persist(int m, int nslices, int spb, int wcap, int ecap, const WinLo win, MatView A,
                  const double* __restrict__ rhs, int ld_rhs, double* __restrict__ xout, int ld_x,
                  double* pg, double* __restrict__ part, double rtol2, double atol2, int maxit,
                  SysState<double>* st) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double smem[];
  __shared__ double wred[kPersistThreads / 32][2];
  __shared__ double bcast[2];
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int s0 = blockIdx.x * spb;
  const int s1 = min(nslices, s0 + spb);
  const int nsl = s1 > s0 ? s1 - s0 : 0;
  const int R0 = s0 * kSlice;
  const int nrow = nsl ? min(s1 * kSlice, m) - R0 : 0;  // rows owned by the block
  const int cap = spb * kSlice;
  const int off0 = R0 - win.lo[blockIdx.x];            // window index of the first own row
  // contiguous slice ranges per warp (a strided assignment resonates with
  // the grid-line period and piles the irregular boundary slices on a few
  // warps)
  const int spw = (nsl + kPersistWarps - 1) / kPersistWarps;
  const int wbase = warp * spw;
  const int qb = nsl ? __ldg(A.slice_ptr + s0) / kSlice : 0;
  const int qe = nsl ? __ldg(A.slice_ptr + s1) / kSlice : 0;
  const int nq = qe - qb;                   // slots of the block
  double* pw = smem;                        // p window (own rows + halo), wcap
  double* sr = pw + wcap;                   // r, cap
  double* hv = sr + cap;                    // slot value headers, nq
  double* ev = hv + nq;                     // explicit slot values, ecap*32
  float* sd = reinterpret_cast<float*>(ev + ecap * kSlice);  // D^-1 (fp32: a preconditioner)
  int* hc = reinterpret_cast<int*>(sd + cap);  // slot column headers / explicit ids, nq
  int* ec = hc + nq;                        // explicit slot window columns, ecap*32
  int* eq = ec + ecap * kSlice;             // slot id of each explicit slot, ecap
  int* spl = eq + ecap;                     // slice_ptr of the block, nsl + 1
  int* suni = spl + (nsl + 1);              // 1: every slot of the slice uniform
  __shared__ int nexp_sh;
  const int wlo = R0 - off0;
  PCHK(wlo >= 0, 1);
  PCHK(nq <= ecap * 0 + spb * MAXW, 2);
  for (int t = threadIdx.x; t < nq; t += blockDim.x) {
    hv[t] = __ldg(A.ua + qb + t);
    hc[t] = __ldg(A.colhdr + qb + t);
  }
  for (int t = threadIdx.x; t <= nsl; t += blockDim.x) spl[t] = __ldg(A.slice_ptr + s0 + t);
  for (int t = threadIdx.x; t < wcap; t += blockDim.x) pw[t] = 0.0;
  __syncthreads();
  // number the explicit (non-uniform column or value) slots of the block
  if (warp == 0) {
    int cnt = 0;
    for (int b0 = 0; b0 < nq; b0 += 32) {
      const int qq = b0 + lane;
      const bool ex = qq < nq && (hc[qq] == kNonUniform || isnan(hv[qq]));
      const unsigned bal = __ballot_sync(0xffffffffu, ex);
      if (ex) {
        const int e = cnt + __popc(bal & ((1u << lane) - 1u));
        PCHK(e < ecap, 3);
        if (e < ecap) {
          eq[e] = qq;
          hc[qq] = kExplicitBase + e;
        }
      }
      cnt += __popc(bal);
    }
    if (lane == 0) nexp_sh = min(cnt, ecap);
  }
  __syncthreads();
  // stage their columns (as window indices) and values
  for (int e = warp; e < nexp_sh; e += kPersistWarps) {
    const int P0 = (qb + eq[e]) * kSlice;  // SELL position of lane 0
    int lo = 0, hi = nsl;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (spl[mid] <= P0) lo = mid; else hi = mid;
    }
    const int lr2 = lo * kSlice + lane;
    if (lr2 < nrow) {
      ec[e * kSlice + lane] = __ldg(A.sell_col + P0 + lane) - wlo;
      ev[e * kSlice + lane] = __ldg(A.a + P0 + lane);
    } else {
      ec[e * kSlice + lane] = 0;
      ev[e * kSlice + lane] = 0.0;
    }
  }
  for (int t = threadIdx.x; t < nsl; t += blockDim.x) {
    int uni = 1;
    for (int qq = spl[t] / kSlice - qb; qq < spl[t + 1] / kSlice - qb; ++qq)
      if (hc[qq] >= kExplicitBase && hc[qq] < kExplicitBase + (1 << 24)) uni = 0;
    suni[t] = uni;
  }
  __syncthreads();

  auto reduce2 = [&](double a, double b, int slot, double& ra, double& rb) {
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
      wred[warp][0] = a;
      wred[warp][1] = b;
    }
    __syncthreads();
    if (warp == 0) {
      double ta = lane < kPersistWarps ? wred[lane][0] : 0.0;
      double tb = lane < kPersistWarps ? wred[lane][1] : 0.0;
      ta = warp_sum(ta);
      tb = warp_sum(tb);
      if (lane == 0) {
        part[slot * 2 * G + blockIdx.x] = ta;
        part[slot * 2 * G + G + blockIdx.x] = tb;
      }
    }
    grid.sync();
    if (warp == 0) {
      double ta = 0.0, tb = 0.0;
#pragma unroll
      for (int k = 0; k < kMaxPersistBlocks / 32; ++k) {
        const int q = lane + 32 * k;
        if (q < G) {
          ta += __ldcg(part + slot * 2 * G + q);
          tb += __ldcg(part + slot * 2 * G + G + q);
        }
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
  double q[RMAX], xr[RMAX];
#pragma unroll
  for (int j = 0; j < RMAX; ++j) {
    q[j] = xr[j] = 0.0;
    const int lr = (wbase + j) * kSlice + lane;
    if (j < spw && lr < nrow) {
      const int row = R0 + lr;
      const int dp = A.diag_pos[row];
      const float di = (float)(1.0 / (dp >= 0 ? A.a[dp] : 0.0));
      const double b = rhs[(int64_t)row * ld_rhs];
      sr[lr] = b;
      sd[lr] = di;
      rho_p += b * (di * b);
      bb_p += b * b;
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
  long long t_prev = 0;
  auto stamp = [&](int k) {
    if (TRACE && threadIdx.x == 0 && its >= 2 && its < 12) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (k > 0) part[(4 + k - 1) * G + blockIdx.x] += (double)(t - t_prev);
      t_prev = t;
    }
  };
  while (!done) {
    stamp(0);
    // ---- A: p = z + beta p  (z = D^-1 r), publish p
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
      const int lr = (wbase + j) * kSlice + lane;
      if (j < spw && lr < nrow) {
        PCHK(off0 + lr < wcap && lr < cap, 7);
        const double pj = (double)sd[lr] * sr[lr] + beta * pw[off0 + lr];
        pw[off0 + lr] = pj;
        __stcg(pg + R0 + lr, pj);
      }
    }
    stamp(1);
    grid.sync();
    stamp(2);
    // halo of the window from the published p
    if (nsl) {
      for (int c = threadIdx.x; c < off0; c += blockDim.x) pw[c] = __ldcg(pg + (R0 - off0) + c);
      const int wlo = R0 - off0;
      for (int c = off0 + nrow + threadIdx.x; c < wcap && wlo + c < m; c += blockDim.x)
        pw[c] = __ldcg(pg + wlo + c);
    }
    __syncthreads();
    stamp(3);
    // ---- B: q = B p, mu = p.q  (gathers from the shared-memory window)
    double mu_p = 0.0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
      const int sj = wbase + j;  // slice within the block
      const int lr = sj * kSlice + lane;
      if (j < spw && lr < nrow) {
        const int base = spl[sj];
        const int width = (spl[sj + 1] - base) / kSlice;
        const int ql = base / kSlice - qb;
        double acc = 0.0;
        if (suni[sj]) {
          // pure stencil: every lane applies the slice's (offset, value) pairs
          const double* pr = pw + off0 + lr;
#pragma unroll
          for (int kk = 0; kk < MAXW; ++kk)
            if (kk < width) {
              PCHK(off0 + lr + hc[ql + kk] >= 0 && off0 + lr + hc[ql + kk] < wcap, 4);
              PCHK(ql + kk >= 0 && ql + kk < nq, 5);
              acc += hv[ql + kk] * pr[hc[ql + kk]];
            }
        } else {
#pragma unroll
          for (int kk = 0; kk < MAXW; ++kk) {
            if (kk < width) {
              const int h = hc[ql + kk];
              int c;
              double av;
              if (h >= kExplicitBase && h < kExplicitBase + (1 << 24)) {
                const int e = (h - kExplicitBase) * kSlice + lane;
                c = ec[e];
                av = ev[e];
              } else {
                c = off0 + lr + h;
                av = hv[ql + kk];
              }
              PCHK(c >= 0 && c < wcap, 6);
              acc += av * pw[c];
            }
          }
        }
        q[j] = acc;
        mu_p += pw[off0 + lr] * acc;
      }
    }
    stamp(4);
    double mu, unused;
    reduce2(mu_p, 0.0, 1, mu, unused);
    stamp(5);
    if (!isfinite(mu) || mu == 0.0) {
      code = 2;
      break;
    }
    const double alpha = rho / mu;
    // ---- C: x += alpha p, r -= alpha q, z = D^-1 r; rz, rr
    double rz_p = 0.0, rr_p = 0.0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
      const int lr = (wbase + j) * kSlice + lane;
      if (j < spw && lr < nrow) {
        xr[j] += alpha * pw[off0 + lr];
        const double r = sr[lr] - alpha * q[j];
        sr[lr] = r;
        rz_p += r * ((double)sd[lr] * r);
        rr_p += r * r;
      }
    }
    stamp(6);
    double rz;
    reduce2(rz_p, rr_p, 0, rz, rr);
    stamp(7);
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
#pragma unroll
  for (int j = 0; j < RMAX; ++j) {
    const int lr = (wbase + j) * kSlice + lane;
    if (j < spw && lr < nrow) xout[(int64_t)(R0 + lr) * ld_x] = xr[j];
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

__global__ void k_explicit_per_slice(int64_t ns, const int* __restrict__ slice_ptr,
                                     const int* __restrict__ colhdr, const double* __restrict__ ua,
                                     int* __restrict__ cnt) {
  const int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sl >= ns) return;
  int c = 0;
  for (int q = slice_ptr[sl] / kSlice; q < slice_ptr[sl + 1] / kSlice; ++q)
    if (colhdr[q] == kNonUniform || isnan(ua[q])) ++c;
  cnt[sl] = c;
}

// Launch the persistent solver when the block's rows and p window fit in
// shared memory; returns 1 when handled, 0 when the caller should use the
// two-kernel path.
template <int RMAX, int MAXW, bool TRACE>
static int try_persist(irk_ctx* ctx, const Pattern* P, const MatView& A, const double* rhs,
                       int64_t ld_rhs, double* x, int64_t ld_x, double rtol, double atol,
                       int maxit, int* its_host, double* rel_host, int* status) {
  const char* gov = getenv("IRK_PERSIST_BLOCKS");
  const int G = gov ? std::min(atoi(gov), ctx->num_sms) : ctx->num_sms;
  const int64_t m = P->nrows, ns = P->nslices;
  if (G > kMaxPersistBlocks || ns == 0 || (int64_t)P->h_cmin.size() != ns) return 0;
  const int64_t spb = (ns + G - 1) / G;
  if ((spb + kPersistWarps - 1) / kPersistWarps > RMAX || P->maxw > MAXW) return 0;
  // per-block p windows and the largest one
  WinLo win{};
  int64_t wcap = 0;
  int64_t maxslots = 0;
  std::vector<int> sp;
  for (int b = 0; b < G; ++b) {
    const int64_t s0 = (int64_t)b * spb, s1 = std::min<int64_t>(ns, s0 + spb);
    if (s0 >= s1) {
      win.lo[b] = 0;
      continue;
    }
    int64_t lo = s0 * kSlice, hi = std::min<int64_t>(s1 * kSlice, m) - 1;
    for (int64_t q = s0; q < s1; ++q) {
      lo = std::min<int64_t>(lo, P->h_cmin[q]);
      hi = std::max<int64_t>(hi, P->h_cmax[q]);
    }
    win.lo[b] = (int)lo;
    wcap = std::max<int64_t>(wcap, hi - lo + 1);
    maxslots = std::max<int64_t>(maxslots, spb * P->maxw);
  }
  // explicit (non-uniform) slots per block, staged in shared memory
  int64_t ecap = 0;
  {
    int* d_cnt = nullptr;
    if (cudaMalloc(&d_cnt, ns * sizeof(int)) != cudaSuccess) return 0;
    k_explicit_per_slice<<<(unsigned)((ns + 255) / 256), 256, 0, ctx->stream>>>(
        ns, A.slice_ptr, A.colhdr, A.ua, d_cnt);
    std::vector<int> cnt(ns);
    cudaMemcpyAsync(cnt.data(), d_cnt, ns * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(d_cnt);
    ctx->launches++;
    for (int b = 0; b < G; ++b) {
      int64_t e = 0;
      for (int64_t q = (int64_t)b * spb; q < std::min<int64_t>(ns, (int64_t)(b + 1) * spb); ++q)
        e += cnt[q];
      ecap = std::max(ecap, e);
    }
  }
  const size_t smem = (size_t)(wcap + spb * kSlice + maxslots + ecap * kSlice) * sizeof(double) +
                      (size_t)spb * kSlice * sizeof(float) +
                      (size_t)(maxslots + ecap * kSlice + ecap + 2 * spb + 2) * sizeof(int) + 64;
  if (m >= INT32_MAX / 2 || ld_rhs >= INT32_MAX || ld_x >= INT32_MAX) return 0;
  if (smem > 220 * 1024) return 0;
  static size_t configured[64] = {0};
  const int dev = ctx->device & 63;
  if (configured[dev] < smem) {
    if (cudaFuncSetAttribute(k_pcg_persist<RMAX, MAXW, TRACE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(220 * 1024)) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    configured[dev] = 220 * 1024;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_persist<RMAX, MAXW, TRACE>, kPersistThreads,
                                                    smem) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  if (ensure_red(ctx, 12 * (size_t)G + 64) != IRK_OK) return 0;
  if (ensure_work(ctx, 1024 + ((m * sizeof(double) + 255) & ~(size_t)255)) != IRK_OK) return 0;
  if (ensure_pinned(ctx, sizeof(SysState<double>) + 64) != IRK_OK) return 0;
  if (TRACE) {
    cudaMemsetAsync(ctx->red, 0, 12 * (size_t)G * sizeof(double), ctx->stream);
    cudaMemsetAsync(ctx->work, 0, 1024, ctx->stream);
  }
  SysState<double>* st = reinterpret_cast<SysState<double>*>(ctx->work);
  double* pg = reinterpret_cast<double*>(ctx->work + 1024);
  double* part = ctx->red;
  double rtol2 = rtol * rtol, atol2 = atol * atol;
  int mm = (int)m, nsl = (int)ns, spbv = (int)spb, lr = (int)ld_rhs, lx = (int)ld_x;
  int mi = maxit, wc = (int)wcap, ecp = (int)ecap;
  MatView Av = A;
  const double* rh = rhs;
  double* xo = x;
  void* args[] = {&mm, &nsl, &spbv, &wc, &ecp, &win, &Av, &rh, &lr, &xo, &lx, &pg, &part,
                  &rtol2, &atol2, &mi, &st};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k_pcg_persist<RMAX, MAXW, TRACE>, dim3(G),
                                              dim3(kPersistThreads), args, smem, ctx->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  ctx->launches++;
  if (TRACE) {
    SysState<double> hs;
    cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    fprintf(stderr, "persist check: code %d block %d thread %d (m %ld spb %ld wcap %ld ecap %ld)\n",
            hs.code[7], hs.its[7], hs.its[6], (long)m, (long)spb, (long)wcap, (long)ecap);
    std::vector<double> d((size_t)7 * G);
    cudaMemcpyAsync(d.data(), ctx->red + 4 * G, d.size() * sizeof(double), cudaMemcpyDeviceToHost,
                    ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    const char* nm[7] = {"A", "sync1", "halo", "B", "red_mu", "C", "red_rz"};
    for (int k = 0; k < 7; ++k) {
      double mn = 1e30, mx = 0, sum = 0;
      int arg = 0, argmn = 0;
      for (int b = 0; b < G; ++b) {
        double v = d[(size_t)k * G + b] / 10.0;
        if (v < mn) argmn = b;
        mn = std::min(mn, v);
        if (v > mx) arg = b;
        mx = std::max(mx, v);
        sum += v;
      }
      std::vector<double> srt(d.begin() + (size_t)k * G, d.begin() + (size_t)(k + 1) * G);
      std::sort(srt.begin(), srt.end());
      fprintf(stderr, "persist trace %-7s ns/it: min %8.0f (block %3d) mean %8.0f p90 %8.0f max %8.0f (block %3d)\n",
              nm[k], mn, argmn, sum / G, srt[(size_t)(0.9 * (G - 1))] / 10.0, mx, arg);
    }
  }
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
  // The persistent solver is opt-in (IRK_PERSIST=1) until an intermittent
  // fault seen only after long mixed test sequences is understood.
  const bool persist_off =
      getenv("IRK_NO_PERSIST") != nullptr || getenv("IRK_PERSIST") == nullptr;
  if (nb == 1 && !Bm && !shift_dev && !rowmask_dev && alpha_host[0] == 1.0 && !persist_off) {
    int status = IRK_OK;
    const int mw = A->pat->maxw;
    const bool trace = getenv("IRK_PERSIST_TRACE") != nullptr;
    // smallest register budget that holds the rows of one warp
    const int64_t spb = (A->pat->nslices + ctx->num_sms - 1) / ctx->num_sms;
    const int64_t spw = (spb + kPersistWarps - 1) / kPersistWarps;
#define IRK_TRY_PERSIST(R, W, T)                                                             \
  if (try_persist<R, W, T>(ctx, A->pat, V, rhs_dev, ld_rhs, x_dev, ld_x, rtol, atol, maxit, \
                           its_host, relres_host, &status))                                 \
    return status;
    if (mw <= 8) {
      if (spw <= 4) {
        if (trace) { IRK_TRY_PERSIST(4, 8, true) } else { IRK_TRY_PERSIST(4, 8, false) }
      } else if (spw <= 8) {
        if (trace) { IRK_TRY_PERSIST(8, 8, true) } else { IRK_TRY_PERSIST(8, 8, false) }
      } else {
        if (trace) { IRK_TRY_PERSIST(10, 8, true) } else { IRK_TRY_PERSIST(10, 8, false) }
      }
    } else if (mw <= 16) {
      if (spw <= 4) {
        IRK_TRY_PERSIST(4, 16, false)
      } else if (spw <= 8) {
        IRK_TRY_PERSIST(8, 16, false)
      } else {
        IRK_TRY_PERSIST(10, 16, false)
      }
    }
#undef IRK_TRY_PERSIST
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
