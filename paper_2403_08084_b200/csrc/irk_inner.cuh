// Inner diagonal-block solvers (K4/K5): batched Jacobi-preconditioned CG on
// real SPD blocks and Jacobi-preconditioned COCG on complex-symmetric blocks
// (the 2x2 real-Schur pairs).  Templates shared by irk_inner_real.cu and
// irk_inner_cplx.cu.
//
// These replace the SuperLU factorisation + triangular solves the reference
// uses for every stage block (BlockFactorization / factorize_block,
// /root/reference/pkg/src/implicitrk/sparsela.py:149-191; the preconditioner
// calls block_factors[i].solve at precond.py:116).
//
// Design
//  * nb independent systems share one sparsity pattern and are stored
//    interleaved (row r, system k at r*nb + k): ONE pass over the pattern,
//    the value arrays and the vectors advances every system.
//  * Matrices are read through the slot-uniform SELL headers (colhdr/uval):
//    on structured-grid operators almost every slot is uniform, so the
//    matrix stream shrinks from 12-20 B/nnz to a few header bytes and the
//    iteration's working set (vectors) stays L2-resident.
//  * Each row's column indices and values are loaded up front (MAXW-wide
//    unrolled), then the gathers are issued: one dependency level per row
//    instead of one per entry.
//  * Loop control (convergence, breakdown, iteration cap) lives in device
//    memory; an iteration is two kernels (SpMV fused with the direction
//    update p = z + beta p; x/r/z update) with deterministic last-block
//    reductions, and the host polls a status block once per chunk.
//  * Flagged rows are identity rows; the caller passes matrices whose
//    flagged columns are already eliminated (irk_mat_constrain).
#pragma once

#include <algorithm>
#include <cstdlib>
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
struct alignas(16) SysState {
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
  int fresh;  // 1: written by the init kernel, no iteration decided yet
  int skip;   // external preconditioner: this iteration's z is not needed
};

struct MatView {
  const int* slice_ptr;
  const int* sell_col;
  const int* colhdr;
  const int* diag_pos;
  const double* a;   // values of A (SELL order)
  const double* ua;  // slot-uniform headers of A
  const double* b;   // values of Bm (or nullptr)
  const double* ub;
  int ellw;          // > 0: ELL-32 (slice base = 32 * ellw * slice)
  int sw;            // > 0: stencil-aligned ELL pattern with offsets sd[0..sw)
  int sd[16];
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

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ cplx ld_cg(const cplx* p) {
  const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
  return {v.x, v.y};
}

// Deterministic reduction of per-block partials part[k*G + b] -> out[k]
// by the whole (last) block: every thread loads its <= 4 partials per
// system at once (one L2 round trip), then a fixed-order block reduction.
// Must be called by all threads of the block (G <= 4 * kBlock).
template <typename T, int NB>
__device__ __forceinline__ void reduce_partials(const T* part, int G, T* out) {
  __shared__ T pred[kBlock / 32][NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T v[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) v[k] = s_zero(T{});
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int b = threadIdx.x + c * kBlock;
    if (b < G) {
#pragma unroll
      for (int k = 0; k < NB; ++k) v[k] = s_add(v[k], ld_cg(part + (int64_t)k * G + b));
    }
  }
#pragma unroll
  for (int k = 0; k < NB; ++k) v[k] = s_wsum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NB; ++k) pred[warp][k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < NB) {
    T t = s_zero(T{});
    for (int w = 0; w < kBlock / 32; ++w) t = s_add(t, pred[w][threadIdx.x]);
    out[threadIdx.x] = t;
  }
  __syncthreads();
}


// Three reductions at once (one L2 round trip, one barrier pair): the mu
// and rho partials (T) and the ||r||^2 partials (double) of the previous
// kernels.  Same fixed summation order as reduce_partials.
template <typename T, int NB>
__device__ __forceinline__ void reduce_partials3(const T* pa, const T* pb, const double* pc,
                                                 int G, T* oa, T* ob, double* oc) {
  __shared__ T ra[kBlock / 32][NB], rb[kBlock / 32][NB];
  __shared__ double rc[kBlock / 32][NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T va[NB], vb[NB];
  double vc[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    va[k] = vb[k] = s_zero(T{});
    vc[k] = 0.0;
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int b = threadIdx.x + c * kBlock;
    if (b < G) {
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        va[k] = s_add(va[k], ld_cg(pa + (int64_t)k * G + b));
        vb[k] = s_add(vb[k], ld_cg(pb + (int64_t)k * G + b));
        vc[k] += __ldcg(pc + (int64_t)k * G + b);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    va[k] = s_wsum(va[k]);
    vb[k] = s_wsum(vb[k]);
    vc[k] = warp_sum(vc[k]);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      ra[warp][k] = va[k];
      rb[warp][k] = vb[k];
      rc[warp][k] = vc[k];
    }
  }
  __syncthreads();
  if (threadIdx.x < NB) {
    T ta = s_zero(T{}), tb = s_zero(T{});
    double tc = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) {
      ta = s_add(ta, ra[w][threadIdx.x]);
      tb = s_add(tb, rb[w][threadIdx.x]);
      tc += rc[w][threadIdx.x];
    }
    oa[threadIdx.x] = ta;
    ob[threadIdx.x] = tb;
    oc[threadIdx.x] = tc;
  }
  __syncthreads();
}

template <typename T, int NB>
__device__ __forceinline__ void block_reduce_store(T (&v)[NB], T* part) {
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
__device__ __forceinline__ void block_reduce_store_d(double (&v)[NB], double* part) {
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

// ------------------------------------------------------------------ init
// x = 0, r = b, z = D^-1 r, p_old = 0; rho = r^T z, bb = ||b||^2.
template <typename T, int NB, bool HASB>
__global__ void __launch_bounds__(kBlock)
    k_cg_init(int64_t m, MatView A, const SysParams<T> P, const double* __restrict__ shift,
              const uint8_t* __restrict__ mask, const T* __restrict__ rhs, int64_t ld_rhs,
              T* __restrict__ x, T* __restrict__ r, T* __restrict__ z, T* __restrict__ pold,
              T* __restrict__ dinv, double rtol2, double atol2, SysState<T>* st,
              double* __restrict__ part, unsigned int* counter) {
  IRK_PDL_ENTER();
  T rho[NB];
  double bb[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    rho[k] = s_zero(T{});
    bb[k] = 0.0;
  }
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
    bool mr = mask && mask[row];
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
  block_reduce_store<T, NB>(rho, pr);
  block_reduce_store_d<NB>(bb, pb);
  if (last_block_inner(counter)) {
    __shared__ T srho[NB];
    __shared__ double sbb[NB];
    reduce_partials<T, NB>(pr, G, srho);
    reduce_partials<double, NB>(pb, G, sbb);
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
      st->fresh = 1;
    }
  }
}

// Init of a solve with an external preconditioner (one system): reads the
// strided right-hand side directly (launched eagerly, so no staging copy),
// x = 0, r = b, p_old = 0, bb = ||b||^2; the preconditioner forms z and
// rho afterwards (rho = 0 here).  Last block initialises the state.
template <typename T>
__global__ void __launch_bounds__(kBlock)
    k_cg_init_ext(int64_t m, const T* __restrict__ rhs, int64_t ld_rhs, T* __restrict__ x,
                  T* __restrict__ r, T* __restrict__ pold, double rtol2, double atol2,
                  SysState<T>* st, double* __restrict__ part, unsigned int* counter) {
  IRK_PDL_ENTER();
  double bb = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
    const T b = rhs[row * ld_rhs];
    x[row] = s_zero(T{});
    r[row] = b;
    pold[row] = s_zero(T{});
    bb += s_abs2(b);
  }
  double bbs[1] = {bb};
  block_reduce_store_d<1>(bbs, part);
  if (last_block_inner(counter)) {
    __shared__ double sbb[1];
    reduce_partials<double, 1>(part, gridDim.x, sbb);
    if (threadIdx.x == 0) {
      const double tol2 = fmax(rtol2 * sbb[0], atol2);
      st->rho[0] = s_zero(T{});
      st->bb[0] = sbb[0];
      st->rr[0] = sbb[0];
      st->tol2[0] = tol2;
      st->beta[0] = s_zero(T{});
      st->alpha[0] = s_zero(T{});
      st->its[0] = 0;
      st->code[0] = 0;
      const int act = (sbb[0] > tol2) ? 1 : 0;
      st->active[0] = act;
      st->done = act ? 0 : 1;
      st->iter = 0;
      st->fresh = 1;
    }
  }
}

// --------------------------------------------- tail-free iteration control
// Iteration k is two kernels, A_k (SpMV + direction) and B_k (update), with
// parity c = k & 1.  Neither kernel ends in a last-block reduction: each
// writes per-block partials, and every block of the NEXT kernel reduces
// them redundantly (same fixed order in every block, so all blocks take
// bitwise-identical decisions).  The loop state is double-buffered:
// A_k reads st[c^1] (written by A_{k-1}, or by the init kernel for k = 0),
// applies the convergence / breakdown / cap decisions of iteration k-1 and
// block 0 writes the result to st[c]; B_k reads st[c].  A finished state is
// propagated by every later A (block 0 copies it forward).
template <typename T, int NB>
struct CgPart {
  T* mu;
  T* rz;
  double* rr;
};

template <typename T, int NB>
__host__ __device__ __forceinline__ size_t cg_part_doubles(int G) {
  // rounded to 256 B so every buffer (complex ones included) stays aligned
  return ((size_t)G * NB * (2 * sizeof(T) / 8 + 1) + 31) & ~(size_t)31;
}

template <typename T, int NB>
__host__ __device__ __forceinline__ CgPart<T, NB> cg_part(double* red, int G, int c) {
  double* b = red + c * cg_part_doubles<T, NB>(G);
  T* t = reinterpret_cast<T*>(b);
  return {t, t + (size_t)G * NB, b + 2 * (size_t)G * NB * (sizeof(T) / 8)};
}

template <typename T>
__device__ __forceinline__ void state_copy(SysState<T>* dst, const SysState<T>* src) {
  constexpr int nw = sizeof(SysState<T>) / 4;
  for (int i = threadIdx.x; i < nw; i += blockDim.x)
    reinterpret_cast<int*>(dst)[i] = __ldcg(reinterpret_cast<const int*>(src) + i);
}

// Prologue of A_k: returns true when the solve is finished (all threads).
// Sum of n partials (any n) in a fixed order, all blocks alike.
__device__ __forceinline__ double reduce_partials_n(const double* part, int n) {
  __shared__ double pr[kBlock / 32];
  __shared__ double res;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v = 0.0;
  for (int b = threadIdx.x; b < n; b += kBlock) v += __ldcg(part + b);
  v = warp_sum(v);
  if (lane == 0) pr[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) t += pr[w];
    res = t;
  }
  __syncthreads();
  return res;
}

// ext_rz / n_ext: r.z partials written by a fused external preconditioner
// (its last kernel, n_ext blocks) replace the rz partials; the fresh state
// then takes rho from them (no separate rho kernel after the init).
template <typename T, int NB>
__device__ __forceinline__ bool cg_enter_a(const SysState<T>* sin, SysState<T>* sout,
                                           double* red, int c, int maxit,
                                           T (&beta)[NB], bool (&act)[NB],
                                           const double* ext_rz = nullptr, int n_ext = 0,
                                           int G_loop = 0) {
  __shared__ SysState<T> S;
  __shared__ T smu[NB], srz[NB];
  __shared__ double srr[NB];
  // G_loop: the loop kernels' grid when called from another grid (k_cg_settle)
  const int G = G_loop > 0 ? G_loop : (int)gridDim.x;
  state_copy(&S, sin);
  {
    // issued together with the state loads (unused when the state is fresh
    // from the init kernel); reduce_partials3 synchronises
    const CgPart<T, NB> pin = cg_part<T, NB>(red, G, c ^ 1);
    reduce_partials3<T, NB>(pin.mu, pin.rz, pin.rr, G, smu, srz, srr);
  }
  if constexpr (NB == 1 && sizeof(T) == 8) {
    if (ext_rz) {
      const double v = reduce_partials_n(ext_rz, n_ext);
      if (threadIdx.x == 0) {
        reinterpret_cast<double*>(srz)[0] = v;
        if (S.fresh && !S.done && S.active[0]) {
          if (!isfinite(v) || v == 0.0) {  // as k_cg_rho_init
            S.active[0] = 0;
            S.code[0] = 2;
            S.done = 1;
          } else {
            reinterpret_cast<double*>(S.rho)[0] = v;
          }
        }
      }
      __syncthreads();
    }
  }
  const bool first = S.fresh != 0;
  if (S.done) {
    if (blockIdx.x == 0) {
      constexpr int nw = sizeof(SysState<T>) / 4;
      for (int i = threadIdx.x; i < nw; i += blockDim.x)
        reinterpret_cast<int*>(sout)[i] = reinterpret_cast<const int*>(&S)[i];
    }
    return true;
  }
  if (!first) {
    if (threadIdx.x == 0) {
      int any = 0;
      for (int k = 0; k < NB; ++k) {
        if (!S.active[k]) continue;
        const T muk = smu[k];
        if (!s_finite(muk) || s_isnull(muk)) {  // B_{k-1} skipped the update
          S.active[k] = 0;
          S.code[k] = 2;
          continue;
        }
        S.mu[k] = muk;
        S.its[k] += 1;
        S.rr[k] = srr[k];
        if (!(srr[k] > S.tol2[k])) {
          S.active[k] = 0;  // converged (or NaN residual: flagged below)
          if (!isfinite(srr[k])) S.code[k] = 2;
        } else if (S.its[k] >= maxit) {
          S.active[k] = 0;
          S.code[k] = 1;
        } else if (!s_finite(srz[k]) || s_isnull(srz[k])) {
          S.active[k] = 0;
          S.code[k] = 2;
        } else {
          S.beta[k] = s_div(srz[k], S.rho[k]);
          S.rho[k] = srz[k];
        }
        any |= S.active[k];
      }
      S.iter += 1;
      S.done = any ? 0 : 1;
    }
  }
  if (threadIdx.x == 0) S.fresh = 0;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    beta[k] = S.beta[k];
    act[k] = S.active[k] != 0;
  }
  const bool done = S.done != 0;
  if (blockIdx.x == 0) {
    constexpr int nw = sizeof(SysState<T>) / 4;
    for (int i = threadIdx.x; i < nw; i += blockDim.x)
      reinterpret_cast<int*>(sout)[i] = reinterpret_cast<const int*>(&S)[i];
  }
  __syncthreads();
  return done;
}

// Loop condition with early settlement (external-preconditioner solves, at
// a parity-0 boundary: after the straight-line prefix iterations and after
// every WHILE pass).  When the preconditioner application of the last
// iteration was skipped (sin->skip: the next A kernel will end the solve),
// this one-CTA kernel takes that A kernel's state transition itself
// (cg_enter_a over the loop grid's partials: sin -> sout, idempotent) and
// clears the loop condition, so a finished solve does not run one more
// WHILE pass of no-op kernels.
template <typename T, int NB>
__global__ void __launch_bounds__(kBlock)
    k_cg_settle(cudaGraphConditionalHandle h, const SysState<T>* sin, SysState<T>* sout,
                double* red, int G, int maxit, const double* ext_rz, int n_ext) {
  IRK_PDL_ENTER();
  __shared__ int sflag[2];
  if (threadIdx.x == 0) {
    sflag[0] = __ldcg(&sin->done) || __ldcg(&sout->done);
    sflag[1] = __ldcg(&sin->skip);
  }
  __syncthreads();
  bool finished = sflag[0] != 0;
  if (!finished && sflag[1]) {
    T beta[NB];
    bool act[NB];
    finished = cg_enter_a<T, NB>(sin, sout, red, 0, maxit, beta, act, ext_rz, n_ext, G);
  }
  if (threadIdx.x == 0) cudaGraphSetConditional(h, finished ? 0u : 1u);
}

// Prologue of B_k: alpha = rho / mu from A_k's partials; true when finished.
template <typename T, int NB>
__device__ __forceinline__ bool cg_enter_b(const SysState<T>* st, double* red, int c,
                                           T (&alpha)[NB], bool (&act)[NB]) {
  __shared__ T smu[NB], srho[NB];
  __shared__ int sact[NB], sdone;
  if (threadIdx.x < NB) {
    srho[threadIdx.x] = ld_cg(&st->rho[threadIdx.x]);
    sact[threadIdx.x] = __ldcg(&st->active[threadIdx.x]);
  }
  if (threadIdx.x == 0) sdone = __ldcg(&st->done);
  reduce_partials<T, NB>(cg_part<T, NB>(red, gridDim.x, c).mu, gridDim.x, smu);
  if (sdone) return true;
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    const T muk = smu[k];
    act[k] = sact[k] && s_finite(muk) && !s_isnull(muk);
    alpha[k] = act[k] ? s_div(srho[k], muk) : s_zero(T{});
  }
  return false;
}

// ------------------------------------------------- SpMV + direction update
// p_new = z + beta p_old (computed on the fly for every gathered column),
// q = B p_new, mu = p_new^T q;  alpha = rho / mu by the last block.
template <typename T, int NB, bool HASB, int MAXW>
__global__ void __launch_bounds__(kBlock, 4)
    k_cg_spmv(int64_t m, MatView A, const SysParams<T> P, const double* __restrict__ shift,
              const uint8_t* __restrict__ mask, const T* __restrict__ z,
              const T* __restrict__ pold, T* __restrict__ pnew, T* __restrict__ q,
              const SysState<T>* sin, SysState<T>* sout, double* red, int c, int maxit,
              const double* ext_rz, int n_ext) {
  IRK_PDL_ENTER();
  T beta[NB];
  bool act[NB];
  if (cg_enter_a<T, NB>(sin, sout, red, c, maxit, beta, act, ext_rz, n_ext)) return;
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
    if (mask && mask[row]) {
#pragma unroll
      for (int k = 0; k < NB; ++k) acc[k] = pr[k];
    } else {
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
      if (MAXW > 0) {
        int cc[MAXW > 0 ? MAXW : 1];
        double av[MAXW > 0 ? MAXW : 1], bv[MAXW > 0 ? MAXW : 1];
#pragma unroll
        for (int kk = 0; kk < MAXW; ++kk) {
          if (kk < width) {
            const int pos = base + kk * kSlice + lane;
            cc[kk] = sell_col_at(A.colhdr, A.sell_col, q0 + kk, pos, row);
            av[kk] = sell_val_at(A.ua, A.a, q0 + kk, pos);
            bv[kk] = HASB ? sell_val_at(A.ub, A.b, q0 + kk, pos) : 0.0;
          }
        }
#pragma unroll
        for (int kk = 0; kk < MAXW; ++kk) {
          if (kk < width) {
#pragma unroll
            for (int k = 0; k < NB; ++k) {
              const int64_t qc = (int64_t)cc[kk] * NB + k;
              T pc = s_add(z[qc], s_mul(beta[k], pold[qc]));
              acc[k] = s_add(acc[k], s_mul(s_coef(P.alpha[k], P.beta[k], av[kk], bv[kk]), pc));
            }
          }
        }
      } else {
        for (int kk = 0; kk < width; ++kk) {
          const int pos = base + kk * kSlice + lane;
          const int c = sell_col_at(A.colhdr, A.sell_col, q0 + kk, pos, row);
          const double av = sell_val_at(A.ua, A.a, q0 + kk, pos);
          const double bv = HASB ? sell_val_at(A.ub, A.b, q0 + kk, pos) : 0.0;
#pragma unroll
          for (int k = 0; k < NB; ++k) {
            const int64_t qc = (int64_t)c * NB + k;
            T pc = s_add(z[qc], s_mul(beta[k], pold[qc]));
            acc[k] = s_add(acc[k], s_mul(s_coef(P.alpha[k], P.beta[k], av, bv), pc));
          }
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
      const int64_t qi = row * NB + k;
      pnew[qi] = pr[k];
      q[qi] = acc[k];
      mu[k] = s_add(mu[k], s_mul(pr[k], acc[k]));
    }
  }
  block_reduce_store<T, NB>(mu, cg_part<T, NB>(red, gridDim.x, c).mu);
}

// Stencil variant of k_cg_spmv (one real system, stencil-aligned ELL
// pattern of width W, e.g. the P1/Q1 grid operators).  The gathers of
// p = z + beta p_old at the W stencil offsets are issued immediately, in
// parallel with the slice's slot headers (lane k loads slot k once per
// slice); z and p_old carry `pad` >= max |offset| readable elements on both
// sides, so speculative gathers of boundary rows stay inside the
// allocation.  A slice whose headers all match the stencil with uniform
// values (the interior) then needs one shuffle + FMA per entry; any other
// slice is recomputed through the SELL arrays.
template <int W, bool HASB>
__global__ void __launch_bounds__(kBlock, 4)
    k_cg_spmv_st(int m, MatView A, const SysParams<double> P, const double* __restrict__ shift,
                 const uint8_t* __restrict__ mask, const double* __restrict__ z,
                 const double* __restrict__ pold, double* __restrict__ pnew,
                 double* __restrict__ q, const SysState<double>* sin, SysState<double>* sout,
                 double* red, int cpar, int maxit, const double* ext_rz, int n_ext) {
  IRK_PDL_ENTER();
  double betas[1];
  bool acts[1];
  if (cg_enter_a<double, 1>(sin, sout, red, cpar, maxit, betas, acts, ext_rz, n_ext)) return;
  const double beta = betas[0];
  const bool act = acts[0];
  const int lane = threadIdx.x & 31;
  const int nsl = (m + kSlice - 1) / kSlice;
  const int wstride = gridDim.x * (blockDim.x / 32);
  const double al = P.alpha[0], be = P.beta[0];
  double mu = 0.0;
  for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) / 32; sl < nsl; sl += wstride) {
    const int row = sl * kSlice + lane;
    const bool valid = row < m;
    const int q0 = sl * W;
    const bool hl = lane < W;
    const int hd = hl ? __ldg(A.colhdr + q0 + lane) : 0;
    const double ha = hl ? __ldg(A.ua + q0 + lane) : 0.0;
    const double hb = (HASB && hl) ? __ldg(A.ub + q0 + lane) : 0.0;
    const double pr = z[row] + beta * pold[row];
    const bool flagged = valid && mask && mask[row];
    double ps[W];
#pragma unroll
    for (int kk = 0; kk < W; ++kk) {
      const int c = row + A.sd[kk];
      ps[kk] = z[c] + beta * pold[c];
    }
    const bool ok = __all_sync(0xffffffffu, !hl || (hd == A.sd[lane < W ? lane : 0] &&
                                                    !isnan(ha) && !(HASB && isnan(hb))));
    double acc = 0.0;
    if (ok) {
      const double hc = HASB ? al * ha + be * hb : al * ha;
#pragma unroll
      for (int kk = 0; kk < W; ++kk) acc += __shfl_sync(0xffffffffu, hc, kk) * ps[kk];
    } else if (valid) {
      const int base = sl * kSlice * W;
#pragma unroll
      for (int kk = 0; kk < W; ++kk) {
        const int pos = base + kk * kSlice + lane;
        const int c = sell_col_at(A.colhdr, A.sell_col, q0 + kk, pos, row);
        const double av = sell_val_at(A.ua, A.a, q0 + kk, pos);
        const double bv = HASB ? sell_val_at(A.ub, A.b, q0 + kk, pos) : 0.0;
        acc += (HASB ? al * av + be * bv : al * av) * (z[c] + beta * pold[c]);
      }
    }
    if (shift && valid) acc += shift[row] * pr;
    if (flagged) acc = pr;
    if (valid && act) {
      pnew[row] = pr;
      q[row] = acc;
      mu += pr * acc;
    }
  }
  double mus[1] = {mu};
  block_reduce_store<double, 1>(mus, cg_part<double, 1>(red, gridDim.x, cpar).mu);
}

__device__ __forceinline__ double ldv(const double* p) { return __ldg(p); }
__device__ __forceinline__ cplx ldv(const cplx* p) {
  const double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return {v.x, v.y};
}

// Stencil variant of k_cg_spmv for NB batched systems and complex
// scalars (the block-Jacobi surrogate blocks, the Schur-pair COCG): one warp
// per SELL slice; the slot headers are loaded once per slice (lane k holds
// slot k) and checked with one warp vote while the gathers at the stencil
// offsets are already in flight (z and p_old carry a readable halo of `pad`
// rows); a plain stencil slice then forms each system's coefficient from
// the broadcast headers.  Other slices take the SELL row path.
template <typename T, int NB, int W, bool HASB>
__global__ void __launch_bounds__(kBlock, 2)
    k_cg_spmv_stn(int m, MatView A, const SysParams<T> P, const double* __restrict__ shift,
                  const uint8_t* __restrict__ mask, const T* __restrict__ z,
                  const T* __restrict__ pold, T* __restrict__ pnew, T* __restrict__ q,
                  const SysState<T>* sin, SysState<T>* sout, double* red, int cpar, int maxit) {
  IRK_PDL_ENTER();
  T beta[NB];
  bool act[NB];
  if (cg_enter_a<T, NB>(sin, sout, red, cpar, maxit, beta, act)) return;
  const int lane = threadIdx.x & 31;
  const int nsl = (m + kSlice - 1) / kSlice;
  const int wstride = gridDim.x * (blockDim.x / 32);
  T mu[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) mu[k] = s_zero(T{});
  for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) / 32; sl < nsl; sl += wstride) {
    const int row = sl * kSlice + lane;
    const bool valid = row < m;
    const int q0 = sl * W;
    const bool hl = lane < W;
    const int hd = hl ? __ldg(A.colhdr + q0 + lane) : 0;
    const double ha = hl ? __ldg(A.ua + q0 + lane) : 0.0;
    const double hb = (HASB && hl) ? __ldg(A.ub + q0 + lane) : 0.0;
    T pr[NB], acc[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const int64_t qi = (int64_t)row * NB + k;
      pr[k] = s_add(ldv(z + qi), s_mul(beta[k], ldv(pold + qi)));
      acc[k] = s_zero(T{});
    }
    const bool ok = __all_sync(0xffffffffu, !hl || (hd == A.sd[lane < W ? lane : 0] &&
                                                    !isnan(ha) && !(HASB && isnan(hb))));
    if (ok) {
#pragma unroll
      for (int kk = 0; kk < W; ++kk) {
        const double a = __shfl_sync(0xffffffffu, ha, kk);
        const double b = HASB ? __shfl_sync(0xffffffffu, hb, kk) : 0.0;
        const int64_t qc = (int64_t)(row + A.sd[kk]) * NB;
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          const T pc = s_add(ldv(z + qc + k), s_mul(beta[k], ldv(pold + qc + k)));
          acc[k] = s_add(acc[k], s_mul(s_coef(P.alpha[k], P.beta[k], a, b), pc));
        }
      }
    } else if (valid) {
      const int base = sl * kSlice * W;
#pragma unroll
      for (int kk = 0; kk < W; ++kk) {
        const int pos = base + kk * kSlice + lane;
        const int c = sell_col_at(A.colhdr, A.sell_col, q0 + kk, pos, row);
        const double av = sell_val_at(A.ua, A.a, q0 + kk, pos);
        const double bv = HASB ? sell_val_at(A.ub, A.b, q0 + kk, pos) : 0.0;
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          const int64_t qc = (int64_t)c * NB + k;
          const T pc = s_add(ldv(z + qc), s_mul(beta[k], ldv(pold + qc)));
          acc[k] = s_add(acc[k], s_mul(s_coef(P.alpha[k], P.beta[k], av, bv), pc));
        }
      }
    }
    if (!valid) continue;
    const bool flagged = mask && mask[row];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      if (shift) acc[k] = s_add(acc[k], s_mul(s_real<T>(shift[(int64_t)row * NB + k]), pr[k]));
      if (flagged) acc[k] = pr[k];
      if (!act[k]) continue;
      const int64_t qi = (int64_t)row * NB + k;
      pnew[qi] = pr[k];
      q[qi] = acc[k];
      mu[k] = s_add(mu[k], s_mul(pr[k], acc[k]));
    }
  }
  block_reduce_store<T, NB>(mu, cg_part<T, NB>(red, gridDim.x, cpar).mu);
}

// x += alpha p, r -= alpha q, z = D^-1 r; partials of rho' = r^T z and
// rr = ||r||^2 (the next A kernel decides convergence / cap / beta).
// EXTZ: an external preconditioner forms z (and the r.z partials) after
// this kernel; only x, r and ||r||^2 are updated here.
template <typename T, int NB, bool EXTZ = false>
__global__ void __launch_bounds__(kBlock)
    k_cg_update(int64_t m, const T* __restrict__ p, const T* __restrict__ q,
                const T* __restrict__ dinv, T* __restrict__ x, T* __restrict__ r,
                T* __restrict__ z, const SysState<T>* st, double* red, int c) {
  IRK_PDL_ENTER();
  T alpha[NB];
  bool act[NB];
  if (cg_enter_b<T, NB>(st, red, c, alpha, act)) return;
  T rho[NB];
  double rr[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    rho[k] = s_zero(T{});
    rr[k] = 0.0;
  }
  // small NB: U rows per thread per pass with every load issued before the
  // stores (memory-level parallelism); large NB: one row, system by system
  constexpr int NW = NB * (int)(sizeof(T) / 8);
  constexpr int U = NW <= 1 ? 2 : 1;
  const int64_t TT = (int64_t)gridDim.x * blockDim.x;
  if constexpr (NW <= 2) {
    for (int64_t row0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row0 < m;
         row0 += U * TT) {
      T pk[U][NB], qk[U][NB], dk[U][NB], xk[U][NB], rk[U][NB];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t row = row0 + u * TT;
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          if (row < m && act[k]) {
            const int64_t qi = row * NB + k;
            pk[u][k] = p[qi];
            qk[u][k] = q[qi];
            dk[u][k] = EXTZ ? s_zero(T{}) : dinv[qi];
            xk[u][k] = x[qi];
            rk[u][k] = r[qi];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t row = row0 + u * TT;
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          if (row < m && act[k]) {
            const int64_t qi = row * NB + k;
            x[qi] = s_add(xk[u][k], s_mul(alpha[k], pk[u][k]));
            T rn = s_sub(rk[u][k], s_mul(alpha[k], qk[u][k]));
            r[qi] = rn;
            if (!EXTZ) {
              T zn = s_mul(dk[u][k], rn);
              z[qi] = zn;
              rho[k] = s_add(rho[k], s_mul(rn, zn));
            }
            rr[k] += s_abs2(rn);
          }
        }
      }
    }
  } else {
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m; row += TT) {
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        if (!act[k]) continue;
        const int64_t qi = row * NB + k;
        T pk = p[qi];
        x[qi] = s_add(x[qi], s_mul(alpha[k], pk));
        T rk = s_sub(r[qi], s_mul(alpha[k], q[qi]));
        r[qi] = rk;
        if (!EXTZ) {
          T zk = s_mul(dinv[qi], rk);
          z[qi] = zk;
          rho[k] = s_add(rho[k], s_mul(rk, zk));
        }
        rr[k] += s_abs2(rk);
      }
    }
  }
  const CgPart<T, NB> po = cg_part<T, NB>(red, gridDim.x, c);
  if (!EXTZ) block_reduce_store<T, NB>(rho, po.rz);
  block_reduce_store_d<NB>(rr, po.rr);
}

// r.z partials of iteration parity c after an external preconditioner
// (one system; the unconjugated bilinear form for complex COCG).  Same grid
// as the A/B kernels.
template <typename T>
__global__ void __launch_bounds__(kBlock)
    k_cg_dot_rz(int64_t m, const T* __restrict__ r, const T* __restrict__ z, double* red, int c,
                const int* skip) {
  IRK_PDL_ENTER();
  if (skip && *skip) return;
  T v = s_zero(T{});
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    v = s_add(v, s_mul(r[i], z[i]));
  T vs[1] = {v};
  block_reduce_store<T, 1>(vs, cg_part<T, 1>(red, gridDim.x, c).rz);
}

// After the init kernel: rho = r.z for an external preconditioner's z
// (last-block reduction, once per solve); breakdown ends the solve.
template <typename T>
__global__ void __launch_bounds__(kBlock)
    k_cg_rho_init(int64_t m, const T* __restrict__ r, const T* __restrict__ z, SysState<T>* st,
                  double* part, unsigned int* counter) {
  IRK_PDL_ENTER();
  T v = s_zero(T{});
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    v = s_add(v, s_mul(r[i], z[i]));
  T vs[1] = {v};
  T* pt = reinterpret_cast<T*>(part);
  block_reduce_store<T, 1>(vs, pt);
  if (last_block_inner(counter)) {
    __shared__ T srho[1];
    reduce_partials<T, 1>(pt, gridDim.x, srho);
    if (threadIdx.x == 0 && !st->done) {
      st->rho[0] = srho[0];
      if (st->active[0] && (!s_finite(srho[0]) || s_isnull(srho[0]))) {
        st->active[0] = 0;
        st->code[0] = 2;
        st->done = 1;
      }
    }
  }
}

// The skip predicate (shared by k_cg_skip and the fused preconditioners):
// the next A kernel will end the solve (converged, cap, finished).
template <typename T>
__device__ __forceinline__ bool cg_skip_pred(const SysState<T>* st, double rr, int maxit) {
  return __ldcg(&st->done) || !__ldcg(&st->active[0]) || !(rr > __ldcg(&st->tol2[0])) ||
         __ldcg(&st->its[0]) + 1 >= maxit;
}

// After the update kernel of an iteration with an external preconditioner:
// decide from the ||r||^2 partials (same reduction order as the next A
// kernel) whether that A kernel will end the solve (converged, cap,
// non-finite); then the preconditioner application and r.z are skipped.
template <typename T>
__global__ void __launch_bounds__(kBlock)
    k_cg_skip(SysState<T>* st, const double* red, int G, int c, int maxit) {
  IRK_PDL_ENTER();
  __shared__ double srr[1];
  reduce_partials<double, 1>(cg_part<T, 1>(const_cast<double*>(red), G, c).rr, G, srr);
  if (threadIdx.x == 0) st->skip = cg_skip_pred(st, srr[0], maxit);
}

// Loop condition of the graph-resident CG loop: continue while neither
// state buffer is finished.
template <typename T>
__global__ void k_cg_cond(cudaGraphConditionalHandle h, const SysState<T>* a,
                          const SysState<T>* b) {
  IRK_PDL_ENTER();
  if (threadIdx.x == 0 && blockIdx.x == 0)
    cudaGraphSetConditional(h, (__ldcg(&a->done) || __ldcg(&b->done)) ? 0u : 1u);
}

// Deferred status: the finished state's (max iterations, worst code,
// loop iteration count) of one solve into the context's solve log.
template <typename T>
__global__ void k_cg_log(const SysState<T>* a, const SysState<T>* b, int nb, int body_kernels,
                         int prefix, int settle, int* out) {
  IRK_PDL_ENTER();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const SysState<T>* f = (a->done != b->done) ? (a->done ? a : b) : (a->iter >= b->iter ? a : b);
  int its = 0, code = 0;
  for (int k = 0; k < nb; ++k) {
    its = max(its, f->its[k]);
    int c = f->code[k];
    if (c == 0 && f->active[k]) c = 1;
    if (c == 2 && f->rr[k] <= f->tol2[k]) c = 0;  // breakdown after convergence
    code = max(code, c);
  }
  out[0] = its;
  out[1] = code;
  // passes of the graph-resident loop: iterations in pairs after the prefix;
  // without the settling condition one more pass observes the finished state
  const int rest = max(f->iter - prefix, 0);
  out[2] = settle ? (rest + 1) / 2 : rest / 2 + 1;
  out[3] = body_kernels;
}

// External preconditioner z = P^-1 r for the real one-system CG (the
// geometric multigrid of irk_mg.cu): a fixed, graph-capturable kernel
// sequence on the given stream.
// Skip decision of a fused preconditioner application (what k_cg_skip
// decides): st == nullptr -> always apply (the init application).
struct SkipCtl {
  SysState<double>* st = nullptr;
  const double* rr = nullptr;  // ||r||^2 partials of the update kernel (G of them)
  int G = 0, maxit = 0;
};

struct CgPrec {
  uint64_t uid = 0;  // unique per instance (graph-cache key; addresses get reused)
  // stop: device flag; when nonzero at run time the kernels do nothing (the
  // solve finished inside a graph-resident loop)
  virtual int apply(irk_ctx* ctx, cudaStream_t s, const double* r, double* z,
                    const int* stop) = 0;
  // Fused variant (0 partials: not supported): the first kernel takes the
  // skip decision itself and publishes it in st->skip for the others; the
  // last kernel writes fused_rz_count() partials of r.z to rz_part.
  virtual int fused_rz_count() { return 0; }
  // CG iterations worth issuing straight-line with the init sequence (the
  // iterations a typical solve needs; < 0: the default, IRK_CG_PREFIX)
  virtual int prefix_iters() { return -1; }
  virtual int apply_fused(irk_ctx* ctx, cudaStream_t s, const double* r, double* z,
                          const SkipCtl& sk, double* rz_part) {
    return IRK_EINVAL;
  }
  virtual ~CgPrec() {}
};


template <typename T, int NB>
__global__ void k_cg_store(int64_t m, const T* __restrict__ x, T* __restrict__ out,
                           int64_t ld_out) {
  IRK_PDL_ENTER();
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < NB; ++k) out[row * ld_out + k] = x[row * NB + k];
  }
}

// ------------------------------------------------------------ host driver

template <typename T>
struct Workspace {
  SysState<T>* st;
  T *x, *r, *z, *p0, *p1, *q, *dinv;
  T* rb;        // right-hand side staged contiguously (graph-stable address)
  int64_t pad;  // readable elements before/after z, p0, p1 (stencil gathers)
};

// rb[row*NB + k] = rhs[row*ld + k]
template <typename T, int NB>
__global__ void k_cg_stage_rhs(int64_t m, const T* __restrict__ rhs, int64_t ld,
                               T* __restrict__ rb) {
  IRK_PDL_ENTER();
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < NB; ++k) rb[row * NB + k] = rhs[row * ld + k];
  }
}

// zero the `pad` elements before and after each of a, b, c (length len)
template <typename T>
__global__ void k_zero_halos(T* a, T* b, T* c, int64_t len, int64_t pad) {
  IRK_PDL_ENTER();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 6 * pad;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = i / (2 * pad), j = i % (2 * pad);
    T* base = w == 0 ? a : (w == 1 ? b : c);
    base[j < pad ? j - pad : len + (j - pad)] = s_zero(T{});
  }
}

// pad > 0: z, p0 and p1 get `pad` extra elements (zeroed) on both sides
template <typename T>
int carve(irk_ctx* ctx, int64_t m, int nb, Workspace<T>& w, int64_t pad = 0) {
  size_t vec = (size_t)m * nb * sizeof(T);
  vec = (vec + 255) & ~(size_t)255;
  size_t pb = ((size_t)pad * nb * sizeof(T) + 255) & ~(size_t)255;
  size_t head = (2 * sizeof(SysState<T>) + 255) & ~(size_t)255;  // st[0], st[1]
  IRK_TRY(ensure_work(ctx, head + 8 * vec + 6 * pb));
  char* b = ctx->work;
  w.st = reinterpret_cast<SysState<T>*>(b);
  b += head;
  w.pad = pad;
  w.rb = reinterpret_cast<T*>(b);
  b += vec;
  T** v[7] = {&w.x, &w.r, &w.q, &w.dinv, &w.z, &w.p0, &w.p1};
  for (int i = 0; i < 7; ++i) {
    if (i >= 4) b += pb;
    *v[i] = reinterpret_cast<T*>(b);
    b += vec;
    if (i >= 4) b += pb;
  }
  if (pad > 0) {
    const int64_t n = 6 * pad * nb;
    IRK_CUDA(launch(k_zero_halos<T>, (unsigned)std::min<int64_t>((n + kBlock - 1) / kBlock, 1024),
                    kBlock, 0, ctx->stream, w.z, w.p0, w.p1, m * nb, pad * nb));
    ctx->launches++;
  }
  return IRK_OK;
}

template <typename T, int NB, bool HASB, int MAXW>
int run_cg(irk_ctx* ctx, int64_t m, const MatView& A, const SysParams<T>& P, const double* shift,
           const uint8_t* mask, const T* rhs, int64_t ld_rhs, T* xout, int64_t ld_x, double rtol,
           double atol, int maxit, int* its_host, double* relres_host, CgPrec* prec = nullptr) {
  constexpr bool kExtOk = NB == 1;
  IRK_REQUIRE(!prec || kExtOk, "run_cg: external preconditioner needs one system");
  Workspace<T> w;
  int64_t pad = 0;
  if (A.sw > 0) {
    for (int k = 0; k < A.sw; ++k) pad = std::max<int64_t>(pad, std::abs(A.sd[k]));
    pad += kSlice;
  }
  IRK_TRY(carve<T>(ctx, m, NB, w, pad));
  const int G = grid_for(ctx, m, kBlock, 4);
  // a fused preconditioner writes its r.z partials (two parities) past the
  // loop and init partials
  const int n_ext = (prec && NB == 1 && sizeof(T) == 8) ? prec->fused_rz_count() : 0;
  const size_t red_base = 2 * cg_part_doubles<T, NB>(G) + (size_t)G * NB * 4 + 64;
  IRK_TRY(ensure_red(ctx, red_base + 2 * (size_t)n_ext));
  IRK_TRY(ensure_pinned(ctx, 4 * sizeof(SysState<T>) + 64));
  cudaStream_t s = ctx->stream;
  unsigned int* cnt = ctx->counters + 4;
  SysState<T>* st0 = w.st;
  SysState<T>* st1 = w.st + 1;
  // init: state "before iteration 0" in st[1]; its partials go past the
  // two iteration partial buffers.  The right-hand side is first staged into
  // the workspace so the init sequence (init kernel, and for an external
  // preconditioner its first application and rho = r.z) has fixed launch
  // arguments and replays as one cached graph.
  double* red = ctx->red;
  static const bool graph_off = getenv("IRK_NO_GRAPH") != nullptr;
  // One graph per deferred solve (external preconditioner, graph-resident
  // loop): the init kernel, the solve and the closing log / store kernels are
  // captured together; the three kernels whose arguments change from solve to
  // solve (rhs, log slot, output) are updated in the instantiated graph
  // before every replay, so no eager kernel sits between consecutive solve
  // graphs (each eager <-> graph boundary costs ~9 us of GPU idle).  Env
  // IRK_NO_ONEGRAPH: eager init / log / store around the graph.
  static const bool onegraph_off = getenv("IRK_NO_ONEGRAPH") != nullptr;
  static const bool while_off_ = getenv("IRK_NO_WHILE") != nullptr;
  static const bool split_while_ = getenv("IRK_SPLIT_WHILE") != nullptr;
  // A solve issued while ctx->stream is being captured (the preconditioner
  // application of a device-resident FGMRES cycle, irk_fgmres.cu) becomes a
  // straight-line kernel sequence of the caller's graph: init, exactly
  // `maxit` iterations (kernels of a finished solve do nothing), store.  No
  // graph launch, no WHILE node (conditional nodes cannot sit in a child
  // graph), no log entry: the caller passes the fixed iteration count.
  cudaStreamCaptureStatus capst = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &capst) != cudaSuccess) capst = cudaStreamCaptureStatusNone;
  const bool captured = capst == cudaStreamCaptureStatusActive;
  if (captured) {
    IRK_REQUIRE(kExtOk && prec != nullptr && !its_host && !relres_host && maxit > 0 && maxit <= 8,
                "run_cg: only a deferred externally preconditioned solve of at most 8 fixed "
                "iterations can be captured");
  }
  const bool onegraph = kExtOk && prec != nullptr && !onegraph_off && !graph_off && !while_off_ &&
                        !split_while_ && maxit > 0 && !its_host && !relres_host && ctx->log_on &&
                        !captured;
  if constexpr (kExtOk) {
    if (prec && !onegraph) {
      // external preconditioner: the eager init reads the strided rhs itself
      launch(k_cg_init_ext<T>, G, kBlock, 0, s, m, rhs, ld_rhs, w.x, w.r, w.p0, rtol * rtol,
             atol * atol, st1, red + 2 * cg_part_doubles<T, NB>(G), cnt);
      IRK_CHECK_LAUNCH(ctx);
    }
  }
  if (!prec) {
    launch(k_cg_stage_rhs<T, NB>, grid_for(ctx, m), kBlock, 0, s, m, rhs, ld_rhs, w.rb);
    IRK_CHECK_LAUNCH(ctx);
  }
  auto init_body = [&](cudaStream_t cs) -> int {
    if (!prec) {
      launch(k_cg_init<T, NB, HASB>, G, kBlock, 0, cs, m, A, P, shift, mask, w.rb, NB, w.x, w.r,
             w.z, w.p0, w.dinv, rtol * rtol, atol * atol, st1,
             red + 2 * cg_part_doubles<T, NB>(G), cnt);
      IRK_CHECK_LAUNCH(ctx);
    }
    if constexpr (kExtOk) {
      if (prec && n_ext) {
        // rho comes from the preconditioner's r.z partials (parity 1, read
        // by A_0), taken by the first A kernel
        IRK_TRY(prec->apply_fused(ctx, cs, reinterpret_cast<double*>(w.r),
                                  reinterpret_cast<double*>(w.z), SkipCtl{},
                                  red + red_base + n_ext));
      } else if (prec) {
        IRK_TRY(prec->apply(ctx, cs, reinterpret_cast<double*>(w.r),
                            reinterpret_cast<double*>(w.z), nullptr));
        launch(k_cg_rho_init<T>, G, kBlock, 0, cs, m, w.r, w.z, st1,
               red + 2 * cg_part_doubles<T, NB>(G), cnt);
        IRK_CHECK_LAUNCH(ctx);
      }
    }
    return IRK_OK;
  };
  // pinned mirrors: two polls in flight, each of both states
  SysState<T>* hst = reinterpret_cast<SysState<T>*>(ctx->pinned);
  const int chunk = m < 65536 ? 8 : 16;
  constexpr bool kStencil = NB == 1 && sizeof(T) == 8 && MAXW > 0;
  static const bool stencil_off = getenv("IRK_NO_STENCIL") != nullptr;
  const bool stencil = kStencil && !stencil_off && w.pad > 0 && m < INT_MAX / 2 &&
                       (A.sw == 3 || A.sw == 5 || A.sw == 7 || A.sw == 9);
  // batched / complex systems on the P1 grid stencils (7-point 2D, 15-point 3D)
  constexpr bool kStencilN = !kStencil && MAXW > 0 && NB <= 4;
  constexpr int kWN = MAXW == 8 ? 7 : 15;
  const bool stencil_n = kStencilN && !stencil_off && w.pad > 0 && m < INT_MAX / 2 && A.sw == kWN;
  T* pbuf[2] = {w.p0, w.p1};
  // kernel A of iteration `it` (parity it & 1; the state says whether it
  // is the first one after the init)
  auto launch_a = [&](cudaStream_t cs, int it) -> int {
    const int c = it & 1;
    T* pold = pbuf[c];
    T* pnew = pbuf[c ^ 1];
    SysState<T>* sin = c ? st0 : st1;
    SysState<T>* sout = c ? st1 : st0;
    if constexpr (kStencil) {
      if (stencil) {
        const double* zz = reinterpret_cast<const double*>(w.z);
        const double* po = reinterpret_cast<const double*>(pold);
        double* pn = reinterpret_cast<double*>(pnew);
        double* qq = reinterpret_cast<double*>(w.q);
        const SysParams<double>& Pd = reinterpret_cast<const SysParams<double>&>(P);
        const SysState<double>* si = reinterpret_cast<const SysState<double>*>(sin);
        SysState<double>* so = reinterpret_cast<SysState<double>*>(sout);
        const double* ext = n_ext ? red + red_base + (size_t)(c ^ 1) * n_ext : nullptr;
#define IRK_ST(WW)                                                                            \
  launch(k_cg_spmv_st<WW, HASB>, G, kBlock, 0, cs, (int)m, A, Pd, shift, mask, zz, po, pn, qq, si, \
                                              so, red, c, maxit, ext, n_ext)
        if (A.sw == 7) IRK_ST(7);
        else if (A.sw == 9) IRK_ST(9);
        else if (A.sw == 5) IRK_ST(5);
        else IRK_ST(3);
#undef IRK_ST
      }
    }
    if constexpr (kStencilN) {
      if (stencil_n) {
        launch(k_cg_spmv_stn<T, NB, kWN, HASB>, G, kBlock, 0, cs, (int)m, A, P, shift, mask, w.z,
               pold, pnew, w.q, sin, sout, red, c, maxit);
        IRK_CHECK_LAUNCH(ctx);
        return IRK_OK;
      }
    }
    if (!stencil)
      launch(k_cg_spmv<T, NB, HASB, MAXW>, G, kBlock, 0, cs, m, A, P, shift, mask, w.z, pold, pnew,
             w.q, sin, sout, red, c, maxit,
             n_ext ? red + red_base + (size_t)(c ^ 1) * n_ext : (const double*)nullptr, n_ext);
    IRK_CHECK_LAUNCH(ctx);
    return IRK_OK;
  };
  auto launch_b = [&](cudaStream_t cs, int it) -> int {
    const int c = it & 1;
    if constexpr (kExtOk) {
      if (prec) {
        launch(k_cg_update<T, NB, true>, G, kBlock, 0, cs, m, pbuf[c ^ 1], w.q, w.dinv, w.x, w.r,
                                                       w.z, c ? st1 : st0, red, c);
        IRK_CHECK_LAUNCH(ctx);
        double* rr_ = reinterpret_cast<double*>(w.r);
        double* zz_ = reinterpret_cast<double*>(w.z);
        SysState<T>* sct = c ? st1 : st0;
        SysState<double>* sc = reinterpret_cast<SysState<double>*>(sct);  // real path only
        if (n_ext) {
          // the preconditioner decides the skip and writes r.z partials
          SkipCtl sk;
          sk.st = sc;
          sk.rr = cg_part<double, 1>(red, G, c).rr;
          sk.G = G;
          sk.maxit = maxit;
          return prec->apply_fused(ctx, cs, rr_, zz_, sk, red + red_base + (size_t)c * n_ext);
        }
        launch(k_cg_skip<T>, 1, kBlock, 0, cs, sct, red, G, c, maxit);
        IRK_CHECK_LAUNCH(ctx);
        IRK_TRY(prec->apply(ctx, cs, rr_, zz_, &sct->skip));
        launch(k_cg_dot_rz<T>, G, kBlock, 0, cs, m, w.r, w.z, red, c, &sct->skip);
        IRK_CHECK_LAUNCH(ctx);
        return IRK_OK;
      }
    }
    launch(k_cg_update<T, NB>, G, kBlock, 0, cs, m, pbuf[c ^ 1], w.q, w.dinv, w.x, w.r, w.z,
                                             c ? st1 : st0, red, c);
    IRK_CHECK_LAUNCH(ctx);
    return IRK_OK;
  };
  // iterations [it0, it0 + n)
  auto chunk_body = [&](cudaStream_t cs, int it0, int n) -> int {
    for (int t = 0; t < n; ++t) {
      IRK_TRY(launch_a(cs, it0 + t));
      IRK_TRY(launch_b(cs, it0 + t));
    }
    return IRK_OK;
  };
  // iterations issued with the init sequence (external preconditioner and
  // graph-resident loop only; even, so the loop keeps its parities)
  static const int prefix_env =
      getenv("IRK_CG_PREFIX") ? std::max(0, atoi(getenv("IRK_CG_PREFIX")) & ~1) : 4;
  static const bool while_off = getenv("IRK_NO_WHILE") != nullptr;  // A/B: chunked graphs
  const int prefix_hint = prec && !getenv("IRK_CG_PREFIX") ? prec->prefix_iters() : -1;
  const int prefix = (prec && maxit > 0 && !graph_off && !while_off)
                         ? (prefix_hint >= 0 ? (prefix_hint & ~1) : prefix_env)
                         : 0;
  if (captured) {
    IRK_TRY(init_body(s));
    IRK_TRY(chunk_body(s, 0, maxit));
    launch(k_cg_store<T, NB>, grid_for(ctx, m), kBlock, 0, s, m, w.x, xout, ld_x);
    IRK_CHECK_LAUNCH(ctx);
    return IRK_OK;
  }
  // The key holds every launch argument of the loop kernels.
  GraphKey key;
  key.add((const void*)&k_cg_spmv<T, NB, HASB, MAXW>).add((const void*)&k_cg_update<T, NB>);
  key.add(stencil).add(stencil_n).add(n_ext);
  key.add(m).add(G).add(A).add(P).add(shift).add(mask).add(w).add(red);
  key.add(maxit).add(prec ? prec->uid : (uint64_t)0);
  int64_t body_kernels = 0;  // kernels per pass of the graph-resident loop
  // CG iterations per WHILE pass: even, so every pass starts on parity 0
  static const int body_its =
      getenv("IRK_WHILE_BODY") ? 2 * std::max(1, atoi(getenv("IRK_WHILE_BODY")) / 2) : 2;
  // the loop condition at a parity-0 boundary: with an external
  // preconditioner the settling kernel (IRK_NO_SETTLE: the plain condition)
  static const bool settle_off = getenv("IRK_NO_SETTLE") != nullptr;
  const bool settle = prec != nullptr && !settle_off;
  auto launch_cond = [&](cudaStream_t cs, cudaGraphConditionalHandle h) -> int {
    if (settle)
      launch(k_cg_settle<T, NB>, 1, kBlock, 0, cs, h, (const SysState<T>*)st1, st0, red, (int)G,
             maxit, n_ext ? red + red_base + (size_t)n_ext : (const double*)nullptr, n_ext);
    else
      launch(k_cg_cond<T>, 1, 32, 0, cs, h, st0, st1);
    IRK_CHECK_LAUNCH(ctx);
    return IRK_OK;
  };
  auto while_body = [&](cudaStream_t cs, cudaGraphConditionalHandle h) -> int {
    // body_its is even: the loop kernels alternate the two state parities
    IRK_TRY(chunk_body(cs, 0, body_its));
    return launch_cond(cs, h);
  };
  static const bool split_while = getenv("IRK_SPLIT_WHILE") != nullptr;  // A/B: two graphs
  bool looped = false;
  if (maxit > 0 && !graph_off && !while_off && !split_while) {
    // init + the first `prefix` iterations + the conditional WHILE loop in
    // ONE graph (no second graph launch per solve)
    GraphKey kc;
    kc.add((const void*)&k_cg_init<T, NB, HASB>).add(m).add(G).add(A).add(P).add(shift);
    kc.add(mask).add(w).add(red).add(cnt).add(rtol).add(atol);
    kc.add(prec ? prec->uid : (uint64_t)0).add(prefix).add(stencil).add(maxit).add(n_ext);
    kc.k += key.k;
    kc.add(2).add(body_its).add(settle).add(onegraph);
    if constexpr (kExtOk) {
      if (onegraph) {
        IRK_TRY(log_reserve(ctx));
        cudaGraphNode_t un[3] = {nullptr, nullptr, nullptr};
        const int gs = grid_for(ctx, m);
        IRK_TRY(graph_launch_prefix_while(
            ctx, kc.k,
            [&](cudaStream_t cs, cudaGraphConditionalHandle h) -> int {
              launch(k_cg_init_ext<T>, G, kBlock, 0, cs, m, rhs, ld_rhs, w.x, w.r, w.p0,
                     rtol * rtol, atol * atol, st1, red + 2 * cg_part_doubles<T, NB>(G), cnt);
              IRK_CHECK_LAUNCH(ctx);
              un[0] = capture_tail(cs);
              IRK_TRY(init_body(cs));
              IRK_TRY(chunk_body(cs, 0, prefix));
              if (settle && prefix > 0) return launch_cond(cs, h);
              return IRK_OK;
            },
            while_body, &body_kernels,
            [&](cudaStream_t cs) -> int {
              // after the WHILE node (not a kernel: no programmatic edge)
              launch_plain(k_cg_log<T>, 1, 32, 0, cs, st0, st1, NB, (int)body_kernels, prefix,
                           (int)settle, ctx->solve_log + 4 * ctx->log_n);
              IRK_CHECK_LAUNCH(ctx);
              un[1] = capture_tail(cs);
              launch(k_cg_store<T, NB>, gs, kBlock, 0, cs, m, w.x, xout, ld_x);
              IRK_CHECK_LAUNCH(ctx);
              un[2] = capture_tail(cs);
              return IRK_OK;
            },
            un, 3,
            [&](cudaGraphExec_t ex, const cudaGraphNode_t* nd) -> int {
              IRK_CUDA(exec_set_kernel_args(ex, nd[0], k_cg_init_ext<T>, dim3(G), dim3(kBlock), m,
                                            rhs, ld_rhs, w.x, w.r, w.p0, rtol * rtol, atol * atol,
                                            st1, red + 2 * cg_part_doubles<T, NB>(G), cnt));
              IRK_CUDA(exec_set_kernel_args(ex, nd[1], k_cg_log<T>, dim3(1), dim3(32), st0, st1, NB,
                                            (int)body_kernels, prefix, (int)settle,
                                            ctx->solve_log + 4 * ctx->log_n));
              IRK_CUDA(exec_set_kernel_args(ex, nd[2], k_cg_store<T, NB>, dim3(gs), dim3(kBlock), m,
                                            w.x, xout, ld_x));
              return IRK_OK;
            }));
        ctx->log_n++;
        return IRK_OK;
      }
    }
    IRK_TRY(graph_launch_prefix_while(
        ctx, kc.k,
        [&](cudaStream_t cs, cudaGraphConditionalHandle h) -> int {
          IRK_TRY(init_body(cs));
          IRK_TRY(chunk_body(cs, 0, prefix));
          // a solve that finished inside the prefix skips the loop
          if (settle && prefix > 0) return launch_cond(cs, h);
          return IRK_OK;
        },
        while_body, &body_kernels));
    looped = true;
  } else {
    GraphKey ki;
    ki.add((const void*)&k_cg_init<T, NB, HASB>).add(m).add(G).add(A).add(P).add(shift);
    ki.add(mask).add(w).add(red).add(cnt).add(rtol).add(atol);
    ki.add(prec ? prec->uid : (uint64_t)0).add(prefix).add(stencil).add(maxit).add(n_ext);
    if (graph_off) {
      IRK_TRY(init_body(s));
    } else {
      // the first `prefix` iterations ride in the init graph (straight-line
      // graphs run the V-cycle-preconditioned iteration ~20 us faster than
      // the body of the conditional WHILE node); later ones are no-ops once
      // the state is finished
      IRK_TRY(graph_launch(ctx, ki.k, [&](cudaStream_t cs) -> int {
        IRK_TRY(init_body(cs));
        return chunk_body(cs, 0, prefix);
      }));
    }
  }
  if (looped) {
    // init, prefix and loop went out as one graph above
  } else if (maxit > 0 && !graph_off && !while_off) {
    // The whole iteration loop is ONE graph: a conditional WHILE node whose
    // body runs two iterations (both parities) and then sets the loop
    // condition from the device state; termination never returns to the
    // host.  The body's kernels do nothing once the state is finished.
    GraphKey kw = key;
    kw.add(1).add(body_its);
    IRK_TRY(graph_launch_while(ctx, kw.k, while_body, &body_kernels));
  } else {
    // Chunked issue with one chunk in flight ahead of the host check; full
    // chunks replay a cached CUDA graph (host launch cost once per chunk).
    const int chunk = m < 65536 ? 8 : 16;
    int issued = 0, poll = 0;
    if (maxit > 0) {
      IRK_TRY(launch_a(s, 0));
      IRK_TRY(launch_b(s, 0));
      issued = 1;
    }
    for (;;) {
      if (issued >= maxit) break;
      if (issued + chunk <= maxit && !graph_off) {
        GraphKey kp = key;
        kp.add(issued & 1).add(chunk);
        const int it0 = issued;
        IRK_TRY(graph_launch(ctx, kp.k,
                             [&](cudaStream_t cs) { return chunk_body(cs, it0, chunk); }));
        issued += chunk;
      } else {
        const int n = std::min(chunk, maxit - issued);
        IRK_TRY(chunk_body(s, issued, n));
        issued += n;
      }
      SysState<T>* hp = hst + 2 * (poll & 1);
      IRK_CUDA(cudaMemcpyAsync(hp, w.st, 2 * sizeof(SysState<T>), cudaMemcpyDeviceToHost, s));
      IRK_CUDA(cudaEventRecord(ctx->ev[poll & 1], s));
      if (poll > 0) {
        IRK_CUDA(cudaEventSynchronize(ctx->ev[(poll - 1) & 1]));
        const SysState<T>* hq = hst + 2 * ((poll - 1) & 1);
        if (hq[0].done || hq[1].done) break;
      }
      poll++;
    }
    // finalising A: applies the decisions of the last issued iteration (cap)
    IRK_TRY(launch_a(s, issued));
  }
  if (!its_host && !relres_host && ctx->log_on) {
    // deferred status: log the outcome on the device, no host round trip
    IRK_TRY(log_reserve(ctx));
    launch(k_cg_log<T>, 1, 32, 0, s, st0, st1, NB, (int)body_kernels, prefix,
                                 (int)(settle && looped), ctx->solve_log + 4 * ctx->log_n);
    IRK_CHECK_LAUNCH(ctx);
    ctx->log_n++;
    launch(k_cg_store<T, NB>, grid_for(ctx, m), kBlock, 0, s, m, w.x, xout, ld_x);
    IRK_CHECK_LAUNCH(ctx);
    return IRK_OK;
  }
  IRK_CUDA(cudaMemcpyAsync(hst, w.st, 2 * sizeof(SysState<T>), cudaMemcpyDeviceToHost, s));
  launch(k_cg_store<T, NB>, grid_for(ctx, m), kBlock, 0, s, m, w.x, xout, ld_x);
  IRK_CHECK_LAUNCH(ctx);
  IRK_CUDA(cudaStreamSynchronize(s));
  // the latest state: the finished one (or the later iteration)
  const SysState<T>& fs = (hst[0].done != hst[1].done) ? (hst[0].done ? hst[0] : hst[1])
                          : (hst[0].iter >= hst[1].iter ? hst[0] : hst[1]);
  // body passes executed by the graph-resident loop: iterations in pairs,
  // plus the pass in which the finished state was observed
  if (body_kernels) {
    const int64_t rest = std::max(fs.iter - prefix, 0);
    ctx->launches += body_kernels * ((settle && looped) ? (rest + 1) / 2 : rest / 2 + 1);
  }
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
int dispatch_flags(irk_ctx* ctx, int64_t m, int maxw, const MatView& A, const SysParams<T>& P,
                   const double* shift, const uint8_t* mask, const T* rhs, int64_t ld_rhs, T* x,
                   int64_t ld_x, double rtol, double atol, int maxit, int* its, double* rel) {
  const bool hb = A.b != nullptr;
#define IRK_RUN(HB, W)                                                                         \
  return run_cg<T, NB, HB, W>(ctx, m, A, P, shift, mask, rhs, ld_rhs, x, ld_x, rtol, atol, maxit, \
                              its, rel)
  if (maxw <= 8) {
    if (hb) IRK_RUN(true, 8);
    IRK_RUN(false, 8);
  }
  if (maxw <= 16) {
    if (hb) IRK_RUN(true, 16);
    IRK_RUN(false, 16);
  }
  if (hb) IRK_RUN(true, 0);
  IRK_RUN(false, 0);
#undef IRK_RUN
}

inline MatView make_view(const irk_mat* A, const irk_mat* Bm) {
  const Pattern* p = A->pat;
  MatView v{p->slice_ptr, p->sell_col, p->colhdr, p->diag_pos, A->val, A->uval,
            Bm ? Bm->val : nullptr, Bm ? Bm->uval : nullptr, p->ellw, 0, {}};
  if (p->ellw > 0 && (int)p->stencil.size() == p->ellw && p->ellw <= 16) {
    v.sw = p->ellw;
    for (int k = 0; k < v.sw; ++k) v.sd[k] = p->stencil[k];
  }
  return v;
}

}  // namespace irk
