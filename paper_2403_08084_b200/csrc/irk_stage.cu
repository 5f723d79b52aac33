// Stage-operator kernels on the stage-interleaved m-by-s layout (K2, K6-K9).
//
// Reference anchors (under /root/reference/pkg/src/implicitrk/):
//   KroneckerStageOperator.apply   sparsela.py:222-235
//   ConstrainedStageOperator.apply bcs.py:114-120
//   constrain_stage_system         bcs.py:123-142
//   assemble_linear_stage_system   stepper.py:275-302
//   _stage_value_system            stepper.py:305-313
//   step_linear update             stepper.py:352-361
//   step_newton residual/stages    stepper.py:502-524
#include <cstdlib>
#include <vector>

#include "irk_internal.cuh"

namespace irk {

struct Coef2 {
  double c1[kMaxStages * kMaxStages];
  double c2[kMaxStages * kMaxStages];
};

struct KPtrs {
  const double* k[kMaxStages];
};

// Out_r = C1 (M Y)_r + dt C2 (K Y)_r  (shared K)
// Out_r,i = (C1 (M Y)_r)_i + dt (K_i (C2 Y))_r,i  (per-stage K_i)
// mask: flagged rows are identity; flagged columns must already be
// eliminated from M and K (irk_mat_constrain with diagonal 0).
// MAXW > 0: all column indices / values of the row are loaded first, then
// the stage-vector gathers are issued (one dependency level per row).
template <int S, bool PERSTAGE, int MAXW>
__global__ void __launch_bounds__(kBlock)
    k_stage_apply(int64_t m, const int* __restrict__ slice_ptr, const int* __restrict__ sell_col,
                  const double* __restrict__ mval, KPtrs kp, const Coef2 cf, double dt,
                  const uint8_t* __restrict__ mask, const double* __restrict__ Y,
                  double* __restrict__ Out, int ellw) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  // no early exit on flagged rows: the row result is computed (the matrices
  // carry zero rows there) and replaced at the end, so every load issues
  // without waiting for the mask
  const bool flagged = mask && mask[r];
  const int64_t s = r / kSlice;
  const int lane = (int)(r % kSlice);
  int base, width;
  if (ellw) {
    base = (int)(s * kSlice * ellw);
    width = ellw;
  } else {
    base = __ldg(slice_ptr + s);
    width = (__ldg(slice_ptr + s + 1) - base) / kSlice;
  }
  double a[S], b[S];
#pragma unroll
  for (int i = 0; i < S; ++i) a[i] = b[i] = 0.0;
  if (MAXW > 0 && !PERSTAGE) {
    int cc[MAXW > 0 ? MAXW : 1];
    double mv[MAXW > 0 ? MAXW : 1], kv[MAXW > 0 ? MAXW : 1];
#pragma unroll
    for (int k = 0; k < MAXW; ++k) {
      if (k < width) {
        const int pos = base + k * kSlice + lane;
        cc[k] = __ldg(sell_col + pos);
        mv[k] = __ldg(mval + pos);
        kv[k] = __ldg(kp.k[0] + pos);
      }
    }
#pragma unroll
    for (int k = 0; k < MAXW; ++k) {
      if (k < width) {
        const double* yc = Y + (int64_t)cc[k] * S;
#pragma unroll
        for (int i = 0; i < S; ++i) {
          const double y = __ldg(yc + i);
          a[i] += mv[k] * y;
          b[i] += kv[k] * y;
        }
      }
    }
  } else {
    for (int k = 0; k < width; ++k) {
      const int pos = base + k * kSlice + lane;
      const int c = __ldg(sell_col + pos);
      const double m_ = __ldg(mval + pos);
      double y[S];
#pragma unroll
      for (int i = 0; i < S; ++i) y[i] = __ldg(Y + (int64_t)c * S + i);
      if (!PERSTAGE) {
        const double k_ = __ldg(kp.k[0] + pos);
#pragma unroll
        for (int i = 0; i < S; ++i) {
          a[i] += m_ * y[i];
          b[i] += k_ * y[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < S; ++i) {
          a[i] += m_ * y[i];
          double w = 0.0;
#pragma unroll
          for (int j = 0; j < S; ++j) w += cf.c2[i * S + j] * y[j];
          b[i] += __ldg(kp.k[i] + pos) * w;
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < S; ++i) {
    double o = 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j) o += cf.c1[i * S + j] * a[j];
    if (!PERSTAGE) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) t += cf.c2[i * S + j] * b[j];
      o += dt * t;
    } else {
      o += dt * b[i];
    }
    Out[r * S + i] = flagged ? Y[r * S + i] : o;
  }
}

// Windowed variant of K2 (shared K), one warp per SELL slice.  When every
// slot of the slice has a uniform column offset (slot-uniform header), the
// stage-block rows the slice touches form a few contiguous windows
// (offsets closer than kWinGap rows are merged: on the 2D P1 grid the 7
// offsets give 3 windows of ~34 rows; a decreasing offset, e.g. an ELL
// padding slot, starts a new window so offsets never decrease inside one).  The warp copies those windows with
// fully coalesced loads into its shared-memory buffer and every entry's
// stage values are then read from shared memory; the matrix values are
// still streamed per entry (16 B/nnz, the column index is implied by the
// header).  Other slices use the per-entry gather path.

constexpr int kWinBatch = 4;  // buffer rows per lane with loads in flight

template <int S, int MAXW>
__global__ void __launch_bounds__(kBlock, MAXW <= 10 ? 3 : 2)
    k_stage_apply_win(int64_t m, int64_t nslices, const int* __restrict__ slice_ptr,
                      const int* __restrict__ sell_col, const int* __restrict__ colhdr,
                      const double* __restrict__ mval, const double* __restrict__ kval,
                      const Coef2 cf, double dt, const uint8_t* __restrict__ mask,
                      const double* __restrict__ Y, double* __restrict__ Out, int ellw,
                      int wrows) {
  extern __shared__ double wsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t sl = (int64_t)blockIdx.x * (kBlock / 32) + warp;
  if (sl >= nslices) return;
  constexpr int SP = (S % 2 == 0) ? S + 1 : S;  // odd row stride: no bank conflicts
  double* buf = wsm + (size_t)warp * wrows * SP;
  const int64_t r0 = sl * kSlice, r = r0 + lane;
  int base, width;
  if (ellw) {
    base = (int)(sl * kSlice * ellw);
    width = ellw;
  } else {
    base = __ldg(slice_ptr + sl);
    width = (__ldg(slice_ptr + sl + 1) - base) / kSlice;
  }
  const int q0 = base / kSlice;
  const bool flagged = r < m && mask && mask[r];
  // matrix values of the row (coalesced across the warp), issued first
  double mv[MAXW], kv[MAXW];
#pragma unroll
  for (int k = 0; k < MAXW; ++k) {
    if (k < width) {
      mv[k] = __ldg(mval + base + k * kSlice + lane);
      kv[k] = __ldg(kval + base + k * kSlice + lane);
    }
  }
  // slot offsets: lane k < width holds d_k
  const int d = lane < width ? __ldg(colhdr + q0 + lane) : 0;
  bool uni = __all_sync(0xffffffffu, lane >= width || d != kNonUniform);
  double a[S], b[S];
#pragma unroll
  for (int i = 0; i < S; ++i) a[i] = b[i] = 0.0;
  if (uni) {
    const WinLayout L = win_layout(d, width);
    if (L.total <= wrows) {
      // copy the windows into the buffer: lane l moves buffer rows l, l+32,
      // ... (S doubles each), kWinBatch rows per batch with all loads issued
      // before the stores; global row = buffer row + r0 + dfirst_w - wbase_w
      const int rshift = (int)r0 + L.dfirst - L.wbase;  // valid on end lanes
      for (int g = 0; g < L.total; g += 32 * kWinBatch) {
        int sh[kWinBatch];
#pragma unroll
        for (int c = 0; c < kWinBatch; ++c) sh[c] = 0;
        unsigned ends = L.ends;
        while (ends) {
          const int e = __ffs(ends) - 1;
          ends &= ends - 1;
          const int wb = __shfl_sync(0xffffffffu, L.wbase, e);
          const int sf = __shfl_sync(0xffffffffu, rshift, e);
#pragma unroll
          for (int c = 0; c < kWinBatch; ++c)
            if (g + c * 32 + lane >= wb) sh[c] = sf;
        }
        double v[kWinBatch][S];
#pragma unroll
        for (int c = 0; c < kWinBatch; ++c) {
          const int br = g + c * 32 + lane;
          const int64_t gr = (int64_t)br + sh[c];
          const bool in = br < L.total && gr >= 0 && gr < m;
#pragma unroll
          for (int i = 0; i < S; ++i) v[c][i] = in ? __ldg(Y + gr * S + i) : 0.0;
        }
#pragma unroll
        for (int c = 0; c < kWinBatch; ++c) {
          const int br = g + c * 32 + lane;
          if (br < L.total) {
#pragma unroll
            for (int i = 0; i < S; ++i) buf[br * SP + i] = v[c][i];
          }
        }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < MAXW; ++k) {
        if (k < width) {
          const int o = __shfl_sync(0xffffffffu, L.row, k);
          const double* yr = buf + (o + lane) * SP;
#pragma unroll
          for (int i = 0; i < S; ++i) {
            const double y = yr[i];
            a[i] += mv[k] * y;
            b[i] += kv[k] * y;
          }
        }
      }
    } else {
      uni = false;
    }
  }
  if (!uni && r < m) {
#pragma unroll
    for (int k = 0; k < MAXW; ++k) {
      if (k < width) {
        const int c = __ldg(sell_col + base + k * kSlice + lane);
        const double* yc = Y + (int64_t)c * S;
#pragma unroll
        for (int i = 0; i < S; ++i) {
          const double y = __ldg(yc + i);
          a[i] += mv[k] * y;
          b[i] += kv[k] * y;
        }
      }
    }
  }
  if (r >= m) return;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    double o = 0.0, t = 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      o += cf.c1[i * S + j] * a[j];
      t += cf.c2[i * S + j] * b[j];
    }
    Out[r * S + i] = flagged ? Y[r * S + i] : o + dt * t;
  }
}

// Stencil variant of the windowed K2 for stencil-aligned ELL patterns: the
// window layout of a plain stencil slice (every slot at the pattern's
// stencil offset) is the same for all of them, so it is computed once on
// the host and passed in (no per-slice shuffles / scans); a warp vote on
// the slot headers selects it, other slices gather per entry.
struct StLayout {
  int nwin, total;
  int wstart[16], wbase[16], wend[16];  // window w: rows [r0+wstart, ...), buffer rows [wbase, wend)
  int srow[16];                         // buffer row of slot k for lane 0
  int sd[16];                           // stencil offsets
};

template <int S, int W, int NW>
__global__ void __launch_bounds__(kBlock, W <= 8 ? 3 : 2)
    k_stage_apply_std(int64_t m, int64_t nslices, const StLayout SL,
                      const int* __restrict__ sell_col, const int* __restrict__ colhdr,
                      const double* __restrict__ mval, const double* __restrict__ kval,
                      const Coef2 cf, double dt, const uint8_t* __restrict__ mask,
                      const double* __restrict__ Y, double* __restrict__ Out) {
  extern __shared__ double wsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t sl = (int64_t)blockIdx.x * (kBlock / 32) + warp;
  if (sl >= nslices) return;
  constexpr int SP = (S % 2 == 0) ? S + 1 : S;
  double* buf = wsm + (size_t)warp * SL.total * SP;
  const int64_t r0 = sl * kSlice, r = r0 + lane;
  const int base = (int)(sl * kSlice * W);
  const int q0 = (int)(sl * W);
  const bool flagged = r < m && mask && mask[r];
  double mv[W], kv[W];
#pragma unroll
  for (int k = 0; k < W; ++k) {
    mv[k] = __ldg(mval + base + k * kSlice + lane);
    kv[k] = __ldg(kval + base + k * kSlice + lane);
  }
  const int d = lane < W ? __ldg(colhdr + q0 + lane) : 0;
  const bool std_slice = __all_sync(0xffffffffu, lane >= W || d == SL.sd[lane < W ? lane : 0]);
  double a[S], b[S];
#pragma unroll
  for (int i = 0; i < S; ++i) a[i] = b[i] = 0.0;
  if (std_slice) {
    // copy the windows: buffer row br of window w is stage row r0 + wstart_w + br - wbase_w
    const int64_t lim = m * S;
    for (int g = 0; g < SL.total; g += 32 * kWinBatch) {
      double v[kWinBatch][S];
#pragma unroll
      for (int c = 0; c < kWinBatch; ++c) {
        const int br = g + c * 32 + lane;
        int sh = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w)
          if (br >= SL.wbase[w]) sh = SL.wstart[w] - SL.wbase[w];
        const int64_t g0 = (r0 + br + sh) * S;
        const bool in = br < SL.total && g0 >= 0 && g0 < lim;
#pragma unroll
        for (int i = 0; i < S; ++i) v[c][i] = in ? __ldg(Y + g0 + i) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < kWinBatch; ++c) {
        const int br = g + c * 32 + lane;
        if (br < SL.total) {
#pragma unroll
          for (int i = 0; i < S; ++i) buf[br * SP + i] = v[c][i];
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const double* yr = buf + (SL.srow[k] + lane) * SP;
#pragma unroll
      for (int i = 0; i < S; ++i) {
        const double y = yr[i];
        a[i] += mv[k] * y;
        b[i] += kv[k] * y;
      }
    }
  } else if (r < m) {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int c = sell_col_at(colhdr, sell_col, q0 + k, base + k * kSlice + lane, r);
      const double* yc = Y + (int64_t)c * S;
#pragma unroll
      for (int i = 0; i < S; ++i) {
        const double y = __ldg(yc + i);
        a[i] += mv[k] * y;
        b[i] += kv[k] * y;
      }
    }
  }
  if (r >= m) return;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    double o = 0.0, t = 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      o += cf.c1[i * S + j] * a[j];
      t += cf.c2[i * S + j] * b[j];
    }
    Out[r * S + i] = flagged ? Y[r * S + i] : o + dt * t;
  }
}

// host: window layout of a sorted stencil (the win_layout rule)
static bool stencil_layout(const std::vector<int>& sd, StLayout& L) {
  const int W = (int)sd.size();
  if (W < 1 || W > 16) return false;
  L = StLayout{};
  int nw = 0, total = 0, start = 0;
  std::vector<int> win(W);
  for (int k = 0; k < W; ++k) {
    if (k == 0 || sd[k] < sd[k - 1] || sd[k] - sd[k - 1] > kWinGap) {
      if (k > 0) {
        L.wend[nw - 1] = L.wbase[nw - 1] + (sd[k - 1] - L.wstart[nw - 1]) + kSlice;
        total = L.wend[nw - 1];
      }
      if (nw == 16) return false;
      L.wstart[nw] = sd[k];
      L.wbase[nw] = total;
      start = k;
      ++nw;
    }
    win[k] = nw - 1;
  }
  (void)start;
  L.wend[nw - 1] = L.wbase[nw - 1] + (sd[W - 1] - L.wstart[nw - 1]) + kSlice;
  total = L.wend[nw - 1];
  L.nwin = nw;
  L.total = total;
  for (int k = 0; k < W; ++k) {
    L.srow[k] = L.wbase[win[k]] + sd[k] - L.wstart[win[k]];
    L.sd[k] = sd[k];
  }
  return true;
}

struct Mat8 {
  double q[kMaxStages * kMaxStages];
};

#include "irk_stage_bulk.cuh"

// launch k_stage_apply_bulk<s, W, KT> on a persistent grid (resident CTAs
// per SM from the occupancy API, queried once per instantiation)
template <int S, int W, int KT, int NST, bool VD = false>
static void launch_bulk_s(irk_ctx* ctx, int64_t m, int64_t ns, int64_t ntiles,
                          const BulkLayout& BL, size_t sm, const Pattern* P, const double* mv,
                          const double* kv, const Coef2& cf, double dt, const uint8_t* mask,
                          const double* Y, double* Out) {
  static int occ = 0;
  static size_t occ_sm = 0;
  if (!occ || occ_sm != sm) {
    cudaFuncSetAttribute(k_stage_apply_bulk<S, W, KT, NST, VD>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stage_apply_bulk<S, W, KT, NST, VD>,
                                                  KT * 32, sm);
    occ = std::max(occ, 1);
    occ_sm = sm;
  }
  const unsigned gb = (unsigned)std::min<int64_t>(ntiles, (int64_t)ctx->num_sms * occ);
  k_stage_apply_bulk<S, W, KT, NST, VD><<<gb, KT * 32, sm, ctx->stream>>>(
      m, ns, ntiles, BL, P->sell_col, P->colhdr, mv, kv, cf, dt, mask, Y, Out);
}
template <int W, int KT, int NST, bool VD = false>
static void launch_bulk(irk_ctx* ctx, int s, int64_t m, int64_t ns, int64_t ntiles,
                        const BulkLayout& BL, size_t sm, const Pattern* P, const double* mv,
                        const double* kv, const Coef2& cf, double dt, const uint8_t* mask,
                        const double* Y, double* Out) {
  switch (s) {
    case 1: launch_bulk_s<1, W, KT, NST, VD>(ctx, m, ns, ntiles, BL, sm, P, mv, kv, cf, dt, mask, Y, Out); break;
    case 2: launch_bulk_s<2, W, KT, NST, VD>(ctx, m, ns, ntiles, BL, sm, P, mv, kv, cf, dt, mask, Y, Out); break;
    case 3: launch_bulk_s<3, W, KT, NST, VD>(ctx, m, ns, ntiles, BL, sm, P, mv, kv, cf, dt, mask, Y, Out); break;
    default: launch_bulk_s<4, W, KT, NST, VD>(ctx, m, ns, ntiles, BL, sm, P, mv, kv, cf, dt, mask, Y, Out); break;
  }
}

// Semilinear per-stage Jacobian K_i = kscale K + M diag(D_i):
// Out_r,i = (C1 (M Y))_i + dt*kscale (C2 (K Y))_i + dt (M (D_i o (C2 Y)_i))_r
template <int S>
__global__ void __launch_bounds__(kBlock)
    k_stage_apply_semi(int64_t m, const int* __restrict__ slice_ptr,
                       const int* __restrict__ sell_col, const double* __restrict__ mval,
                       const double* __restrict__ kval, const Coef2 cf, double dt, double kscale,
                       const double* __restrict__ D, const uint8_t* __restrict__ mask,
                       const double* __restrict__ Y, double* __restrict__ Out) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  if (mask && mask[r]) {
#pragma unroll
    for (int i = 0; i < S; ++i) Out[r * S + i] = Y[r * S + i];
    return;
  }
  int64_t s = r / kSlice;
  int lane = (int)(r % kSlice);
  int base = __ldg(slice_ptr + s), width = (__ldg(slice_ptr + s + 1) - base) / kSlice;
  double a[S], b[S], e[S];
#pragma unroll
  for (int i = 0; i < S; ++i) a[i] = b[i] = e[i] = 0.0;
  for (int k = 0; k < width; ++k) {
    int pos = base + k * kSlice + lane;
    int c = __ldg(sell_col + pos);
    double mv = __ldg(mval + pos), kv = __ldg(kval + pos);
    double y[S];
#pragma unroll
    for (int i = 0; i < S; ++i) y[i] = __ldg(Y + (int64_t)c * S + i);
#pragma unroll
    for (int i = 0; i < S; ++i) {
      a[i] += mv * y[i];
      b[i] += kv * y[i];
      double w = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) w += cf.c2[i * S + j] * y[j];
      e[i] += mv * (__ldg(D + (int64_t)c * S + i) * w);
    }
  }
#pragma unroll
  for (int i = 0; i < S; ++i) {
    double o = 0.0, t = 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      o += cf.c1[i * S + j] * a[j];
      t += cf.c2[i * S + j] * b[j];
    }
    Out[r * S + i] = o + dt * (kscale * t + e[i]);
  }
}

__global__ void k_stage_mix(int64_t m, int so, int si, const Mat8 Q, const double* __restrict__ X,
                            double* __restrict__ Y) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    double x[kMaxStages];
#pragma unroll
    for (int j = 0; j < kMaxStages; ++j) x[j] = j < si ? X[r * si + j] : 0.0;
#pragma unroll
    for (int i = 0; i < kMaxStages; ++i) {
      if (i >= so) break;
      double o = 0.0;
#pragma unroll
      for (int j = 0; j < kMaxStages; ++j) o += Q.q[i * kMaxStages + j] * x[j];
      Y[r * so + i] = o;
    }
  }
}

// Slot-uniform SELL row access (colhdr/uval headers: one broadcast load per
// slot instead of the 12 B per entry of sell_col + val)
struct SellRow {
  int q0, base, width, lane;
  __device__ __forceinline__ SellRow(const int* __restrict__ slice_ptr, int ellw, int64_t r) {
    const int64_t sl = r / kSlice;
    lane = (int)(r % kSlice);
    if (ellw) {
      base = (int)(sl * kSlice * ellw);
      width = ellw;
    } else {
      base = __ldg(slice_ptr + sl);
      width = (__ldg(slice_ptr + sl + 1) - base) / kSlice;
    }
    q0 = base / kSlice;
  }
};

// out[r*ld] = R[r*s+i] - sum_c C[r,c] sum_{j in J} coef[j] X[c*s+j]  (masked);
// J = the stages with a nonzero coefficient (jmask), gathered only those
template <int S, int W>
__global__ void __launch_bounds__(kBlock)
    k_stage_couple(int64_t m, int i, const int* __restrict__ slice_ptr, int ellw,
                   const int* __restrict__ colhdr, const int* __restrict__ sell_col,
                   const double* __restrict__ uval, const double* __restrict__ cval,
                   const Mat8 coef, unsigned jmask, const uint8_t* __restrict__ mask,
                   const double* __restrict__ R, const double* __restrict__ X,
                   double* __restrict__ out, int64_t ld_out) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  double rv = R[r * S + i];
  if (mask && mask[r]) {
    out[r * ld_out] = rv;
    return;
  }
  const SellRow sr(slice_ptr, ellw, r);
  double acc = 0.0;
  if (W > 0) {
    // ELL pattern of width W: every header, column and gather of the row is
    // issued before the first use (one dependency level)
    int cs[W > 0 ? W : 1];
    double av[W > 0 ? W : 1];
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int pos = sr.base + k * kSlice + sr.lane;
      cs[k] = sell_col_at(colhdr, sell_col, sr.q0 + k, pos, r);
      av[k] = sell_val_at(uval, cval, sr.q0 + k, pos);
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {
      double w = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j)
        if (jmask & (1u << j)) w += coef.q[j] * __ldg(X + (int64_t)cs[k] * S + j);
      acc += av[k] * w;
    }
  } else {
    for (int k = 0; k < sr.width; ++k) {
      const int pos = sr.base + k * kSlice + sr.lane;
      const int c = sell_col_at(colhdr, sell_col, sr.q0 + k, pos, r);
      double w = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j)
        if (jmask & (1u << j)) w += coef.q[j] * __ldg(X + (int64_t)c * S + j);
      acc += sell_val_at(uval, cval, sr.q0 + k, pos) * w;
    }
  }
  out[r * ld_out] = rv - acc;
}

// Out_r,i = a (B u)_r + sum_j G_ij F_r,j
template <int S>
__global__ void __launch_bounds__(kBlock)
    k_stage_rhs(int64_t m, const int* __restrict__ slice_ptr, int ellw,
                const int* __restrict__ colhdr, const int* __restrict__ sell_col,
                const double* __restrict__ ubval, const double* __restrict__ bval, double a,
                const double* __restrict__ u, const Mat8 G, const double* __restrict__ F,
                double* __restrict__ Out) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  double bu = 0.0;
  if (bval) {
    const SellRow sr(slice_ptr, ellw, r);
    for (int k = 0; k < sr.width; ++k) {
      const int pos = sr.base + k * kSlice + sr.lane;
      bu += sell_val_at(ubval, bval, sr.q0 + k, pos) *
            __ldg(u + sell_col_at(colhdr, sell_col, sr.q0 + k, pos, r));
    }
    bu *= a;
  } else if (u) {
    bu = a * u[r];  // B = identity
  }
  double f[S];
  if (F) {
#pragma unroll
    for (int j = 0; j < S; ++j) f[j] = F[r * S + j];
  }
#pragma unroll
  for (int i = 0; i < S; ++i) {
    double o = bu;
    if (F) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) t += G.q[i * S + j] * f[j];
      o += t;
    }
    Out[r * S + i] = o;
  }
}

template <int S>
__global__ void k_stage_update(int64_t m, double a, const double* __restrict__ u, const Mat8 w,
                               int copy_stage, const double* __restrict__ X,
                               double* __restrict__ un) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (copy_stage >= 0) {
      un[r] = X[r * S + copy_stage];
      continue;
    }
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < S; ++i) acc += w.q[i] * X[r * S + i];
    un[r] = (a == 0.0 ? 0.0 : a * u[r]) + acc;
  }
}

__global__ void k_stage_scale(int64_t m, int s, const Mat8 w, const double* __restrict__ v,
                              const double* __restrict__ D, double* __restrict__ out) {
  int64_t n = m * s;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = q / s;
    int i = (int)(q - r * s);
    out[q] = w.q[i] * v[r] * (D ? D[q] : 1.0);
  }
}

__global__ void k_stage_get(int64_t m, int s, int i, const double* __restrict__ X,
                            double* __restrict__ x) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x)
    x[r] = X[r * s + i];
}

__global__ void k_stage_set(int64_t m, int s, int i, const double* __restrict__ x,
                            double* __restrict__ X) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x)
    X[r * s + i] = x[r];
}

__global__ void k_to_interleaved(int64_t m, int s, const double* __restrict__ sm,
                                 double* __restrict__ il) {
  int64_t n = m * s;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = q / s;
    int i = (int)(q - r * s);
    il[q] = sm[(int64_t)i * m + r];
  }
}

__global__ void k_to_stage_major(int64_t m, int s, const double* __restrict__ il,
                                 double* __restrict__ sm) {
  int64_t n = m * s;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = q / m;
    int64_t r = q - i * m;
    sm[q] = il[r * s + i];
  }
}

__global__ void k_bc_scatter(int s, int64_t nb, const int64_t* __restrict__ idx,
                             const double* __restrict__ V, double* __restrict__ X) {
  int64_t n = nb * s;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = q / nb, k = q - i * nb;
    X[idx[k] * s + i] = V[q];
  }
}

__global__ void k_bc_gather(int64_t nb, const int64_t* __restrict__ idx,
                            const double* __restrict__ x, double* __restrict__ v) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nb;
       k += (int64_t)gridDim.x * blockDim.x)
    v[k] = x[idx[k]];
}

// DAE boundary values of the stage unknowns from the boundary state on the
// device (bcs.py:58-96): W[i,k] = (G[i,k] - u[idx[k]]) / dt, out = W (W
// unknowns) or A^-1 W (derivative unknowns; Ainv row-major s x s, by value)
__global__ void k_bc_dae(int s, int64_t nb, const int64_t* __restrict__ idx,
                         const double* __restrict__ G, const double* __restrict__ u, double dt,
                         Mat8 Ainv, int derivative, double* __restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nb;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double ub = u[idx[k]];
    double w[kMaxStages];
    for (int i = 0; i < s; ++i) w[i] = (G[(int64_t)i * nb + k] - ub) / dt;
    for (int i = 0; i < s; ++i) {
      double v = w[i];
      if (derivative) {
        v = 0.0;
        for (int j = 0; j < s; ++j) v += Ainv.q[i * kMaxStages + j] * w[j];
      }
      out[(int64_t)i * nb + k] = v;
    }
  }
}

__global__ void k_bc_zero(int s, int64_t nb, const int64_t* __restrict__ idx,
                          double* __restrict__ X) {
  int64_t n = nb * s;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = q / s;
    int i = (int)(q - k * s);
    X[idx[k] * s + i] = 0.0;
  }
}

__global__ void k_bc_mask(int64_t nb, const int64_t* __restrict__ idx, uint8_t* __restrict__ mask) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nb;
       k += (int64_t)gridDim.x * blockDim.x)
    mask[idx[k]] = 1;
}

// Semilinear stacked residual (stage-derivative unknowns X):
//   U_c = u_c + dt (A X_c),  R_r,i = (M X)_r,i + kscale (K U)_r,i + (M g(U))_r,i - F_r,i
//   D_r,i = g'(U_r,i)
struct Poly {
  double c[8];
  int n;
};

__device__ __forceinline__ double poly_eval(const Poly& p, double x) {
  double acc = 0.0;
  for (int q = p.n - 1; q >= 0; --q) acc = acc * x + p.c[q];
  return acc;
}
__device__ __forceinline__ double poly_deriv(const Poly& p, double x) {
  double acc = 0.0;
  for (int q = p.n - 1; q >= 1; --q) acc = acc * x + q * p.c[q];
  return acc;
}

template <int S, bool MASK>
__global__ void __launch_bounds__(kBlock)
    k_semilinear_residual(int64_t m, const int* __restrict__ slice_ptr,
                          const int* __restrict__ sell_col, const double* __restrict__ mval,
                          const double* __restrict__ kval, const Mat8 A, double dt,
                          double kscale, const Poly g, const double* __restrict__ u,
                          const double* __restrict__ X, const double* __restrict__ F,
                          const uint8_t* __restrict__ mask, double* __restrict__ R,
                          double* __restrict__ D) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  // own-row stage states for the Jacobian weights
  {
    double x[S];
#pragma unroll
    for (int j = 0; j < S; ++j) x[j] = X[r * S + j];
    double ur = u[r];
#pragma unroll
    for (int i = 0; i < S; ++i) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) t += A.q[i * S + j] * x[j];
      D[r * S + i] = poly_deriv(g, ur + dt * t);
    }
  }
  if (MASK && mask[r]) {
#pragma unroll
    for (int i = 0; i < S; ++i) R[r * S + i] = 0.0;
    return;
  }
  int64_t s = r / kSlice;
  int lane = (int)(r % kSlice);
  int base = __ldg(slice_ptr + s), width = (__ldg(slice_ptr + s + 1) - base) / kSlice;
  double acc[S];
#pragma unroll
  for (int i = 0; i < S; ++i) acc[i] = 0.0;
  for (int k = 0; k < width; ++k) {
    int pos = base + k * kSlice + lane;
    int c = __ldg(sell_col + pos);
    double mv = __ldg(mval + pos), kv = __ldg(kval + pos);
    double x[S];
#pragma unroll
    for (int j = 0; j < S; ++j) x[j] = __ldg(X + (int64_t)c * S + j);
    double uc = __ldg(u + c);
#pragma unroll
    for (int i = 0; i < S; ++i) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) t += A.q[i * S + j] * x[j];
      double U = uc + dt * t;
      acc[i] += mv * x[i] + kscale * kv * U + mv * poly_eval(g, U);
    }
  }
#pragma unroll
  for (int i = 0; i < S; ++i) R[r * S + i] = acc[i] - (F ? F[r * S + i] : 0.0);
}

template <typename T>
static void load_mat(T& dst, const double* src, int s) {
  for (int q = 0; q < kMaxStages * kMaxStages; ++q) dst.q[q] = 0.0;
  if (src)
    for (int q = 0; q < s * s; ++q) dst.q[q] = src[q];
}

}  // namespace irk

using namespace irk;

#define IRK_STAGE_SWITCH(S_, CALL)                                            \
  switch (S_) {                                                               \
    case 1: { constexpr int SS = 1; CALL; } break;                             \
    case 2: { constexpr int SS = 2; CALL; } break;                             \
    case 3: { constexpr int SS = 3; CALL; } break;                             \
    case 4: { constexpr int SS = 4; CALL; } break;                             \
    case 5: { constexpr int SS = 5; CALL; } break;                             \
    case 6: { constexpr int SS = 6; CALL; } break;                             \
    case 7: { constexpr int SS = 7; CALL; } break;                             \
    case 8: { constexpr int SS = 8; CALL; } break;                             \
    default: break;                                                           \
  }
#define IRK_STAGE_SWITCH4(S_, CALL)                                           \
  switch (S_) {                                                               \
    case 1: { constexpr int SS = 1; CALL; } break;                             \
    case 2: { constexpr int SS = 2; CALL; } break;                             \
    case 3: { constexpr int SS = 3; CALL; } break;                             \
    case 4: { constexpr int SS = 4; CALL; } break;                             \
    default: break;                                                           \
  }

extern "C" {

int irk_stage_apply(irk_ctx* ctx, int s, const double* C1_host, const double* C2_host, double dt,
                    const irk_mat* M, const irk_mat* const* Ks, int nK,
                    const uint8_t* rowmask_dev, const double* Y_dev, double* Out_dev) {
  IRK_REQUIRE(ctx && C1_host && C2_host && M && Ks && Y_dev && Out_dev,
              "irk_stage_apply: NULL argument");
  IRK_REQUIRE(s >= 1 && s <= kMaxStages, "irk_stage_apply: 1 <= s <= %d", kMaxStages);
  IRK_REQUIRE(nK == 1 || nK == s, "irk_stage_apply: nK must be 1 or s");
  KPtrs kp{};
  for (int i = 0; i < nK; ++i) {
    IRK_REQUIRE(Ks[i] && Ks[i]->pat == M->pat,
                "irk_stage_apply: K blocks must share M's pattern (use irk_mat_union)");
    kp.k[i] = Ks[i]->val;
  }
  Coef2 cf{};
  for (int q = 0; q < s * s; ++q) {
    cf.c1[q] = C1_host[q];
    cf.c2[q] = C2_host[q];
  }
  const Pattern* P = M->pat;
  int64_t m = P->nrows;
  if (m == 0) return IRK_OK;
  unsigned g = (unsigned)((m + kBlock - 1) / kBlock);
  const bool per = nK > 1;
  const int mw = P->maxw;
#define IRK_LAUNCH_SA(PER, W)                                                             \
  IRK_STAGE_SWITCH(s, (k_stage_apply<SS, PER, W><<<g, kBlock, 0, ctx->stream>>>(          \
                          m, P->slice_ptr, P->sell_col, M->val, kp, cf, dt, rowmask_dev, \
                          Y_dev, Out_dev, P->ellw)))
  static const bool win_off = getenv("IRK_NO_WINDOW") != nullptr;
  static const bool std_off = getenv("IRK_NO_STD_WINDOW") != nullptr;
  // stencil patterns: precomputed window layout
  if (!per && !win_off && !std_off && s <= 4 && P->ellw > 0 &&
      (int)P->stencil.size() == P->ellw && (P->ellw == 7 || P->ellw == 15 || P->ellw == 3)) {
    StLayout SL;
    if (stencil_layout(P->stencil, SL)) {
      const size_t smem = (size_t)(kBlock / 32) * SL.total * (s % 2 == 0 ? s + 1 : s) *
                          sizeof(double);
      if (smem <= 96 * 1024) {
        const int64_t ns = P->nslices;
        const unsigned gw = (unsigned)((ns + kBlock / 32 - 1) / (kBlock / 32));
        static bool attr_done = false;
        if (!attr_done) {
          for (int ss = 1; ss <= 4; ++ss) {
#define IRK_STD_ATTR(W, NW)                                                                 \
  IRK_STAGE_SWITCH4(ss, (cudaFuncSetAttribute(k_stage_apply_std<SS, W, NW>,                 \
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                              96 * 1024)))
            IRK_STD_ATTR(3, 1) IRK_STD_ATTR(7, 3) IRK_STD_ATTR(15, 8)
#undef IRK_STD_ATTR
          }
          attr_done = true;
        }
#define IRK_LAUNCH_STD(W, NW)                                                                 \
  IRK_STAGE_SWITCH4(s, (k_stage_apply_std<SS, W, NW><<<gw, kBlock, smem, ctx->stream>>>(      \
                          m, ns, SL, P->sell_col, P->colhdr, M->val, kp.k[0], cf, dt,         \
                          rowmask_dev, Y_dev, Out_dev)))
        // window-lookup unrolled over NW >= SL.nwin windows (extra entries
        // repeat the last window's base, so they never match first)
        for (int w = SL.nwin; w < 16; ++w) {
          SL.wbase[w] = 1 << 30;
          SL.wstart[w] = 0;
        }
        // bulk-asynchronous tiles (k_stage_apply_bulk); env IRK_NO_BULK: the
        // per-warp window copies of k_stage_apply_std
        static const bool bulk_off = getenv("IRK_NO_BULK") != nullptr;
        // The 15-point 3D stencil: values direct (VD: only the row mask and
        // the 7 Y windows ride the bulk copies, the value slabs go straight
        // to registers), 4-slice tiles, 2-stage ring: 29 KB per stage, three
        // CTAs per SM.  With the value slabs staged too a stage takes 60 KB,
        // one 4-warp CTA per SM is resident and its compute phase bounds the
        // kernel.  Measured at config 3, s = 4 (profiles/r02/s5_k2vd.log,
        // s5_ncu_full.log): VD 52.4 us (0.97 of the copy peak in algorithmic
        // bytes), VD with 8-slice tiles 66.5, staged values 99 (4-slice, 2- or
        // 3-stage ring) / 88 (6-slice), per-warp copies (k_stage_apply_std)
        // 77.4 us.  IRK_BULK3 = std | staged | vd8 selects the others
        // (IRK_BULK3_KT = 4 or 6 for staged).
        static const char* b3 = getenv("IRK_BULK3");
        static const bool bulk3_off = b3 && !strcmp(b3, "std");
        static const int bulk3_kt = getenv("IRK_BULK3_KT") ? atoi(getenv("IRK_BULK3_KT")) : 4;
        static const int bulk3_vd = !b3 ? 4 : !strcmp(b3, "vd8") ? 8 : !strcmp(b3, "staged") ? 0 : 4;
        // 2D stencil: values direct for s >= 2 (config 2, s = 3: 30.3 -> 28.0 us;
        // neutral at 2048^2; s = 1 keeps the staged slabs, measured 0.80 of the
        // peak there; profiles/r02/s5_k2final.log).  IRK_BULK2 = vd | staged
        // forces one variant.
        static const char* b2 = getenv("IRK_BULK2");
        const bool bulk2_vd = b2 ? !strcmp(b2, "vd") : s >= 2;
        if (!bulk_off && (P->ellw == 7 || (P->ellw == 15 && !bulk3_off))) {
          const bool d3 = P->ellw == 15;
          const bool vd = d3 ? bulk3_vd != 0 : bulk2_vd;
          const int kT = !d3 ? 8 : vd ? bulk3_vd : (bulk3_kt == 6 ? 6 : 4);
          const int nst = vd ? 2 : (d3 && kT == 4 ? 3 : 2);
          BulkLayout BL;
          const int ymis = (int)(((uintptr_t)Y_dev & 15) / 8);
          if (bulk_layout(SL, P->ellw, s, kT, ymis, BL)) {
            const size_t sm =
                nst * ((vd ? (size_t)0 : (size_t)2 * kT * P->ellw * kSlice) + kT * kSlice / 8 +
                       (size_t)BL.rows_total * s) *
                sizeof(double);
            if (sm <= 200 * 1024) {
              const int64_t ntiles = (ns + kT - 1) / kT;
              if (!d3 && bulk2_vd)
                launch_bulk<7, 8, 2, true>(ctx, s, m, ns, ntiles, BL, sm, P, M->val, kp.k[0], cf, dt,
                                           rowmask_dev, Y_dev, Out_dev);
              else if (vd && kT == 8)
                launch_bulk<15, 8, 2, true>(ctx, s, m, ns, ntiles, BL, sm, P, M->val, kp.k[0], cf,
                                            dt, rowmask_dev, Y_dev, Out_dev);
              else if (vd)
                launch_bulk<15, 4, 2, true>(ctx, s, m, ns, ntiles, BL, sm, P, M->val, kp.k[0], cf,
                                            dt, rowmask_dev, Y_dev, Out_dev);
              else if (!d3)
                launch_bulk<7, 8, 2>(ctx, s, m, ns, ntiles, BL, sm, P, M->val, kp.k[0], cf, dt,
                                     rowmask_dev, Y_dev, Out_dev);
              else if (kT == 6)
                launch_bulk<15, 6, 2>(ctx, s, m, ns, ntiles, BL, sm, P, M->val, kp.k[0], cf, dt,
                                      rowmask_dev, Y_dev, Out_dev);
              else
                launch_bulk<15, 4, 3>(ctx, s, m, ns, ntiles, BL, sm, P, M->val, kp.k[0], cf, dt,
                                      rowmask_dev, Y_dev, Out_dev);
              IRK_CHECK_LAUNCH(ctx);
              return IRK_OK;
            }
          }
        }
        if (P->ellw == 7 && SL.nwin <= 3) {
          IRK_LAUNCH_STD(7, 3)
        } else if (P->ellw == 15 && SL.nwin <= 8) {
          IRK_LAUNCH_STD(15, 8)
        } else if (P->ellw == 3 && SL.nwin <= 1) {
          IRK_LAUNCH_STD(3, 1)
        } else {
          goto generic_window;
        }
#undef IRK_LAUNCH_STD
        IRK_CHECK_LAUNCH(ctx);
        return IRK_OK;
      }
    }
  }
generic_window:
  const int wrows = P->win_rows;
  const size_t wsmem = (size_t)(kBlock / 32) * wrows * (s % 2 == 0 ? s + 1 : s) * sizeof(double);
  constexpr size_t kWinSmemMax = 96 * 1024;
  if (!per && !win_off && s <= 4 && mw <= 16 && wrows > 0 && wsmem <= kWinSmemMax) {
    const int64_t ns = P->nslices;
    const unsigned gw = (unsigned)((ns + kBlock / 32 - 1) / (kBlock / 32));
#define IRK_LAUNCH_WIN(W)                                                                       \
  IRK_STAGE_SWITCH4(s, (k_stage_apply_win<SS, W><<<gw, kBlock, wsmem, ctx->stream>>>(            \
                          m, ns, P->slice_ptr, P->sell_col, P->colhdr, M->val, kp.k[0], cf, dt, \
                          rowmask_dev, Y_dev, Out_dev, P->ellw, wrows)))
    static bool attr_set = false;
    if (!attr_set) {
      for (int ss = 1; ss <= 4; ++ss) {
#define IRK_WIN_ATTR(W)                                                              \
  IRK_STAGE_SWITCH4(ss, (cudaFuncSetAttribute(k_stage_apply_win<SS, W>,              \
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                              (int)kWinSmemMax)))
        IRK_WIN_ATTR(4) IRK_WIN_ATTR(8) IRK_WIN_ATTR(10) IRK_WIN_ATTR(12) IRK_WIN_ATTR(16)
#undef IRK_WIN_ATTR
      }
      attr_set = true;
    }
    if (mw <= 4) {
      IRK_LAUNCH_WIN(4)
    } else if (mw <= 8) {
      IRK_LAUNCH_WIN(8)
    } else if (mw <= 10) {
      IRK_LAUNCH_WIN(10)
    } else if (mw <= 12) {
      IRK_LAUNCH_WIN(12)
    } else {
      IRK_LAUNCH_WIN(16)
    }
#undef IRK_LAUNCH_WIN
    IRK_CHECK_LAUNCH(ctx);
    return IRK_OK;
  }
  if (per) {
    IRK_LAUNCH_SA(true, 0)
  } else if (mw <= 8) {
    IRK_LAUNCH_SA(false, 8)
  } else if (mw <= 16) {
    IRK_LAUNCH_SA(false, 16)
  } else {
    IRK_LAUNCH_SA(false, 0)
  }
#undef IRK_LAUNCH_SA
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_stage_apply_semilinear(irk_ctx* ctx, int s, const double* C1_host, const double* C2_host,
                               double dt, const irk_mat* M, const irk_mat* K, double kscale,
                               const double* D_dev, const uint8_t* rowmask_dev,
                               const double* Y_dev, double* Out_dev) {
  IRK_REQUIRE(ctx && C1_host && C2_host && M && K && D_dev && Y_dev && Out_dev,
              "irk_stage_apply_semilinear: NULL argument");
  IRK_REQUIRE(s >= 1 && s <= kMaxStages, "irk_stage_apply_semilinear: bad s");
  IRK_REQUIRE(K->pat == M->pat, "irk_stage_apply_semilinear: M and K must share a pattern");
  Coef2 cf{};
  for (int q = 0; q < s * s; ++q) {
    cf.c1[q] = C1_host[q];
    cf.c2[q] = C2_host[q];
  }
  const Pattern* P = M->pat;
  int64_t m = P->nrows;
  if (m == 0) return IRK_OK;
  unsigned g = (unsigned)((m + kBlock - 1) / kBlock);
  IRK_STAGE_SWITCH(s, (k_stage_apply_semi<SS><<<g, kBlock, 0, ctx->stream>>>(
                          m, P->slice_ptr, P->sell_col, M->val, K->val, cf, dt, kscale, D_dev,
                          rowmask_dev, Y_dev, Out_dev)))
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_stage_mix(irk_ctx* ctx, int64_t m, int s_out, int s_in, const double* Q_host,
                  const double* X_dev, double* Y_dev) {
  IRK_REQUIRE(ctx && Q_host && X_dev && Y_dev, "irk_stage_mix: NULL argument");
  IRK_REQUIRE(s_out >= 1 && s_out <= kMaxStages && s_in >= 1 && s_in <= kMaxStages,
              "irk_stage_mix: bad stage counts");
  IRK_REQUIRE(s_in == s_out || X_dev != Y_dev, "irk_stage_mix: in place needs s_in == s_out");
  if (m == 0) return IRK_OK;
  Mat8 Q;
  for (int q = 0; q < kMaxStages * kMaxStages; ++q) Q.q[q] = 0.0;
  for (int i = 0; i < s_out; ++i)
    for (int j = 0; j < s_in; ++j) Q.q[i * kMaxStages + j] = Q_host[i * s_in + j];
  k_stage_mix<<<grid_for(ctx, m), kBlock, 0, ctx->stream>>>(m, s_out, s_in, Q, X_dev, Y_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_stage_couple(irk_ctx* ctx, int s, int i, const double* coef_host, const irk_mat* C,
                     const uint8_t* rowmask_dev, const double* R_dev, const double* X_dev,
                     double* out_dev, int64_t ld_out) {
  IRK_REQUIRE(ctx && coef_host && C && R_dev && X_dev && out_dev, "irk_stage_couple: NULL argument");
  IRK_REQUIRE(s >= 1 && s <= kMaxStages && i >= 0 && i < s, "irk_stage_couple: bad stage index");
  int64_t m = C->pat->nrows;
  if (m == 0) return IRK_OK;
  Mat8 cf;
  for (int q = 0; q < kMaxStages * kMaxStages; ++q) cf.q[q] = 0.0;
  for (int j = 0; j < s; ++j) cf.q[j] = coef_host[j];
  unsigned jm = 0;
  for (int j = 0; j < s; ++j)
    if (coef_host[j] != 0.0) jm |= 1u << j;
  const Pattern* P = C->pat;
  unsigned g = (unsigned)((m + kBlock - 1) / kBlock);
#define IRK_CPL(WW)                                                                          \
  IRK_STAGE_SWITCH(s, (k_stage_couple<SS, WW><<<g, kBlock, 0, ctx->stream>>>(                   \
                          m, i, P->slice_ptr, P->ellw, P->colhdr, P->sell_col, C->uval, C->val, \
                          cf, jm, rowmask_dev, R_dev, X_dev, out_dev, ld_out)))
  if (P->ellw == 7) {
    IRK_CPL(7)
  } else if (P->ellw == 15) {
    IRK_CPL(15)
  } else {
    IRK_CPL(0)
  }
#undef IRK_CPL
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_stage_rhs(irk_ctx* ctx, int64_t m, int s, double a, const irk_mat* B, const double* u_dev,
                  const double* G_host, const double* F_dev, double* Out_dev) {
  IRK_REQUIRE(ctx && Out_dev, "irk_stage_rhs: NULL argument");
  IRK_REQUIRE(s >= 1 && s <= kMaxStages, "irk_stage_rhs: bad s");
  IRK_REQUIRE(!B || (u_dev && B->pat->nrows == m), "irk_stage_rhs: B/u mismatch");
  if (!B && a == 0.0) u_dev = nullptr;
  IRK_REQUIRE(!F_dev || G_host, "irk_stage_rhs: F needs G");
  if (m == 0) return IRK_OK;
  Mat8 G;
  load_mat(G, G_host, s);
  unsigned g = (unsigned)((m + kBlock - 1) / kBlock);
  const int* sp = B ? B->pat->slice_ptr : nullptr;
  const int* sc = B ? B->pat->sell_col : nullptr;
  const int* ch = B ? B->pat->colhdr : nullptr;
  const int ew = B ? B->pat->ellw : 0;
  const double* bv = B ? B->val : nullptr;
  const double* ub = B ? B->uval : nullptr;
  IRK_STAGE_SWITCH(s, (k_stage_rhs<SS><<<g, kBlock, 0, ctx->stream>>>(m, sp, ew, ch, sc, ub, bv, a,
                                                                      u_dev, G, F_dev, Out_dev)))
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_stage_update(irk_ctx* ctx, int64_t m, int s, double a, const double* u_dev,
                     const double* w_host, int copy_stage, const double* X_dev,
                     double* u_next_dev) {
  IRK_REQUIRE(ctx && X_dev && u_next_dev, "irk_stage_update: NULL argument");
  IRK_REQUIRE(s >= 1 && s <= kMaxStages, "irk_stage_update: bad s");
  IRK_REQUIRE(copy_stage < s, "irk_stage_update: copy_stage out of range");
  IRK_REQUIRE(copy_stage >= 0 || (w_host && (a == 0.0 || u_dev)),
              "irk_stage_update: weights/u missing");
  if (m == 0) return IRK_OK;
  Mat8 w;
  for (int q = 0; q < kMaxStages * kMaxStages; ++q) w.q[q] = 0.0;
  if (w_host)
    for (int i = 0; i < s; ++i) w.q[i] = w_host[i];
  int g = grid_for(ctx, m);
  IRK_STAGE_SWITCH(s, (k_stage_update<SS><<<g, kBlock, 0, ctx->stream>>>(m, a, u_dev, w,
                                                                         copy_stage, X_dev,
                                                                         u_next_dev)))
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_stage_scale(irk_ctx* ctx, int64_t m, int s, const double* w_host, const double* v_dev,
                    const double* D_dev, double* out_dev) {
  IRK_REQUIRE(ctx && w_host && v_dev && out_dev, "irk_stage_scale: NULL argument");
  IRK_REQUIRE(s >= 1 && s <= kMaxStages, "irk_stage_scale: bad s");
  if (m == 0) return IRK_OK;
  Mat8 w;
  for (int q = 0; q < kMaxStages * kMaxStages; ++q) w.q[q] = 0.0;
  for (int i = 0; i < s; ++i) w.q[i] = w_host[i];
  k_stage_scale<<<grid_for(ctx, m * s), kBlock, 0, ctx->stream>>>(m, s, w, v_dev, D_dev, out_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_stage_get(irk_ctx* ctx, int64_t m, int s, int i, const double* X_dev, double* x_dev) {
  IRK_REQUIRE(ctx && X_dev && x_dev && i >= 0 && i < s, "irk_stage_get: bad argument");
  if (m == 0) return IRK_OK;
  k_stage_get<<<grid_for(ctx, m), kBlock, 0, ctx->stream>>>(m, s, i, X_dev, x_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_stage_set(irk_ctx* ctx, int64_t m, int s, int i, const double* x_dev, double* X_dev) {
  IRK_REQUIRE(ctx && X_dev && x_dev && i >= 0 && i < s, "irk_stage_set: bad argument");
  if (m == 0) return IRK_OK;
  k_stage_set<<<grid_for(ctx, m), kBlock, 0, ctx->stream>>>(m, s, i, x_dev, X_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_to_interleaved(irk_ctx* ctx, int64_t m, int s, const double* stage_major_dev,
                       double* interleaved_dev) {
  IRK_REQUIRE(ctx && stage_major_dev && interleaved_dev && s >= 1,
              "irk_to_interleaved: bad argument");
  if (m == 0) return IRK_OK;
  k_to_interleaved<<<grid_for(ctx, m * s), kBlock, 0, ctx->stream>>>(m, s, stage_major_dev,
                                                                    interleaved_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_to_stage_major(irk_ctx* ctx, int64_t m, int s, const double* interleaved_dev,
                       double* stage_major_dev) {
  IRK_REQUIRE(ctx && stage_major_dev && interleaved_dev && s >= 1,
              "irk_to_stage_major: bad argument");
  if (m == 0) return IRK_OK;
  k_to_stage_major<<<grid_for(ctx, m * s), kBlock, 0, ctx->stream>>>(m, s, interleaved_dev,
                                                                    stage_major_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_bc_scatter(irk_ctx* ctx, int s, int64_t nb, const int64_t* idx_dev, const double* V_dev,
                   double* X_dev) {
  IRK_REQUIRE(ctx && s >= 1, "irk_bc_scatter: bad argument");
  if (nb == 0) return IRK_OK;
  k_bc_scatter<<<grid_for(ctx, nb * s), kBlock, 0, ctx->stream>>>(s, nb, idx_dev, V_dev, X_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_bc_gather(irk_ctx* ctx, int64_t nb, const int64_t* idx_dev, const double* x_dev,
                  double* v_dev) {
  IRK_REQUIRE(ctx, "irk_bc_gather: bad argument");
  if (nb == 0) return IRK_OK;
  k_bc_gather<<<grid_for(ctx, nb), kBlock, 0, ctx->stream>>>(nb, idx_dev, x_dev, v_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_bc_dae_values(irk_ctx* ctx, int s, int64_t nb, const int64_t* idx_dev,
                      const double* G_dev, const double* u_dev, double dt,
                      const double* Ainv_host, double* out_dev) {
  IRK_REQUIRE(ctx && s >= 1 && s <= kMaxStages && dt != 0.0, "irk_bc_dae_values: bad argument");
  if (nb == 0) return IRK_OK;
  Mat8 Ai{};
  if (Ainv_host)
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) Ai.q[i * kMaxStages + j] = Ainv_host[i * s + j];
  k_bc_dae<<<grid_for(ctx, nb), kBlock, 0, ctx->stream>>>(s, nb, idx_dev, G_dev, u_dev, dt, Ai,
                                                          Ainv_host ? 1 : 0, out_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_bc_zero(irk_ctx* ctx, int s, int64_t nb, const int64_t* idx_dev, double* X_dev) {
  IRK_REQUIRE(ctx && s >= 1, "irk_bc_zero: bad argument");
  if (nb == 0) return IRK_OK;
  k_bc_zero<<<grid_for(ctx, nb * s), kBlock, 0, ctx->stream>>>(s, nb, idx_dev, X_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_bc_mask(irk_ctx* ctx, int64_t m, int64_t nb, const int64_t* idx_dev, uint8_t* mask_dev) {
  IRK_REQUIRE(ctx && mask_dev, "irk_bc_mask: bad argument");
  if (m) IRK_CUDA(cudaMemsetAsync(mask_dev, 0, m, ctx->stream));
  if (nb == 0) return IRK_OK;
  k_bc_mask<<<grid_for(ctx, nb), kBlock, 0, ctx->stream>>>(nb, idx_dev, mask_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_semilinear_residual(irk_ctx* ctx, int s, const double* A_host, double dt,
                            const irk_mat* M, const irk_mat* K, double kscale, int ncoef,
                            const double* coef_host, const double* u_dev, const double* X_dev,
                            const double* F_dev, const uint8_t* rowmask_dev, double* R_dev,
                            double* D_dev) {
  IRK_REQUIRE(ctx && A_host && M && K && u_dev && X_dev && R_dev && D_dev,
              "irk_semilinear_residual: NULL argument");
  IRK_REQUIRE(s >= 1 && s <= kMaxStages, "irk_semilinear_residual: bad s");
  IRK_REQUIRE(ncoef >= 0 && ncoef <= 8 && (ncoef == 0 || coef_host),
              "irk_semilinear_residual: 0 <= ncoef <= 8");
  IRK_REQUIRE(K->pat == M->pat, "irk_semilinear_residual: M and K must share a pattern");
  Mat8 A;
  load_mat(A, A_host, s);
  Poly g{};
  g.n = ncoef;
  for (int q = 0; q < ncoef; ++q) g.c[q] = coef_host[q];
  const Pattern* P = M->pat;
  int64_t m = P->nrows;
  if (m == 0) return IRK_OK;
  unsigned gr = (unsigned)((m + kBlock - 1) / kBlock);
  if (rowmask_dev) {
    IRK_STAGE_SWITCH(s, (k_semilinear_residual<SS, true><<<gr, kBlock, 0, ctx->stream>>>(
                            m, P->slice_ptr, P->sell_col, M->val, K->val, A, dt, kscale, g,
                            u_dev, X_dev, F_dev, rowmask_dev, R_dev, D_dev)))
  } else {
    IRK_STAGE_SWITCH(s, (k_semilinear_residual<SS, false><<<gr, kBlock, 0, ctx->stream>>>(
                            m, P->slice_ptr, P->sell_col, M->val, K->val, A, dt, kscale, g,
                            u_dev, X_dev, F_dev, nullptr, R_dev, D_dev)))
  }
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

}  // extern "C"
