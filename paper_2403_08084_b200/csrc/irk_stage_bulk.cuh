// K2 on stencil-aligned ELL patterns with bulk-asynchronous tile movement
// (cp.async.bulk global -> shared, completion on an mbarrier), included by
// irk_stage.cu after k_stage_apply_std.
//
// A CTA (kT warps) owns a tile of kT consecutive SELL slices (kT*32 stage
// rows) at a time and walks the tiles t = blockIdx.x, + gridDim.x, ...  The
// tile's operands are contiguous ranges of global memory:
//   * the M and K value slabs of the kT slices (ELL-32: kT*W*32 doubles each),
//   * per stencil window w (contiguous runs of stencil offsets), the stage
//     rows [R0 + wstart_w, R0 + wstart_w + len_w + (kT-1)*32) of Y
//     (interleaved m x S: one contiguous range of rows*S doubles),
// so one elected thread moves the whole tile with 2 + nwin bulk copies into
// one stage of an NST-stage ring (2 on the 7-point 2D stencil, 3 on the
// 15-point 3D one: enough bytes in flight per SM with one resident CTA), and
// the copies of the next NST - 1 tiles are in flight while the warps compute
// tile t (warp = slice, lane = row; every
// slot's stage values come from the window buffer, values from the slabs).
// The DRAM stream is the same as k_stage_apply_std's (values once, Y once
// plus L2-served window overlap, Out once); what changes is that no warp
// waits on its own loads and no register staging / shared stores are spent
// on the copy.  Tiles whose windows leave [0, m) (the first and last few)
// take the per-entry gather path from global memory.

struct BulkLayout {
  int nwin, rows_total;      // buffer rows of one stage
  int wsrc[16];              // window w: first global row relative to R0 (aligned down)
  int wrows[16];             // rows copied (S * rows * 8 bytes is a multiple of 16)
  int wbuf[16];              // first buffer row of window w
  int krow[16];              // buffer row of slot k for slice 0, lane 0
  int sd[16];                // stencil offsets (slot k of a stencil row: row + sd[k])
  int kc;                    // the centre slot (offset 0)
  int lo, hi;                // a tile is interior when R0 + lo >= 0 && R0 + hi <= m
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// VD (values direct): the M and K value slabs are NOT staged (each value is
// used once by one lane: coalesced loads into registers, all issued before
// the mbarrier wait); only the row mask and the Y windows ride the bulk
// copies.  Halves the ring stage on the 15-point 3D stencil (29 instead of
// 60 KB per 4-slice tile), so three CTAs per SM are resident instead of one.
template <int S, int W, int KT, int NST, bool VD = false>
__global__ void __launch_bounds__(KT * 32)
    k_stage_apply_bulk(int64_t m, int64_t nslices, int64_t ntiles, const BulkLayout BL,
                       const int* __restrict__ sell_col,
                       const int* __restrict__ colhdr, const double* __restrict__ mval,
                       const double* __restrict__ kval, const Coef2 cf, double dt,
                       const uint8_t* __restrict__ mask, const double* __restrict__ Y,
                       double* __restrict__ Out) {
  // KT warps: one per slice of the tile
  extern __shared__ __align__(128) double bsm[];
  __shared__ __align__(8) uint64_t bar[NST];  // NST pipeline stages (tiles in flight + 1)
  constexpr int VALG = KT * W * kSlice;  // doubles per value slab of a tile
  constexpr int VAL = VD ? 0 : VALG;     // ... staged in shared memory
  constexpr int MSK = KT * kSlice / 8;   // doubles holding the tile's row-mask bytes
  const int stage_doubles = 2 * VAL + MSK + BL.rows_total * S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NST; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto interior = [&](int64_t t) {
    const int64_t R0 = t * KT * kSlice;
    return R0 + BL.lo >= 0 && R0 + BL.hi <= m && (t + 1) * KT <= nslices;
  };
  // one elected thread issues the tile's bulk copies into stage st
  auto issue = [&](int64_t t, int st) {
    double* base = bsm + (size_t)st * stage_doubles;
    const int64_t R0 = t * KT * kSlice;
    unsigned bytes = 2u * VAL * (unsigned)sizeof(double) + (mask ? MSK * (unsigned)sizeof(double) : 0u);
    for (int w = 0; w < BL.nwin; ++w) bytes += (unsigned)BL.wrows[w] * S * sizeof(double);
    mbar_expect_tx(&bar[st], bytes);
    if constexpr (!VD) {
      const size_t v0 = (size_t)t * VALG;
      bulk_g2s(base, mval + v0, VAL * sizeof(double), &bar[st]);
      bulk_g2s(base + VAL, kval + v0, VAL * sizeof(double), &bar[st]);
    }
    if (mask) bulk_g2s(base + 2 * VAL, mask + R0, MSK * sizeof(double), &bar[st]);
    double* yb = base + 2 * VAL + MSK;
    for (int w = 0; w < BL.nwin; ++w)
      bulk_g2s(yb + (size_t)BL.wbuf[w] * S, Y + (R0 + BL.wsrc[w]) * S,
               (unsigned)BL.wrows[w] * S * sizeof(double), &bar[st]);
  };
  int64_t t = blockIdx.x;
  // bit st of pend: stage st holds (or is receiving) a tile; bit st of ph:
  // the mbarrier phase to wait for
  unsigned pend = 0u, ph = 0u;
#pragma unroll
  for (int i = 0; i < NST; ++i) {
    const int64_t ti = t + (int64_t)i * gridDim.x;
    if (ti < ntiles && interior(ti)) {
      pend |= 1u << i;
      if (threadIdx.x == 0) issue(ti, i);
    }
  }
  for (int st = 0; t < ntiles; t += gridDim.x, st = (st + 1 == NST ? 0 : st + 1)) {
    const int64_t sl = t * KT + warp;
    const int64_t r0 = sl * kSlice, r = r0 + lane;
    bool flagged = false;
    double a[S], b[S], yc[S];
#pragma unroll
    for (int q = 0; q < S; ++q) a[q] = b[q] = yc[q] = 0.0;
    bool done_row = false;
    if ((pend >> st) & 1u) {
      // VD: this lane's values of the slice straight from global memory
      double gm[VD ? W : 1], gk[VD ? W : 1];
      if constexpr (VD) {
        const size_t g0 = (size_t)sl * W * kSlice + lane;
#pragma unroll
        for (int k = 0; k < W; ++k) {
          gm[k] = __ldg(mval + g0 + k * kSlice);
          gk[k] = __ldg(kval + g0 + k * kSlice);
        }
      }
      mbar_wait(&bar[st], (ph >> st) & 1u);
      ph ^= 1u << st;
      const double* base = bsm + (size_t)st * stage_doubles;
      const double* mv = VD ? gm : base + warp * W * kSlice + lane;
      const double* kv = VD ? gk : base + VAL + warp * W * kSlice + lane;
      constexpr int VS = VD ? 1 : kSlice;  // stride of slot k in mv / kv
      const double* yb = base + 2 * VAL + MSK + (size_t)(warp * kSlice + lane) * S;
      if (mask)
        flagged = reinterpret_cast<const uint8_t*>(base + 2 * VAL)[warp * kSlice + lane] != 0;
      const int d = lane < W ? __ldg(colhdr + sl * W + lane) : 0;
      const bool std_slice = __all_sync(0xffffffffu, lane >= W || d == BL.sd[lane < W ? lane : 0]);
      if (std_slice) {
        // Even S: a row of the window buffer is S*8 bytes (a bulk copy cannot
        // pad it), so lanes reading stage q of consecutive rows would hit the
        // same banks 2 (S = 2) or 4 (S = 4) at a time.  Lane l reads its
        // stages rotated by rot(l) instead (register q holds stage
        // (q + rot) % S): the 16 lanes of a 64-bit shared-load phase then
        // cover 16 distinct bank pairs.  The sums are un-rotated below.
        constexpr bool ROT = S % 2 == 0;
        const int rot = ROT ? (S == 4 ? (lane >> 2) & 3 : (lane >> 3) & 1) : 0;
        const double* yq[S];
#pragma unroll
        for (int q = 0; q < S; ++q) yq[q] = yb + (ROT ? ((q + rot) & (S - 1)) : q);
#pragma unroll
        for (int k = 0; k < W; ++k) {
          const double mk = mv[k * VS], kk = kv[k * VS];
          const int ko = BL.krow[k] * S;
#pragma unroll
          for (int q = 0; q < S; ++q) {
            const double y = yq[q][ko];
            a[q] += mk * y;
            b[q] += kk * y;
          }
        }
        const int kco = BL.krow[BL.kc] * S;
#pragma unroll
        for (int q = 0; q < S; ++q) yc[q] = yq[q][kco];
        if constexpr (ROT) {
          // register q holds stage (q + rot) % S: rotate right by rot
#pragma unroll
          for (int sh = 1; sh < S; sh <<= 1) {
            if (rot & sh) {
              double ta[S], tb[S], tc[S];
#pragma unroll
              for (int q = 0; q < S; ++q) {
                ta[(q + sh) & (S - 1)] = a[q];
                tb[(q + sh) & (S - 1)] = b[q];
                tc[(q + sh) & (S - 1)] = yc[q];
              }
#pragma unroll
              for (int q = 0; q < S; ++q) {
                a[q] = ta[q];
                b[q] = tb[q];
                yc[q] = tc[q];
              }
            }
          }
        }
        done_row = true;
      } else if (r < m) {
#pragma unroll
        for (int k = 0; k < W; ++k) {
          const int c = sell_col_at(colhdr, sell_col, (int)(sl * W + k),
                                    (int)(sl * kSlice * W + k * kSlice + lane), r);
          const double mk = mv[k * VS], kk = kv[k * VS];
#pragma unroll
          for (int q = 0; q < S; ++q) {
            const double y = __ldg(Y + (int64_t)c * S + q);
            a[q] += mk * y;
            b[q] += kk * y;
          }
        }
      }
    } else if (sl < nslices && r < m) {
      // boundary tile: per-entry gathers from global memory
      flagged = mask && mask[r];
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int pos = (int)(sl * kSlice * W + k * kSlice + lane);
        const int c = sell_col_at(colhdr, sell_col, (int)(sl * W + k), pos, r);
        const double mk = __ldg(mval + pos), kk = __ldg(kval + pos);
#pragma unroll
        for (int q = 0; q < S; ++q) {
          const double y = __ldg(Y + (int64_t)c * S + q);
          a[q] += mk * y;
          b[q] += kk * y;
        }
      }
    }
    if (r < m && sl < nslices) {
      if (flagged && !done_row) {
#pragma unroll
        for (int q = 0; q < S; ++q) yc[q] = Y[r * S + q];
      }
#pragma unroll
      for (int q = 0; q < S; ++q) {
        double o = 0.0, tt = 0.0;
#pragma unroll
        for (int j = 0; j < S; ++j) {
          o += cf.c1[q * S + j] * a[j];
          tt += cf.c2[q * S + j] * b[j];
        }
        Out[r * S + q] = flagged ? yc[q] : o + dt * tt;
      }
    }
    // every warp is done with stage st: refill it with the tile after next
    __syncthreads();
    const int64_t tn = t + NST * (int64_t)gridDim.x;
    const bool more = tn < ntiles && interior(tn);
    if (threadIdx.x == 0 && more) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(tn, st);
    }
    pend = more ? (pend | (1u << st)) : (pend & ~(1u << st));
  }
}

// host: bulk layout of a stencil (its StLayout windows) for tiles of kT
// slices.  ymis = (Y address mod 16) / 8: the global source of every bulk
// copy must be 16-byte aligned (Krylov basis vectors of odd length start
// 8 bytes off), so windows start on rows of the matching parity (s odd);
// with s even no row shift can fix a misaligned Y (false: the caller falls
// back to the per-warp copies).
static bool bulk_layout(const StLayout& SL, int W, int s, int kT, int ymis, BulkLayout& B) {
  if (s % 2 == 0 && ymis) return false;
  B = BulkLayout{};
  B.nwin = SL.nwin;
  B.kc = -1;
  int rows = 0;
  B.lo = 1 << 30;
  B.hi = -(1 << 30);
  const int tile_rows = kT * kSlice;
  for (int w = 0; w < SL.nwin; ++w) {
    const int len = SL.wend[w] - SL.wbase[w] + tile_rows - kSlice;  // rows of the tile window
    int src = SL.wstart[w];
    int sh = 0;
    if (s % 2 == 1 && ((src - ymis) & 1)) {  // 16-byte aligned source row
      src -= 1;
      sh = 1;
    }
    int cnt = len + sh;
    if (s % 2 == 1 && (cnt & 1)) cnt += 1;  // byte count a multiple of 16
    B.wsrc[w] = src;
    B.wrows[w] = cnt;
    B.wbuf[w] = rows;
    rows += cnt;
    B.lo = std::min(B.lo, src);
    B.hi = std::max(B.hi, src + cnt);
  }
  B.rows_total = rows;
  for (int k = 0; k < W; ++k) {
    int w = -1;
    for (int v = 0; v < SL.nwin; ++v)
      if (SL.srow[k] >= SL.wbase[v] && SL.srow[k] < SL.wend[v]) w = v;
    if (w < 0) return false;
    B.krow[k] = B.wbuf[w] + SL.sd[k] - B.wsrc[w];
    B.sd[k] = SL.sd[k];
    if (SL.sd[k] == 0) B.kc = k;
  }
  return B.kc >= 0;
}
