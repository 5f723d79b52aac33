// Fast sine-transform (DST-I) preconditioner for the 2D grid blocks
// alpha M + beta K with the full-boundary Dirichlet set.
//
// The block's interior operator is ONE 3x3 stencil c[dy][dx] (extracted from
// the assembled matrix and verified against every row by the structured
// multigrid setup, irk_mg.cu k_mg2_row_stencil / k_mg2_verify).  Its
// reflection-symmetrised copy
//   s00 = c00,  s10 = (c[1][0] + c[1][2]) / 2,  s01 = (c[0][1] + c[2][1]) / 2,
//   s11 = (c[0][0] + c[0][2] + c[2][0] + c[2][2]) / 4
// is diagonalised by the 2D sine basis sin(pi j k / N) sin(pi i l / N):
//   lambda(k, l) = s00 + 2 s10 cos(pi k/N) + 2 s01 cos(pi l/N)
//                  + 4 s11 cos(pi k/N) cos(pi l/N),
// so  B_s^-1 = (2/N)^2 S_x S_y Lambda^-1 S_y S_x  (S = DST-I, S S = N/2 I).
// B - B_s only moves the P1 diagonal-edge coupling (weight h^2/12 of the
// mass matrix) between the two diagonals, so the spectrum of B_s^-1 B lies
// in [1 - eps, 1 + eps] with eps ~ h^2 / (12 |beta / alpha|) (1e-4 .. 1e-5 on
// the 1024^2 / 2048^2 workloads): CG reaches 1e-6 in ~2 and 1e-12 in ~3-4
// iterations instead of ~5.5 / ~9 multigrid-PCG ones.  Boundary rows are
// identity (z = r there).
//
// DST-I of length N-1 through a complex FFT of length L = 2N of the odd
// extension y = (0, x_1..x_{N-1}, 0, -x_{N-1}..-x_1):  Y_k = -2i S_k.  Two
// real sequences a, b share one FFT (y = a + i b):  S_a = -Im Y / 2,
// S_b = Re Y / 2.  The FFT runs in shared memory: Stockham autosort passes
// of radix 8 (one radix-2/4 pass for the remainder), each thread holding its
// radix-R butterfly in registers; one twiddle table e^{-2 pi i q / L}.
//
// Three kernels per application (N a power of two, 32 <= N <= 2048):
//   k_dst_rows<L, false>  rows of r      -> T (row DSTs, T has row stride N)
//   k_dst_cols<L>         columns of T   -> column DST, scale (2/N)^2/lambda,
//                                           column DST, back to T (4 columns
//                                           per CTA: one 32-byte sector per row)
//   k_dst_rows<L, true>   rows of T      -> z (row DSTs; boundary z = r)
// Each reads and writes the grid once (L2-resident at these sizes).
#pragma once

namespace irk {

struct DstStencil {
  double s00, s10, s01, s11;
};

__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// (-i) z
__device__ __forceinline__ double2 c_mi(double2 a) { return make_double2(a.y, -a.x); }

// in-register forward DFTs (e^{-2 pi i j k / R}), natural order in and out
__device__ __forceinline__ void dft2(double2* v) {
  const double2 t = v[0];
  v[0] = c_add(t, v[1]);
  v[1] = c_sub(t, v[1]);
}
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 t0 = c_add(x0, x2), t1 = c_sub(x0, x2);
  const double2 t2 = c_add(x1, x3), t3 = c_mi(c_sub(x1, x3));
  x0 = c_add(t0, t2);
  x2 = c_sub(t0, t2);
  x1 = c_add(t1, t3);
  x3 = c_sub(t1, t3);
}
__device__ __forceinline__ void dft8(double2* v) {
  double2 a0 = v[0], a1 = v[2], a2 = v[4], a3 = v[6];
  double2 b0 = v[1], b1 = v[3], b2 = v[5], b3 = v[7];
  dft4(a0, a1, a2, a3);
  dft4(b0, b1, b2, b3);
  constexpr double r = 0.70710678118654752440;
  // w8^1 = (1 - i)/sqrt2, w8^2 = -i, w8^3 = (-1 - i)/sqrt2
  const double2 w1 = make_double2(r * (b1.x + b1.y), r * (b1.y - b1.x));
  const double2 w2 = c_mi(b2);
  const double2 w3 = make_double2(r * (b3.y - b3.x), -r * (b3.x + b3.y));
  v[0] = c_add(a0, b0);
  v[4] = c_sub(a0, b0);
  v[1] = c_add(a1, w1);
  v[5] = c_sub(a1, w1);
  v[2] = c_add(a2, w2);
  v[6] = c_sub(a2, w2);
  v[3] = c_add(a3, w3);
  v[7] = c_sub(a3, w3);
}

// Shared-memory layout of an FFT buffer: element i lives at fpad(i) =
// i + i / 8 (one 16-byte pad per 8 elements).  A Stockham pass writes its
// radix-R outputs at stride Ns elements; unpadded, the strided 16-byte
// stores of the first passes (Ns = 1: lane stride 8 elements = 128 bytes)
// fall on the same 4 banks (32-way conflict).  With the pad the 8 lanes of a
// quarter-warp phase cover 8 distinct bank quads in every pass, and the
// unit-stride reads stay conflict-free.  A buffer of L elements takes
// fpad_len(L) = L + L / 8 elements.
__host__ __device__ constexpr int fpad(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int fpad_len(int L) { return L + (L >> 3); }

// One Stockham pass of radix R, Ns = the product of the earlier radices
// (compile time), over the L-point sequence in buf (in place: every thread
// first reads all its butterflies, then the block syncs, then writes), NT
// threads of the calling group (tid in [0, NT)).  Twiddles: ONE table load
// w = e^{-2 pi i k / (Ns R)} per butterfly, its powers w^2 .. w^{R-1} by
// complex multiplications (the R-1 scattered 16-byte loads per butterfly
// they replace were the kernels' bottleneck: 7 uncoalesced requests per
// thread and pass).
// TL: length of the twiddle table e^{-2 pi i q / TL} (a multiple of L).
template <int L, int R, int NT, int NS, int TL = L>
__device__ __forceinline__ void fft_pass(double2* buf, const double2* __restrict__ tw, int tid) {
  constexpr int ITEMS = L / R / NT;
  static_assert(ITEMS >= 1 && (L / R) % NT == 0, "fft_pass: bad thread count");
  double2 v[ITEMS][R];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int j = tid + it * NT;
    const int k = j % NS;
#pragma unroll
    for (int r = 0; r < R; ++r) v[it][r] = buf[fpad(j + r * (L / R))];
    if constexpr (NS > 1) {
      const double2 w1 = __ldg(tw + k * (TL / (NS * R)));
      if constexpr (R == 2) {
        v[it][1] = c_mul(v[it][1], w1);
      } else {
        const double2 w2 = c_mul(w1, w1), w3 = c_mul(w2, w1);
        v[it][1] = c_mul(v[it][1], w1);
        v[it][2] = c_mul(v[it][2], w2);
        v[it][3] = c_mul(v[it][3], w3);
        if constexpr (R == 8) {
          const double2 w4 = c_mul(w2, w2), w5 = c_mul(w4, w1), w6 = c_mul(w3, w3),
                        w7 = c_mul(w4, w3);
          v[it][4] = c_mul(v[it][4], w4);
          v[it][5] = c_mul(v[it][5], w5);
          v[it][6] = c_mul(v[it][6], w6);
          v[it][7] = c_mul(v[it][7], w7);
        }
      }
    }
    if constexpr (R == 8) dft8(v[it]);
    else if constexpr (R == 4) dft4(v[it][0], v[it][1], v[it][2], v[it][3]);
    else dft2(v[it]);
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int j = tid + it * NT;
    const int k = j % NS;
    const int base = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[fpad(base + r * NS)] = v[it][r];
  }
  __syncthreads();
}

// L / (the largest power of 8 dividing L): the last pass's radix (1: none)
__host__ __device__ constexpr int fft_rem(int L) { return L % 8 == 0 ? fft_rem(L / 8) : L; }

// Forward FFT of L points (power of two, 16 <= L <= 4096) in buf (padded
// layout): radix-8 passes, then one radix-4 or radix-2 pass for the rest.
template <int L, int NT, int NS = 1, int TL = L>
__device__ __forceinline__ void fft_smem(double2* buf, const double2* __restrict__ tw, int tid) {
  if constexpr (NS * 8 <= L) {
    fft_pass<L, 8, NT, NS, TL>(buf, tw, tid);
    fft_smem<L, NT, NS * 8, TL>(buf, tw, tid);
  } else if constexpr (L / NS == 4) {
    fft_pass<L, 4, NT, NS, TL>(buf, tw, tid);
  } else if constexpr (L / NS == 2) {
    fft_pass<L, 2, NT, NS, TL>(buf, tw, tid);
  }
}

#ifdef IRK_DST_2D  // the 2D kernels (irk_mg.cu, after irk_inner.cuh: SkipCtl, cg_skip_pred)
// Row DSTs.  Forward (INV = false): rows gy = 1..N-1 of the grid vector src
// (row stride n1 = N + 1) -> T (row stride N, column k = 1..N-1, column 0
// zero).  Inverse (INV = true): rows of T -> z (row stride n1), the boundary
// of z copied from r.  CTA b takes rows 1 + 2b and 2 + 2b (one complex FFT).
//
// Fused CG (SkipCtl / rz_part, blocks of at least kBlock threads): the
// forward kernel takes the skip decision of k_cg_skip itself (every CTA
// reduces the update kernel's ||r||^2 partials in reduce_partials' order and
// CTA 0 publishes it for the other transform kernels); the inverse kernel
// writes one r.z partial per CTA (rz_part[blockIdx.x]) of the rows it
// writes, so k_cg_dot_rz is not launched.
template <int NT>
__device__ __forceinline__ double dst_reduce_rr(const double* part, int G) {
  // reduce_partials' order (kBlock threads, 4 strided partials each, warp
  // trees, warps in order) on a block of NT threads: NT >= kBlock uses its
  // first kBlock threads, NT = kBlock / 2 gives every thread two of the
  // kBlock virtual threads (t and t + NT: virtual warps w and w + NT / 32)
  static_assert(NT >= kBlock || 2 * NT == kBlock, "dst_reduce_rr: block size");
  constexpr int VT = NT >= kBlock ? 1 : 2;
  __shared__ double pred[kBlock / 32];
  __shared__ double tot;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < kBlock) {
#pragma unroll
    for (int q = 0; q < VT; ++q) {
      const int vt = threadIdx.x + q * NT;
      double v = 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int b = vt + c * kBlock;
        if (b < G) v += __ldcg(part + b);
      }
      v = warp_sum(v);
      if (lane == 0) pred[warp + q * (NT / 32)] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) t += pred[w];
    tot = t;
  }
  __syncthreads();
  return tot;
}

template <int L, bool INV>
__global__ void __launch_bounds__(L / 8)
    k_dst_rows(int N, const double* __restrict__ src, double* __restrict__ dst,
               const double* __restrict__ r, const double2* __restrict__ tw, const int* stop,
               SkipCtl sk, double* __restrict__ rz_part) {
  IRK_PDL_ENTER();
  constexpr int NT = L / 8;
  if constexpr (!INV && NT >= kBlock) {
    if (sk.st) {
      const double rr = dst_reduce_rr<NT>(sk.rr, sk.G);
      const bool skip = cg_skip_pred<double>(sk.st, rr, sk.maxit);
      if (blockIdx.x == 0 && threadIdx.x == 0) sk.st->skip = skip ? 1 : 0;
      if (skip) return;
      stop = nullptr;
    }
  }
  if (stop && *stop) return;
  extern __shared__ double2 dst_buf[];
  double2* buf = dst_buf;
  const int n1 = N + 1;
  const int ra = 1 + 2 * blockIdx.x, rb = ra + 1;
  const bool hb = rb <= N - 1;
  const int sstride = INV ? N : n1;
  const double* sa = src + (size_t)ra * sstride;
  const double* sb = src + (size_t)rb * sstride;
  // INV: the r values of this thread's output points (boundary columns are
  // identity rows, interior ones enter r.z), loaded before the transform so
  // their latency hides behind it
  constexpr int KIT = (L / 2) / NT + 1;
  double pra[INV ? KIT : 1], prb[INV ? KIT : 1];
  if constexpr (INV) {
#pragma unroll
    for (int i = 0; i < KIT; ++i) {
      const int k = threadIdx.x + i * NT;
      pra[i] = k <= N ? r[(size_t)ra * n1 + k] : 0.0;
      prb[i] = (hb && k <= N) ? r[(size_t)rb * n1 + k] : 0.0;
    }
  }
  for (int j = threadIdx.x; j <= N; j += NT) {
    double2 y = make_double2(0.0, 0.0);
    if (j >= 1 && j <= N - 1) y = make_double2(sa[j], hb ? sb[j] : 0.0);
    buf[fpad(j)] = y;
    if (j >= 1 && j <= N - 1) buf[fpad(L - j)] = make_double2(-y.x, -y.y);
  }
  __syncthreads();
  fft_smem<L, NT>(buf, tw, threadIdx.x);
  const int dstride = INV ? n1 : N;
  double* da = dst + (size_t)ra * dstride;
  double* db = dst + (size_t)rb * dstride;
  double rz = 0.0;  // r.z of the points this thread writes (INV, fused CG)
  const bool want_rz = INV && rz_part != nullptr;
#pragma unroll
  for (int i = 0; i < KIT; ++i) {
    const int k = threadIdx.x + i * NT;
    if (k > N) break;
    if (k >= 1 && k <= N - 1) {
      const double2 Y = buf[fpad(k)];
      const double za = -0.5 * Y.y, zb = 0.5 * Y.x;
      da[k] = za;
      if (hb) db[k] = zb;
      if constexpr (INV) rz += pra[i] * za + prb[i] * zb;  // prb = 0 without row b
    } else if constexpr (INV) {
      // boundary columns x = 0, x = N of these rows: identity rows
      da[k] = pra[i];
      if (hb) db[k] = prb[i];
      rz += pra[i] * pra[i] + prb[i] * prb[i];
    } else if (k == 0) {
      da[0] = 0.0;
      if (hb) db[0] = 0.0;
    }
  }
  if (INV) {
    // boundary rows y = 0 (first CTA) and y = N (last CTA): identity rows
    if (blockIdx.x == 0)
      for (int k = threadIdx.x; k <= N; k += NT) {
        const double v = r[k];
        dst[k] = v;
        rz += v * v;
      }
    if (blockIdx.x == gridDim.x - 1)
      for (int k = threadIdx.x; k <= N; k += NT) {
        const double v = r[(size_t)N * n1 + k];
        dst[(size_t)N * n1 + k] = v;
        rz += v * v;
      }
    if (want_rz) {
      // fixed-order block sum (warp trees, then the warps in order)
      __shared__ double wred[NT / 32 > 0 ? NT / 32 : 1];
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      rz = warp_sum(rz);
      if (lane == 0) wred[warp] = rz;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < NT / 32; ++w) t += wred[w];
        rz_part[blockIdx.x] = t;
      }
    }
  }
}

// Column DSTs, spectral scaling and inverse column DSTs on T in place:
// CTA b owns columns 4b .. 4b+3 (column 0 is the zero column), two complex
// FFTs of L points (columns (4b, 4b+1) and (4b+2, 4b+3)), L/4 threads in two
// groups.  coskn[k] = cos(pi k / N).
template <int L>
__global__ void __launch_bounds__(L / 4)
    k_dst_cols(int N, double* __restrict__ T, DstStencil S, const double* __restrict__ coskn,
               const double2* __restrict__ tw, const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  constexpr int NT = L / 8;
  extern __shared__ double2 dst_buf[];
  const int grp = threadIdx.x / NT, tid = threadIdx.x % NT;
  constexpr int LP = fpad_len(L);
  double2* buf = dst_buf + grp * LP;
  const int k0 = 4 * blockIdx.x;
  // load rows 1..N-1 of the 4 columns: thread t takes column t % 4 of row
  // 1 + t / 4 (one 32-byte sector per row)
  for (int t = threadIdx.x; t < 4 * (N - 1); t += 2 * NT) {
    const int l = 1 + (t >> 2), c = t & 3;
    const double v = T[(size_t)l * N + k0 + c];
    double2* b = dst_buf + (c >> 1) * LP;
    if (c & 1) {
      b[fpad(l)].y = v;
      b[fpad(L - l)].y = -v;
    } else {
      b[fpad(l)].x = v;
      b[fpad(L - l)].x = -v;
    }
  }
  if (threadIdx.x < 2) {
    double2* b = dst_buf + threadIdx.x * LP;
    b[fpad(0)] = make_double2(0.0, 0.0);
    b[fpad(N)] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_smem<L, NT>(buf, tw, tid);
  // spectral scaling: column k (a: 4b + 2 grp, b: + 1), row frequency l
  {
    const int ka = k0 + 2 * grp, kb = ka + 1;
    const double cka = coskn[ka], ckb = coskn[kb];
    const double sc = 4.0 / ((double)N * (double)N);
    for (int l = 1 + tid; l <= N - 1; l += NT) {
      const double2 Y = buf[fpad(l)];
      const double cl = coskn[l];
      // column 0 is the zero column (Y = 0 there): any nonzero lambda
      const double la = ka == 0 ? 1.0
                                : S.s00 + 2.0 * S.s10 * cka + cl * (2.0 * S.s01 + 4.0 * S.s11 * cka);
      const double lb = S.s00 + 2.0 * S.s10 * ckb + cl * (2.0 * S.s01 + 4.0 * S.s11 * ckb);
      const double2 y = make_double2(-0.5 * Y.y * sc / la, 0.5 * Y.x * sc / lb);
      buf[fpad(l)] = y;
      buf[fpad(L - l)] = make_double2(-y.x, -y.y);
    }
    if (tid == 0) {
      buf[fpad(0)] = make_double2(0.0, 0.0);
      buf[fpad(N)] = make_double2(0.0, 0.0);
    }
  }
  __syncthreads();
  fft_smem<L, NT>(buf, tw, tid);
  for (int t = threadIdx.x; t < 4 * (N - 1); t += 2 * NT) {
    const int l = 1 + (t >> 2), c = t & 3;
    const double2 Y = dst_buf[(c >> 1) * LP + fpad(l)];
    T[(size_t)l * N + k0 + c] = (c & 1) ? 0.5 * Y.x : -0.5 * Y.y;
  }
}

// ---------------------------------------------------------------------------
// Half-length transforms (N >= 256).  The odd extension above spends a
// complex FFT of length 2N on two real rows although half of its input and
// output is redundant.  Here the pair z = a + i b (two real rows, the DST is
// real-linear) goes through ONE complex FFT of length N:
//   v_0 = 0,  v_j = sin(pi j/N) (z_j + z_{N-j}) + (z_j - z_{N-j}) / 2,
//   V = FFT_N(v);  V^a_k = (V_k + conj V_{N-k}) / 2,
//                  V^b_k = (V_k - conj V_{N-k}) / (2i)   (the two real FFTs),
//   S_{2k}   = -Im V^._k                          (k = 1 .. N/2-1),
//   S_{2k+1} = Re V^._0 / 2 + sum_{i=1..k} Re V^._i  (k = 0 .. N/2-1),
// since sum_j v_j sin(2 pi jk/N) = S_{2k} and sum_j v_j cos(2 pi jk/N) =
// S_{2k+1} - S_{2k-1}.  The running sum is a block scan in a fixed order
// (4 consecutive k per thread, warp shuffles, the warps in order).  Half the
// shared-memory traffic and arithmetic of the length-2N transform; measured
// relative error 2-5e-15 at N = 1024, 2048 against the direct sum.
//
// In: buf[fpad(j)] = z_j (j = 1..N-1).  Out: buf[fpad(k)] = S_k (k = 1..N-1),
// buf[fpad(0)] = 0.  NT = N / 8 threads per transform (tid in [0, NT), whole
// warps); all threads of the CTA call it together (block-wide barriers);
// wtot: NT / 32 shared double2 per transform.  tw = e^{-2 pi i q / (2N)}.
template <int N, int NT>
__device__ __forceinline__ void dsth_transform(double2* buf, const double2* __restrict__ tw,
                                               const double* __restrict__ coskn, int tid,
                                               double2* wtot) {
  static_assert(NT * 8 == N && NT % 32 == 0, "dsth_transform: N / 8 threads, whole warps");
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int j = 1 + tid + i * NT;                 // 1 .. N/2
    const double sj = __ldg(coskn + (N / 2 - j));   // sin(pi j / N) = cos(pi (N/2 - j) / N)
    const double2 zj = buf[fpad(j)], zn = buf[fpad(N - j)];
    const double2 sm = c_add(zj, zn), df = c_sub(zj, zn);
    buf[fpad(j)] = make_double2(fma(sj, sm.x, 0.5 * df.x), fma(sj, sm.y, 0.5 * df.y));
    if (j != N / 2)
      buf[fpad(N - j)] = make_double2(fma(sj, sm.x, -0.5 * df.x), fma(sj, sm.y, -0.5 * df.y));
  }
  if (tid == 0) buf[fpad(0)] = make_double2(0.0, 0.0);
  __syncthreads();
  fft_smem<N, NT, 1, 2 * N>(buf, tw, tid);
  double2 R[4], I[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int k = 4 * tid + e;
    const double2 Vk = buf[fpad(k)], Vn = buf[fpad((N - k) & (N - 1))];
    R[e] = make_double2(0.5 * (Vk.x + Vn.x), 0.5 * (Vk.y + Vn.y));  // Re V^a_k, Re V^b_k
    I[e] = make_double2(0.5 * (Vn.y - Vk.y), 0.5 * (Vk.x - Vn.x));  // S^a_2k,   S^b_2k
  }
  if (tid == 0) R[0] = make_double2(0.5 * R[0].x, 0.5 * R[0].y);
#pragma unroll
  for (int e = 1; e < 4; ++e) R[e] = c_add(R[e], R[e - 1]);
  const int lane = tid & 31, warp = tid >> 5;
  double2 inc = R[3];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double x = __shfl_up_sync(0xffffffffu, inc.x, o);
    const double y = __shfl_up_sync(0xffffffffu, inc.y, o);
    if (lane >= o) inc = make_double2(inc.x + x, inc.y + y);
  }
  if (lane == 31) wtot[warp] = inc;
  double2 off;
  off.x = __shfl_up_sync(0xffffffffu, inc.x, 1);
  off.y = __shfl_up_sync(0xffffffffu, inc.y, 1);
  if (lane == 0) off = make_double2(0.0, 0.0);
  __syncthreads();  // warp totals published; every V read is done
  for (int w = 0; w < warp; ++w) off = c_add(off, wtot[w]);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int k = 4 * tid + e;
    buf[fpad(2 * k)] = k == 0 ? make_double2(0.0, 0.0) : I[e];
    buf[fpad(2 * k + 1)] = c_add(off, R[e]);
  }
  __syncthreads();
}

// Row DSTs by the half-length transform: CTA b takes rows 1 + 2b and 2 + 2b
// (N / 8 threads).  Arguments and fused-CG behaviour as k_dst_rows.
// Register caps at N >= 2048 only (768 resident threads per SM in the row
// kernels, 1024 in the column kernel: the 4.2M-point grid is throughput
// bound, application 143 -> 124 us; at 1024^2 the latency-bound kernels lose
// with the few spills the cap costs, 42 -> 48 us; profiles/r02/s5_regs.log).
template <int N, bool INV>
__global__ void __launch_bounds__(N / 8, N >= 2048 ? 768 / (N / 8) : 0)
    k_dsth_rows(const double* __restrict__ src, double* __restrict__ dst,
                const double* __restrict__ r, const double* __restrict__ coskn,
                const double2* __restrict__ tw, const int* stop, SkipCtl sk,
                double* __restrict__ rz_part) {
  IRK_PDL_ENTER();
  constexpr int NT = N / 8;
  if constexpr (!INV && (NT >= kBlock || 2 * NT == kBlock)) {
    if (sk.st) {
      const double rr = dst_reduce_rr<NT>(sk.rr, sk.G);
      const bool skip = cg_skip_pred<double>(sk.st, rr, sk.maxit);
      if (blockIdx.x == 0 && threadIdx.x == 0) sk.st->skip = skip ? 1 : 0;
      if (skip) return;
      stop = nullptr;
    }
  }
  if (stop && *stop) return;
  extern __shared__ double2 dst_buf[];
  __shared__ double2 wtot[NT / 32];
  double2* buf = dst_buf;
  constexpr int n1 = N + 1;
  const int ra = 1 + 2 * blockIdx.x, rb = ra + 1;
  const bool hb = rb <= N - 1;
  constexpr int sstride = INV ? N : n1;
  const double* sa = src + (size_t)ra * sstride;
  const double* sb = src + (size_t)rb * sstride;
  double pra[INV ? 9 : 1], prb[INV ? 9 : 1];
  if constexpr (INV) {
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const int k = threadIdx.x + i * NT;
      pra[i] = k <= N ? r[(size_t)ra * n1 + k] : 0.0;
      prb[i] = (hb && k <= N) ? r[(size_t)rb * n1 + k] : 0.0;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = threadIdx.x + i * NT;
    if (j >= 1) buf[fpad(j)] = make_double2(sa[j], hb ? sb[j] : 0.0);
  }
  dsth_transform<N, NT>(buf, tw, coskn, threadIdx.x, wtot);
  constexpr int dstride = INV ? n1 : N;
  double* da = dst + (size_t)ra * dstride;
  double* db = dst + (size_t)rb * dstride;
  double rz = 0.0;
  const bool want_rz = INV && rz_part != nullptr;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const int k = threadIdx.x + i * NT;
    if (k > N) break;
    if (k >= 1 && k <= N - 1) {
      const double2 S = buf[fpad(k)];
      da[k] = S.x;
      if (hb) db[k] = S.y;
      if constexpr (INV) rz += pra[i] * S.x + prb[i] * S.y;  // prb = 0 without row b
    } else if constexpr (INV) {
      da[k] = pra[i];  // boundary columns x = 0, x = N: identity rows
      if (hb) db[k] = prb[i];
      rz += pra[i] * pra[i] + prb[i] * prb[i];
    } else if (k == 0) {
      da[0] = 0.0;
      if (hb) db[0] = 0.0;
    }
  }
  if constexpr (INV) {
    if (blockIdx.x == 0)
      for (int k = threadIdx.x; k <= N; k += NT) {
        const double v = r[k];
        dst[k] = v;
        rz += v * v;
      }
    if (blockIdx.x == gridDim.x - 1)
      for (int k = threadIdx.x; k <= N; k += NT) {
        const double v = r[(size_t)N * n1 + k];
        dst[(size_t)N * n1 + k] = v;
        rz += v * v;
      }
    if (want_rz) {
      __shared__ double wred[NT / 32];
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      rz = warp_sum(rz);
      if (lane == 0) wred[warp] = rz;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < NT / 32; ++w) t += wred[w];
        rz_part[blockIdx.x] = t;
      }
    }
  }
}

// Column DSTs, spectral scaling and inverse column DSTs on T in place by the
// half-length transform: CTA b owns columns 4b .. 4b+3 (two transforms, N / 4
// threads in two groups).
template <int N>
__global__ void __launch_bounds__(N / 4, N >= 2048 ? 1024 / (N / 4) : 0)
    k_dsth_cols(double* __restrict__ T, DstStencil S, const double* __restrict__ coskn,
                const double2* __restrict__ tw, const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  constexpr int NT = N / 8, LP = fpad_len(N);
  extern __shared__ double2 dst_buf[];
  __shared__ double2 wtot2[2][NT / 32];
  const int grp = threadIdx.x / NT, tid = threadIdx.x % NT;
  double2* buf = dst_buf + grp * LP;
  const int k0 = 4 * blockIdx.x;
  for (int t = threadIdx.x; t < 4 * (N - 1); t += 2 * NT) {
    const int l = 1 + (t >> 2), c = t & 3;
    const double v = T[(size_t)l * N + k0 + c];
    double2* b = dst_buf + (c >> 1) * LP;
    if (c & 1) b[fpad(l)].y = v;
    else b[fpad(l)].x = v;
  }
  dsth_transform<N, NT>(buf, tw, coskn, tid, wtot2[grp]);
  {
    const int ka = k0 + 2 * grp, kb = ka + 1;
    const double cka = coskn[ka], ckb = coskn[kb];
    const double sc = 4.0 / ((double)N * (double)N);
    for (int l = 1 + tid; l <= N - 1; l += NT) {
      const double2 Y = buf[fpad(l)];
      const double cl = coskn[l];
      // column 0 is the zero column (Y = 0 there): any nonzero lambda
      const double la = ka == 0 ? 1.0
                                : S.s00 + 2.0 * S.s10 * cka + cl * (2.0 * S.s01 + 4.0 * S.s11 * cka);
      const double lb = S.s00 + 2.0 * S.s10 * ckb + cl * (2.0 * S.s01 + 4.0 * S.s11 * ckb);
      buf[fpad(l)] = make_double2(Y.x * sc / la, Y.y * sc / lb);
    }
  }
  dsth_transform<N, NT>(buf, tw, coskn, tid, wtot2[grp]);
  for (int t = threadIdx.x; t < 4 * (N - 1); t += 2 * NT) {
    const int l = 1 + (t >> 2), c = t & 3;
    const double2 Y = dst_buf[(c >> 1) * LP + fpad(l)];
    T[(size_t)l * N + k0 + c] = (c & 1) ? Y.y : Y.x;
  }
}

#endif  // IRK_DST_2D

}  // namespace irk
