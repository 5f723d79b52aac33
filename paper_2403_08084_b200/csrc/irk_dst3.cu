// 3D complex fast sine-transform (DST-I) preconditioner for the Schur-pair
// blocks alpha M + beta K of the Kuhn-split P1 grid (complex alpha, beta;
// Gauss-Legendre stages, precond.py SCHUR kind) with the full-boundary
// Dirichlet set.  The reference factorises these blocks with SuperLU
// (sparsela.py:149-191); here COCG is preconditioned by the exact inverse of
// the block's reflection-symmetrised stencil.
//
// The interior operator is ONE 3x3x3 stencil (15 Kuhn slots), extracted and
// verified against every row by the structured multigrid setup (irk_mgc.cu
// k_mg3_row_stencil / k_mg3_verify).  Averaging each coefficient over the
// reflections of its offset gives a stencil with coefficients s_abc on the
// offsets (+-a, +-b, +-c), diagonalised by the 3D sine basis:
//   lambda(kx, ky, kz) = sum_abc s_abc (2 cx)^a (2 cy)^b (2 cz)^c,
//   c. = cos(pi k. / N),
//   B_s^-1 = (2/N)^3 F Lambda^-1 F,   F = S_x S_y S_z  (S = DST-I, S S = N/2).
// The Kuhn stiffness stencil is the 7-point one (already symmetric); B - B_s
// only moves the mass matrix's face- and body-diagonal couplings between the
// diagonals, so COCG reaches 1e-6 in 3-4 iterations at 96^3, dt = 5e-3
// instead of ~7.4 multigrid V-cycle ones, at a fraction of a V-cycle's cost.
//
// A complex line z = a + i b is ONE complex FFT of length L = 2N of its odd
// extension (the DST is real-linear):  Y_k = -2i S_k(z).  The FFT is the
// shared-memory Stockham autosort of irk_dst.cuh with a radix-3 pass added
// (L = 2^a or 3 * 2^a: 96^3 needs L = 192 = 8 * 8 * 3).
//
// Five launches per application, each reading and writing the grid once
// (14.6 MB at 96^3: L2-resident), 8 lines per CTA:
//   k_dst3<L,0,0>  x lines of r   -> T            (contiguous lines)
//   k_dst3<L,1,1>  y lines of T, in place          (8 adjacent x per CTA: one
//   k_dst3<L,2,2>  z lines of T, in place:          128-byte segment per point
//                  forward, scale by (2/N)^3 / lambda, inverse   of the line)
//   k_dst3<L,1,1>  y lines of T, in place
//   k_dst3<L,0,3>  x lines of T   -> z; boundary points z = r (identity rows)
#include <cmath>

#include "irk_internal.cuh"
#include "irk_dst.cuh"
#include "irk_dst3.cuh"

namespace irk {
namespace {

constexpr int kLpc = 8;  // lines per CTA

// forward 3-point DFT (w = e^{-2 pi i / 3})
__device__ __forceinline__ void dft3(double2* v) {
  constexpr double h = 0.86602540378443864676;
  const double2 s = c_add(v[1], v[2]);
  const double2 d = c_sub(v[1], v[2]);
  const double2 m = make_double2(v[0].x - 0.5 * s.x, v[0].y - 0.5 * s.y);
  const double2 t = make_double2(h * d.y, -h * d.x);  // -i h (b - c)
  v[0] = c_add(v[0], s);
  v[1] = c_add(m, t);
  v[2] = c_sub(m, t);
}

// One Stockham pass of radix R (NS = the product of the earlier radices)
// over the L-point sequence in buf (padded layout fpad of irk_dst.cuh), NT
// threads per sequence (tid in [0, NT)); L / R need not be a multiple of NT.
// All threads of the CTA call it together (block-wide barriers).  One
// twiddle load per butterfly, its powers by complex multiplications.
template <int L, int R, int NT, int NS>
__device__ __forceinline__ void fft_pass_g(double2* buf, const double2* __restrict__ tw, int tid) {
  constexpr int NB = L / R;
  constexpr int ITEMS = (NB + NT - 1) / NT;
  double2 v[ITEMS][R];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int j = tid + it * NT;
    if (j < NB) {
      const int k = j % NS;
#pragma unroll
      for (int r = 0; r < R; ++r) v[it][r] = buf[fpad(j + r * NB)];
      if constexpr (NS > 1) {
        const double2 w1 = __ldg(tw + k * (L / (NS * R)));
        v[it][1] = c_mul(v[it][1], w1);
        if constexpr (R >= 3) {
          const double2 w2 = c_mul(w1, w1);
          v[it][2] = c_mul(v[it][2], w2);
          if constexpr (R >= 4) {
            const double2 w3 = c_mul(w2, w1);
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
      }
      if constexpr (R == 8) dft8(v[it]);
      else if constexpr (R == 4) dft4(v[it][0], v[it][1], v[it][2], v[it][3]);
      else if constexpr (R == 3) dft3(v[it]);
      else dft2(v[it]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int j = tid + it * NT;
    if (j < NB) {
      const int k = j % NS;
      const int base = (j / NS) * NS * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) buf[fpad(base + r * NS)] = v[it][r];
    }
  }
  __syncthreads();
}

__host__ __device__ constexpr int f_rem8(int L) { return L % 8 == 0 ? f_rem8(L / 8) : L; }

// Forward FFT of L = 2^a or 3 * 2^a points in buf (padded layout): radix-8
// passes, one radix-4 or radix-2 pass, one radix-3 pass.
template <int L, int NT, int NS = 1>
__device__ __forceinline__ void fft_smem_g(double2* buf, const double2* __restrict__ tw, int tid) {
  constexpr int rest = L / NS;  // product of the radices still to do
  if constexpr (rest % 8 == 0) {
    fft_pass_g<L, 8, NT, NS>(buf, tw, tid);
    fft_smem_g<L, NT, NS * 8>(buf, tw, tid);
  } else if constexpr (rest % 4 == 0) {
    fft_pass_g<L, 4, NT, NS>(buf, tw, tid);
    fft_smem_g<L, NT, NS * 4>(buf, tw, tid);
  } else if constexpr (rest % 2 == 0) {
    fft_pass_g<L, 2, NT, NS>(buf, tw, tid);
    fft_smem_g<L, NT, NS * 2>(buf, tw, tid);
  } else if constexpr (rest == 3) {
    fft_pass_g<L, 3, NT, NS>(buf, tw, tid);
  } else {
    static_assert(rest == 1, "fft_smem_g: L must be 2^a or 3 * 2^a");
  }
}

__device__ __forceinline__ double2 c_div(double2 a, double2 b) {
  const double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
__device__ __forceinline__ double2 c_fma(double2 a, double t, double2 acc) {
  return make_double2(fma(a.x, t, acc.x), fma(a.y, t, acc.y));
}

// Line transforms of the (N+1)^3 grid vector, N = L / 2, kLpc lines per CTA
// (one group of L / 8 threads per line).
//   AXIS 0: x lines; MODE 0 covers the interior lines (y, z in 1..N-1),
//           MODE 3 every line (y, z in 0..N): interior points transformed,
//           boundary points copied from r.
//   AXIS 1 / 2: y / z lines; CTA = 8 adjacent x (from 1 + 8 g) at one
//           interior z / y.  MODE 1: transform in place; MODE 2: forward,
//           spectral scaling, inverse.
template <int L, int AXIS, int MODE>
__global__ void __launch_bounds__(L)
    k_dst3(const double2* src, double2* dst, const double2* __restrict__ r, Dst3Coef C,
           const double* __restrict__ cosk, const double2* __restrict__ tw, const int* stop) {
  IRK_PDL_ENTER();
  if (stop && *stop) return;
  constexpr int N = L / 2, n1 = N + 1, NT = L / 8, LS = fpad_len(L) + 1;
  constexpr int NI = N - 1;                       // interior points per line
  constexpr int NXG = (NI + kLpc - 1) / kLpc;     // x groups (strided axes)
  static_assert((AXIS == 0) == (MODE == 0 || MODE == 3), "k_dst3: axis/mode combination");
  extern __shared__ double2 dst3_buf[];
  const int g = threadIdx.x / NT, tid = threadIdx.x % NT;
  double2* buf = dst3_buf + g * LS;

  // element (q, j) of the CTA: line q, point j along the axis -> flat index
  // (< 0: not a grid point of this CTA); inter: the point is transformed
  auto locate = [&](int q, int j, bool& inter) -> int64_t {
    if constexpr (AXIS == 0) {
      const int l = blockIdx.x * kLpc + q;
      int y, z;
      if constexpr (MODE == 0) {
        y = 1 + l % NI;
        z = 1 + l / NI;
        inter = l < NI * NI && j >= 1 && j <= NI;
        if (l >= NI * NI) return -1;
      } else {
        y = l % n1;
        z = l / n1;
        if (l >= n1 * n1) {
          inter = false;
          return -1;
        }
        inter = y >= 1 && y <= NI && z >= 1 && z <= NI && j >= 1 && j <= NI;
      }
      return ((int64_t)z * n1 + y) * n1 + j;
    } else {
      const int x = 1 + (blockIdx.x % NXG) * kLpc + q;
      const int o = 1 + blockIdx.x / NXG;
      inter = x <= NI && j >= 1 && j <= NI;
      if (x > NI) return -1;
      return AXIS == 1 ? ((int64_t)o * n1 + j) * n1 + x : ((int64_t)j * n1 + o) * n1 + x;
    }
  };

  for (int e = threadIdx.x; e < kLpc * n1; e += L) {
    int q, j;
    if constexpr (AXIS == 0) {
      q = e / n1;
      j = e - q * n1;
    } else {
      q = e % kLpc;
      j = e / kLpc;
    }
    bool inter;
    const int64_t at = locate(q, j, inter);
    double2 v = make_double2(0.0, 0.0);
    if (inter) v = src[at];
    double2* b = dst3_buf + q * LS;
    b[fpad(j)] = v;
    if (j >= 1 && j <= NI) b[fpad(L - j)] = make_double2(-v.x, -v.y);
  }
  __syncthreads();
  fft_smem_g<L, NT>(buf, tw, tid);

  if constexpr (MODE == 2) {
    // line g: kx = x, ky = o (AXIS 2: o is y); lambda(kz) = P + Q 2 cos(pi kz/N)
    const int x = 1 + (blockIdx.x % NXG) * kLpc + g;
    const int o = 1 + blockIdx.x / NXG;
    const double tx = 2.0 * cosk[x <= N ? x : N], ty = 2.0 * cosk[o];
    const double txy = tx * ty;
    double2 P = c_fma(C.s[3], txy, c_fma(C.s[2], ty, c_fma(C.s[1], tx, C.s[0])));
    double2 Q = c_fma(C.s[7], txy, c_fma(C.s[6], ty, c_fma(C.s[5], tx, C.s[4])));
    if (x > NI) {
      P = make_double2(1.0, 0.0);
      Q = make_double2(0.0, 0.0);
    }
    for (int l = 1 + tid; l <= NI; l += NT) {
      const double2 Y = buf[fpad(l)];
      const double2 lam = c_fma(Q, 2.0 * cosk[l], P);
      const double2 y = c_div(make_double2(-0.5 * C.sc * Y.y, 0.5 * C.sc * Y.x), lam);
      buf[fpad(l)] = y;
      buf[fpad(L - l)] = make_double2(-y.x, -y.y);
    }
    if (tid == 0) {
      buf[fpad(0)] = make_double2(0.0, 0.0);
      buf[fpad(N)] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    fft_smem_g<L, NT>(buf, tw, tid);
  }

  for (int e = threadIdx.x; e < kLpc * n1; e += L) {
    int q, j;
    if constexpr (AXIS == 0) {
      q = e / n1;
      j = e - q * n1;
    } else {
      q = e % kLpc;
      j = e / kLpc;
    }
    bool inter;
    const int64_t at = locate(q, j, inter);
    if (at < 0) continue;
    if (inter) {
      const double2 Y = dst3_buf[q * LS + fpad(j)];
      dst[at] = make_double2(-0.5 * Y.y, 0.5 * Y.x);
    } else if constexpr (MODE == 3) {
      dst[at] = r[at];
    }
  }
}

template <int L>
int prepare_l() {
  const int smem = kLpc * (fpad_len(L) + 1) * (int)sizeof(double2);
  IRK_CUDA(cudaFuncSetAttribute(k_dst3<L, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  IRK_CUDA(cudaFuncSetAttribute(k_dst3<L, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  IRK_CUDA(cudaFuncSetAttribute(k_dst3<L, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  IRK_CUDA(cudaFuncSetAttribute(k_dst3<L, 0, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  return IRK_OK;
}

template <int L>
int apply_l(irk_ctx* ctx, cudaStream_t s, const Dst3Plan& P, const double2* r, double2* z,
            const int* stop) {
  constexpr int N = L / 2, n1 = N + 1, NI = N - 1, NXG = (NI + kLpc - 1) / kLpc;
  const size_t smem = (size_t)kLpc * (fpad_len(L) + 1) * sizeof(double2);
  const double2* T = P.T;
  launch(k_dst3<L, 0, 0>, (NI * NI + kLpc - 1) / kLpc, L, smem, s, r, P.T, r, P.C, P.cosk, P.tw,
         stop);
  launch(k_dst3<L, 1, 1>, NXG * NI, L, smem, s, T, P.T, r, P.C, P.cosk, P.tw, stop);
  launch(k_dst3<L, 2, 2>, NXG * NI, L, smem, s, T, P.T, r, P.C, P.cosk, P.tw, stop);
  launch(k_dst3<L, 1, 1>, NXG * NI, L, smem, s, T, P.T, r, P.C, P.cosk, P.tw, stop);
  launch(k_dst3<L, 0, 3>, (n1 * n1 + kLpc - 1) / kLpc, L, smem, s, T, z, r, P.C, P.cosk, P.tw,
         stop);
  ctx->launches += 5;
  return cudaPeekAtLastError() == cudaSuccess ? IRK_OK : IRK_ECUDA;
}

}  // namespace

#define IRK_DST3_SIZES(X) X(24) X(32) X(48) X(64) X(96) X(128) X(192) X(256) X(384)

bool dst3_supported(int N) {
  switch (2 * N) {
#define X(L) case L:
    IRK_DST3_SIZES(X)
#undef X
    return true;
  }
  return false;
}

int dst3_prepare(int N) {
  switch (2 * N) {
#define X(L) case L: return prepare_l<L>();
    IRK_DST3_SIZES(X)
#undef X
  }
  set_error("dst3: no sine-transform plan for N = %d", N);
  return IRK_EINVAL;
}

int dst3_apply(irk_ctx* ctx, cudaStream_t s, const Dst3Plan& P, const double2* r, double2* z,
               const int* stop) {
  switch (2 * P.N) {
#define X(L) case L: return apply_l<L>(ctx, s, P, r, z, stop);
    IRK_DST3_SIZES(X)
#undef X
  }
  set_error("dst3: no sine-transform plan for N = %d", P.N);
  return IRK_EINVAL;
}

}  // namespace irk
