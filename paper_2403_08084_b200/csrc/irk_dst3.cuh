// 3D complex fast sine-transform (DST-I) preconditioner of the Kuhn P1
// Schur-pair blocks alpha M + beta K (complex alpha, beta) with the
// full-boundary Dirichlet set: the interface irk_mgc.cu drives (kernels in
// irk_dst3.cu).
#pragma once

#include <cuda_runtime.h>

struct irk_ctx;

namespace irk {

// s[a + 2 b + 4 c]: the reflection-symmetrised stencil coefficient of the
// offsets (+-a, +-b, +-c), a, b, c in {0, 1}; the sine mode (kx, ky, kz) has
//   lambda = sum_abc s_abc (2 cos(pi kx/N))^a (2 cos(pi ky/N))^b (2 cos(pi kz/N))^c
struct Dst3Coef {
  double2 s[8];
  double sc;  // (2/N)^3
};

struct Dst3Plan {
  int N = 0;
  Dst3Coef C{};
  double2* T = nullptr;            // (N+1)^3 spectral work array (layout of the grid vectors)
  const double2* tw = nullptr;     // e^{-2 pi i q / (2N)}, q < 2N
  const double* cosk = nullptr;    // cos(pi k / N), k = 0..N
};

// N for which a transform plan exists (2N = 2^a or 3 * 2^a, 24 <= 2N <= 384)
bool dst3_supported(int N);
// kernel attributes (dynamic shared memory) of the plan for N
int dst3_prepare(int N);
// z = B_s^-1 r on the grid vectors (interior: F Lambda^-1 F, boundary z = r);
// r != z, 16-byte aligned.  Five launches on stream s.
int dst3_apply(irk_ctx* ctx, cudaStream_t s, const Dst3Plan& P, const double2* r, double2* z,
               const int* stop);

}  // namespace irk
