// Finite-element load vectors and error norms on the structured grids of
// the manufactured-solution problems (SURVEY §8 f, row 3).
//
// Reference anchors (under /root/reference/pkg/src/implicitrk/):
//   _elements / _quad_rule   problems.py:158-191 (1D P1, 2D Q1, 2-point Gauss)
//   assemble_load            problems.py:194-202
//   l2_error / h1_error      problems.py:205-232
//   heat_mms_1d / _2d        problems.py:113-149
//
// Layout: element e of the 2D grid is (ex, ey), e = ey*N + ex, local nodes
// (ex,ey), (ex+1,ey), (ex,ey+1), (ex+1,ey+1); 1D element e has nodes e, e+1.
// Quadrature-point data are q-major: f[q*nelem + e].
#include <cmath>
#include <vector>

#include "irk_internal.cuh"

namespace irk {

constexpr int kMaxQ = 4;  // 2x2 Gauss (2D) / 2 points (1D)

struct FeRule {
  int nq, nl;
  double w[kMaxQ];
  double phi[kMaxQ][4];
};

// out[v] = sum_q sum_{e adjacent to v, ascending} w_q (f[q][e] phi_q[a(e,v)]):
// the reference's np.add.at accumulation order (quadrature points outer,
// elements ascending inner), rounded step by step (no FMA contraction), so
// the result is bitwise identical for identical f values.
__global__ void k_fe_load(int dim, int64_t N, FeRule R, const double* __restrict__ f,
                          double* __restrict__ out) {
  const int64_t n1 = N + 1;
  const int64_t nv = dim == 1 ? n1 : n1 * n1;
  const int64_t ne = dim == 1 ? N : N * N;
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  int64_t el[4];
  int loc[4];
  int cnt = 0;
  if (dim == 1) {
    if (v - 1 >= 0) { el[cnt] = v - 1; loc[cnt++] = 1; }
    if (v < N) { el[cnt] = v; loc[cnt++] = 0; }
  } else {
    const int64_t i = v % n1, j = v / n1;
    if (i > 0 && j > 0) { el[cnt] = (j - 1) * N + (i - 1); loc[cnt++] = 3; }
    if (i < N && j > 0) { el[cnt] = (j - 1) * N + i; loc[cnt++] = 2; }
    if (i > 0 && j < N) { el[cnt] = j * N + (i - 1); loc[cnt++] = 1; }
    if (i < N && j < N) { el[cnt] = j * N + i; loc[cnt++] = 0; }
  }
  double acc = 0.0;
  for (int q = 0; q < R.nq; ++q) {
    for (int c = 0; c < cnt; ++c) {
      const double fv = f[(int64_t)q * ne + el[c]];
      acc = __dadd_rn(acc, __dmul_rn(R.w[q], __dmul_rn(fv, R.phi[q][loc[c]])));
    }
  }
  out[v] = acc;
}

// Forcing of the built-in manufactured solutions evaluated on the device at
// the quadrature points: kind 1 = heat_mms_1d, kind 2 = heat_mms_2d.
struct QPts {
  double xi[kMaxQ], eta[kMaxQ];
};

__global__ void k_fe_mms_forcing(int kind, int64_t N, int nq, double t, const QPts Q,
                                 double* __restrict__ f) {
  const int64_t ne = kind == 1 ? N : N * N;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const double h = 1.0 / (double)N;
  const double pi = 3.141592653589793;
  const double decay = exp(-0.1 * t);
  for (int q = 0; q < nq; ++q) {
    double val;
    if (kind == 1) {
      const double x = (double)e * h + Q.xi[q] * h;
      val = (pi * pi - 0.1) * (decay * sin(pi * x));
    } else {
      const int64_t ex = e % N, ey = e / N;
      const double x = (double)ex * h + Q.xi[q] * h, y = (double)ey * h + Q.eta[q] * h;
      val = (2.0 * pi * pi - 0.1) * (decay * sin(pi * x) * cos(pi * y));
    }
    f[(int64_t)q * ne + e] = val;
  }
}

// Per-block partial sums of sum_q w_q [ (u_h . phi_q - uex)^2
//   + sum_d (u_h . dphi_qd - gex_d)^2 ] (gradient part only when gex given).
struct FeGrad {
  double dphi[kMaxQ][2][4];
};

__global__ void k_fe_err(int dim, int64_t N, FeRule R, FeGrad D, const double* __restrict__ u,
                         const double* __restrict__ uex, const double* __restrict__ gex,
                         double* __restrict__ part) {
  const int64_t n1 = N + 1;
  const int64_t ne = dim == 1 ? N : N * N;
  double acc = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    double ul[4];
    if (dim == 1) {
      ul[0] = u[e];
      ul[1] = u[e + 1];
    } else {
      const int64_t b = (e / N) * n1 + (e % N);
      ul[0] = u[b];
      ul[1] = u[b + 1];
      ul[2] = u[b + n1];
      ul[3] = u[b + n1 + 1];
    }
    for (int q = 0; q < R.nq; ++q) {
      double uh = 0.0;
      for (int a = 0; a < R.nl; ++a) uh += ul[a] * R.phi[q][a];
      const double d0 = uh - (uex ? uex[(int64_t)q * ne + e] : 0.0);
      double s = d0 * d0;
      if (gex) {
        for (int d = 0; d < dim; ++d) {
          double gh = 0.0;
          for (int a = 0; a < R.nl; ++a) gh += ul[a] * D.dphi[q][d][a];
          const double dd = gh - gex[((int64_t)q * dim + d) * ne + e];
          s += dd * dd;
        }
      }
      acc += R.w[q] * s;
    }
  }
  __shared__ double red[kBlock / 32];
  double v[1] = {acc};
  block_sum<1>(v, red);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

static FeRule make_rule(int dim, int64_t N, FeGrad* D) {
  const double g0 = 0.5 - 0.5 / std::sqrt(3.0), g1 = 0.5 + 0.5 / std::sqrt(3.0);
  const double gp[2] = {g0, g1};
  const double h = 1.0 / (double)N;
  FeRule R{};
  if (dim == 1) {
    R.nq = 2;
    R.nl = 2;
    for (int q = 0; q < 2; ++q) {
      const double xi = gp[q];
      R.w[q] = 0.5 * h;
      R.phi[q][0] = 1 - xi;
      R.phi[q][1] = xi;
      if (D) {
        D->dphi[q][0][0] = -1.0 / h;
        D->dphi[q][0][1] = 1.0 / h;
      }
    }
  } else {
    R.nq = 4;
    R.nl = 4;
    int q = 0;
    for (int a = 0; a < 2; ++a) {
      for (int b = 0; b < 2; ++b, ++q) {
        const double xi = gp[a], eta = gp[b];
        R.w[q] = 0.5 * 0.5 * h * h;
        R.phi[q][0] = (1 - xi) * (1 - eta);
        R.phi[q][1] = xi * (1 - eta);
        R.phi[q][2] = (1 - xi) * eta;
        R.phi[q][3] = xi * eta;
        if (D) {
          D->dphi[q][0][0] = -(1 - eta) / h;
          D->dphi[q][0][1] = (1 - eta) / h;
          D->dphi[q][0][2] = -eta / h;
          D->dphi[q][0][3] = eta / h;
          D->dphi[q][1][0] = -(1 - xi) / h;
          D->dphi[q][1][1] = -xi / h;
          D->dphi[q][1][2] = (1 - xi) / h;
          D->dphi[q][1][3] = xi / h;
        }
      }
    }
  }
  return R;
}

}  // namespace irk

using namespace irk;

extern "C" {

int irk_fe_load(irk_ctx* ctx, int dim, int64_t N, const double* f_dev, double* out_dev) {
  IRK_REQUIRE(ctx && f_dev && out_dev, "irk_fe_load: NULL argument");
  IRK_REQUIRE(dim == 1 || dim == 2, "irk_fe_load: dim must be 1 or 2");
  IRK_REQUIRE(N >= 1, "irk_fe_load: N >= 1");
  const FeRule R = make_rule(dim, N, nullptr);
  const int64_t nv = dim == 1 ? N + 1 : (N + 1) * (N + 1);
  k_fe_load<<<(unsigned)((nv + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(dim, N, R, f_dev,
                                                                              out_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_fe_mms_forcing(irk_ctx* ctx, int kind, int64_t N, double t, double* f_dev) {
  IRK_REQUIRE(ctx && f_dev, "irk_fe_mms_forcing: NULL argument");
  IRK_REQUIRE(kind == 1 || kind == 2, "irk_fe_mms_forcing: kind must be 1 or 2");
  IRK_REQUIRE(N >= 1, "irk_fe_mms_forcing: N >= 1");
  const double g0 = 0.5 - 0.5 / std::sqrt(3.0), g1 = 0.5 + 0.5 / std::sqrt(3.0);
  // quadrature order of make_rule: 1D g0, g1; 2D (xi, eta) = (g0,g0), (g0,g1),
  // (g1,g0), (g1,g1) (xi outer, as _quad_rule)
  QPts Q{};
  if (kind == 1) {
    Q.xi[0] = g0;
    Q.xi[1] = g1;
  } else {
    const double a[4] = {g0, g0, g1, g1}, b[4] = {g0, g1, g0, g1};
    for (int q = 0; q < 4; ++q) {
      Q.xi[q] = a[q];
      Q.eta[q] = b[q];
    }
  }
  const int64_t ne = kind == 1 ? N : N * N;
  k_fe_mms_forcing<<<(unsigned)((ne + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
      kind, N, kind == 1 ? 2 : 4, t, Q, f_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_fe_error_sq(irk_ctx* ctx, int dim, int64_t N, const double* u_dev, const double* uex_dev,
                    const double* gex_dev, double* result_host) {
  IRK_REQUIRE(ctx && u_dev && result_host, "irk_fe_error_sq: NULL argument");
  IRK_REQUIRE(dim == 1 || dim == 2, "irk_fe_error_sq: dim must be 1 or 2");
  IRK_REQUIRE(N >= 1, "irk_fe_error_sq: N >= 1");
  FeGrad D{};
  const FeRule R = make_rule(dim, N, &D);
  const int64_t ne = dim == 1 ? N : N * N;
  const int G = grid_for(ctx, ne, kBlock, 4);
  IRK_TRY(ensure_red(ctx, (size_t)G + 64));
  k_fe_err<<<G, kBlock, 0, ctx->stream>>>(dim, N, R, D, u_dev, uex_dev, gex_dev, ctx->red);
  IRK_CHECK_LAUNCH(ctx);
  std::vector<double> part(G);
  IRK_CUDA(cudaMemcpyAsync(part.data(), ctx->red, G * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  double s = 0.0;
  for (int b = 0; b < G; ++b) s += part[b];
  *result_host = s;
  return IRK_OK;
}

}  // extern "C"
