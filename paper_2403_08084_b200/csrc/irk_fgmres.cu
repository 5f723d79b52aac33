// Device-resident FGMRES cycle: the Arnoldi loop of fgmres
// (/root/reference/pkg/src/implicitrk/sparsela.py:355-394; the host-driven
// version is sparsela.fgmres_device) with no host round trip per iteration.
//
// The host loop of fgmres_device synchronises once per Arnoldi step to read
// the Hessenberg column and run the Givens rotations in Python.  On small
// systems (config 1: n = 2178) that round trip and the Python around it are
// the whole cost of the step (~170 us per iteration against ~20 us of
// kernels).  Here one CUDA graph runs a whole restart cycle:
//
//   WHILE (not frozen) {
//     step graph            w = A P v_j  (right PC: z_j = P v_j, w = A z_j),
//                           captured once by the caller (torch.cuda.graph) on
//                           fixed buffers vj, zj, w
//     k_fg_multidot         h[i] = <V_i, w>, i <= j   (j read on the device)
//     k_fg_orth             w -= V h, h[j+1] = ||w||  (optional CGS2 pass)
//     k_fg_givens           Hessenberg column j, previous rotations, new
//                           rotation, g, residual estimate, convergence /
//                           lucky breakdown (one thread, the reference's
//                           arithmetic order)
//     k_fg_advance          Z_j = z_j, V_{j+1} = v_j = w / h[j+1]; the last
//                           block advances j or freezes the state
//     k_fg_cond             loop condition = not frozen
//   }
//
// then k_fg_backsub (y = R^-1 g, one warp) and k_fg_lincomb (x += Z y).  The
// host reads the iteration count and the residual history once per cycle.
// Reductions are deterministic (block partials summed in block order).
#include "irk_internal.cuh"

namespace irk {

// device state (ints): j, converged, k (columns done), lucky, frozen
enum { kFgJ = 0, kFgConv = 1, kFgK = 2, kFgLucky = 3, kFgFrozen = 4, kFgInts = 8 };

__device__ __forceinline__ bool fg_last_block(unsigned int* counter) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) *counter = 0u;
  return is_last;
}

// h[i] = <V_i, w>, i < k = j + 1 (read from the state)
__global__ void __launch_bounds__(kBlock)
    k_fg_multidot(int64_t n, const int* __restrict__ st, const double* __restrict__ V,
                  int64_t ldv, const double* __restrict__ w, double* __restrict__ partials,
                  unsigned int* counter, double* __restrict__ h) {
  if (__ldcg(st + kFgFrozen)) return;
  const int k = __ldcg(st + kFgJ) + 1;
  __shared__ double acc[kMaxBasis][kBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < k * (kBlock / 32); i += blockDim.x)
    acc[i / (kBlock / 32)][i % (kBlock / 32)] = 0.0;
  __syncthreads();
  for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x; e0 < n; e0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = e0 + threadIdx.x;
    const double wv = e < n ? w[e] : 0.0;
    for (int i = 0; i < k; ++i) {
      double p = e < n ? __ldg(V + (int64_t)i * ldv + e) * wv : 0.0;
      p = warp_sum(p);
      if (lane == 0) acc[i][warp] += p;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < kBlock / 32; ++q) s += acc[i][q];
    partials[(int64_t)i * gridDim.x + blockIdx.x] = s;
  }
  if (fg_last_block(counter)) {
    for (int i = warp; i < k; i += kBlock / 32) {
      double s = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) s += partials[(int64_t)i * gridDim.x + b];
      s = warp_sum(s);
      if (lane == 0) h[i] = s;
    }
  }
}

// w -= sum_{i<k} coef[i] V_i ; out_norm (may be NULL) = ||w||; add (may be
// NULL): coef2 += coef (the CGS2 pass accumulates into h)
__global__ void __launch_bounds__(kBlock)
    k_fg_orth(int64_t n, const int* __restrict__ st, const double* __restrict__ V, int64_t ldv,
              const double* __restrict__ coef, double* __restrict__ w,
              double* __restrict__ partials, unsigned int* counter, double* __restrict__ out_norm,
              double* __restrict__ add) {
  if (__ldcg(st + kFgFrozen)) return;
  const int k = __ldcg(st + kFgJ) + 1;
  __shared__ double hc[kMaxBasis];
  __shared__ double red[8];
  for (int i = threadIdx.x; i < k; i += blockDim.x) hc[i] = coef[i];
  __syncthreads();
  double ss = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double x = w[e];
    for (int i = 0; i < k; ++i) x -= hc[i] * __ldg(V + (int64_t)i * ldv + e);
    w[e] = x;
    ss += x * x;
  }
  double v[1] = {ss};
  block_sum<1>(v, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = v[0];
  if (fg_last_block(counter)) {
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += partials[b];
      s = warp_sum(s);
      if (threadIdx.x == 0 && out_norm) out_norm[k] = sqrt(s);
    }
    if (add)
      for (int i = threadIdx.x; i < k; i += blockDim.x) add[i] += coef[i];
  }
}

// Hessenberg column j (h[0..j+1], h[j+1] = ||w|| before normalisation):
// previous rotations, new rotation, g, residual estimate |g[j+1]|, and the
// stop tests of fgmres (residual <= target, or h[j+1] < breakdown).
// H is column-major with leading dimension ldh.  prm = {target, breakdown}.
__global__ void k_fg_givens(int* __restrict__ st, const double* __restrict__ h,
                            double* __restrict__ H, int ldh, double* __restrict__ cs,
                            double* __restrict__ sn, double* __restrict__ g,
                            double* __restrict__ hist, const double* __restrict__ prm) {
  if (threadIdx.x != 0 || st[kFgFrozen]) return;
  const int j = st[kFgJ];
  double* Hj = H + (int64_t)j * ldh;
  for (int i = 0; i <= j + 1; ++i) Hj[i] = h[i];
  const bool lucky = Hj[j + 1] < prm[1];
  for (int i = 0; i < j; ++i) {
    const double t = cs[i] * Hj[i] + sn[i] * Hj[i + 1];
    Hj[i + 1] = -sn[i] * Hj[i] + cs[i] * Hj[i + 1];
    Hj[i] = t;
  }
  double d = hypot(Hj[j], Hj[j + 1]);
  if (d == 0.0) {
    cs[j] = 1.0;
    sn[j] = 0.0;
    d = 1e-300;
  } else {
    cs[j] = Hj[j] / d;
    sn[j] = Hj[j + 1] / d;
  }
  Hj[j] = d;
  Hj[j + 1] = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
  const double res = fabs(g[j + 1]);
  hist[j + 1] = res;
  st[kFgConv] = (res <= prm[0] || lucky) ? 1 : 0;
  st[kFgLucky] = lucky ? 1 : 0;
  st[kFgK] = j + 1;
}

// Z_j = z_j (store_z), V_{j+1} = v_j = w / h[j+1] (unless lucky); the last
// block advances j, or freezes the state when the cycle ends.
__global__ void __launch_bounds__(kBlock)
    k_fg_advance(int64_t n, int* __restrict__ st, int cycle, const double* __restrict__ prm,
                 const double* __restrict__ h,
                 const double* __restrict__ zj, double* __restrict__ Z, int64_t ldz,
                 const double* __restrict__ w, double* __restrict__ V, int64_t ldv,
                 double* __restrict__ vj, unsigned int* counter) {
  if (__ldcg(st + kFgFrozen)) return;
  const int j = __ldcg(st + kFgJ);
  const int cap = min(cycle, (int)prm[2]);
  const bool stop = __ldcg(st + kFgConv) || j + 1 >= cap;
  const bool scale = !__ldcg(st + kFgLucky) && !stop;
  const double a = scale ? 1.0 / h[j + 1] : 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (Z) Z[(int64_t)j * ldz + e] = zj[e];
    if (scale) {
      const double v = a * w[e];
      V[(int64_t)(j + 1) * ldv + e] = v;
      vj[e] = v;
    }
  }
  if (fg_last_block(counter) && threadIdx.x == 0) {
    if (stop) st[kFgFrozen] = 1;
    else st[kFgJ] = j + 1;
  }
}

__global__ void k_fg_cond(cudaGraphConditionalHandle hnd, const int* st) {
  if (threadIdx.x == 0) cudaGraphSetConditional(hnd, st[kFgFrozen] ? 0u : 1u);
}

// cycle start: state, g = beta e_1, hist[0] = beta, V_0 = v_j = r / beta
__global__ void k_fg_start(int64_t n, int* __restrict__ st, double* __restrict__ g,
                           double* __restrict__ hist, double* __restrict__ prm, int cycle,
                           int cap, double beta, double target, double breakdown,
                           const double* __restrict__ r, double* __restrict__ V0,
                           double* __restrict__ vj) {
  const double a = 1.0 / beta;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = a * r[e];
    V0[e] = v;
    vj[e] = v;
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < kFgInts; i += blockDim.x) st[i] = 0;
    for (int i = threadIdx.x; i <= cycle; i += blockDim.x) g[i] = i == 0 ? beta : 0.0;
    if (threadIdx.x == 0) {
      hist[0] = beta;
      prm[0] = target;
      prm[1] = breakdown;
      prm[2] = cap;
    }
  }
}

// y = R^-1 g on the k x k rotated Hessenberg (fgmres's back-substitution,
// sparsela.py:396-399)
__global__ void k_fg_backsub(const int* __restrict__ st, const double* __restrict__ H, int ldh,
                             const double* __restrict__ g, double* __restrict__ y) {
  if (threadIdx.x != 0) return;
  const int k = st[kFgK];
  for (int i = k - 1; i >= 0; --i) {
    double s = 0.0;
    for (int l = i + 1; l < k; ++l) s += H[(int64_t)l * ldh + i] * y[l];
    y[i] = (g[i] - s) / H[(int64_t)i * ldh + i];
  }
}

// x += sum_{i<k} y[i] Z_i
__global__ void k_fg_lincomb(int64_t n, const int* __restrict__ st, const double* __restrict__ Z,
                             int64_t ldz, const double* __restrict__ y, double* __restrict__ x) {
  const int k = __ldcg(st + kFgK);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double acc = x[e];
    for (int i = 0; i < k; ++i) acc += y[i] * __ldg(Z + (int64_t)i * ldz + e);
    x[e] = acc;
  }
}

}  // namespace irk

using namespace irk;

// work layout (doubles): h [2 kMaxBasis] | H [(cycle+1) cycle] | cs, sn, g,
// hist, y [cycle + 1 each] | prm [8]
struct irk_fgraph {
  int64_t n = 0;
  int cycle = 0;
  double *V = nullptr, *Z = nullptr, *vj = nullptr, *w = nullptr;
  int64_t ldv = 0, ldz = 0;
  double *h = nullptr, *H = nullptr, *cs = nullptr, *sn = nullptr, *g = nullptr;
  double *hist = nullptr, *y = nullptr, *prm = nullptr;
  int* st = nullptr;
  double* red = nullptr;  // the context scratch the graph was built with
  cudaGraphExec_t exec = nullptr;
  int64_t pass_kernels = 0;  // kernels one pass of the WHILE body launches
};

extern "C" {

size_t irk_fgmres_work_doubles(int cycle) {
  return 2 * (size_t)kMaxBasis + (size_t)(cycle + 1) * cycle + 5 * (size_t)(cycle + 1) + 8;
}

int irk_fgmres_graph_create(irk_ctx* ctx, void* step_graph, int64_t n, int cycle, int reorth,
                            double* V, int64_t ldv, double* Z, int64_t ldz, double* vj,
                            const double* zj, double* w, double* work, int* st_dev,
                            irk_fgraph** out) {
  IRK_REQUIRE(ctx && step_graph && V && vj && w && work && st_dev && out,
              "irk_fgmres_graph_create: NULL argument");
  IRK_REQUIRE(cycle >= 1 && cycle < kMaxBasis, "irk_fgmres_graph_create: 1 <= cycle < %d",
              kMaxBasis);
  IRK_REQUIRE(ldv >= n && (!Z || (zj && ldz >= n)), "irk_fgmres_graph_create: bad layout");
  const int G = grid_for(ctx, n, kBlock, 4);
  IRK_TRY(ensure_red(ctx, (size_t)G * kMaxBasis + 64));
  irk_fgraph* fg = new irk_fgraph();
  fg->n = n;
  fg->cycle = cycle;
  fg->V = V, fg->Z = Z, fg->vj = vj, fg->w = w;
  fg->ldv = ldv, fg->ldz = ldz;
  double* p = work;
  fg->h = p, p += 2 * kMaxBasis;
  fg->H = p, p += (size_t)(cycle + 1) * cycle;
  fg->cs = p, p += cycle + 1;
  fg->sn = p, p += cycle + 1;
  fg->g = p, p += cycle + 1;
  fg->hist = p, p += cycle + 1;
  fg->y = p, p += cycle + 1;
  fg->prm = p;
  fg->st = st_dev;
  fg->red = ctx->red;
  if (!ctx->cap_stream)
    IRK_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
  cudaGraph_t graph = nullptr;
  IRK_CUDA(cudaGraphCreate(&graph, 0));
  auto fail = [&](cudaError_t e) {
    cudaGraphDestroy(graph);
    delete fg;
    set_error("irk_fgmres_graph_create: %s", cudaGetErrorString(e));
    return IRK_ECUDA;
  };
  cudaGraphConditionalHandle hnd;
  cudaError_t e = cudaGraphConditionalHandleCreate(&hnd, graph, 1, cudaGraphCondAssignDefault);
  if (e != cudaSuccess) return fail(e);
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = hnd;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t cnode;
  if ((e = cudaGraphAddNode(&cnode, graph, nullptr, 0, &np)) != cudaSuccess) return fail(e);
  cudaGraph_t body = np.conditional.phGraph_out[0];
  cudaGraphNode_t child;
  if ((e = cudaGraphAddChildGraphNode(&child, body, nullptr, 0, (cudaGraph_t)step_graph)) !=
      cudaSuccess)
    return fail(e);
  if ((e = cudaStreamBeginCaptureToGraph(ctx->cap_stream, body, &child, nullptr, 1,
                                         cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
    return fail(e);
  cudaStream_t cs = ctx->cap_stream;
  double* red = ctx->red;
  k_fg_multidot<<<G, kBlock, 0, cs>>>(n, st_dev, V, ldv, w, red, ctx->counters + 8, fg->h);
  k_fg_orth<<<G, kBlock, 0, cs>>>(n, st_dev, V, ldv, fg->h, w, red, ctx->counters + 9,
                                  reorth ? nullptr : fg->h, nullptr);
  if (reorth) {
    double* h2 = fg->h + kMaxBasis;
    k_fg_multidot<<<G, kBlock, 0, cs>>>(n, st_dev, V, ldv, w, red, ctx->counters + 8, h2);
    k_fg_orth<<<G, kBlock, 0, cs>>>(n, st_dev, V, ldv, h2, w, red, ctx->counters + 9, fg->h,
                                    fg->h);
  }
  k_fg_givens<<<1, 32, 0, cs>>>(st_dev, fg->h, fg->H, cycle + 1, fg->cs, fg->sn, fg->g, fg->hist,
                                fg->prm);
  k_fg_advance<<<G, kBlock, 0, cs>>>(n, st_dev, cycle, fg->prm, fg->h, zj, Z, ldz, w, V, ldv, vj,
                                     ctx->counters + 10);
  k_fg_cond<<<1, 32, 0, cs>>>(hnd, st_dev);
  cudaGraph_t got = nullptr;
  e = cudaStreamEndCapture(cs, &got);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(e);
  e = cudaGraphInstantiate(&fg->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    delete fg;
    set_error("irk_fgmres_graph_create: instantiate: %s", cudaGetErrorString(e));
    return IRK_ECUDA;
  }
  // launch accounting of a replay: the kernel nodes of the captured
  // application plus the Arnoldi kernels above, per pass
  {
    size_t nn = 0;
    if (cudaGraphGetNodes((cudaGraph_t)step_graph, nullptr, &nn) == cudaSuccess && nn > 0) {
      std::vector<cudaGraphNode_t> nodes(nn);
      if (cudaGraphGetNodes((cudaGraph_t)step_graph, nodes.data(), &nn) == cudaSuccess) {
        for (size_t i = 0; i < nn; ++i) {
          cudaGraphNodeType ty;
          if (cudaGraphNodeGetType(nodes[i], &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel)
            fg->pass_kernels++;
        }
      }
    }
    fg->pass_kernels += reorth ? 7 : 5;
  }
  *out = fg;
  return IRK_OK;
}

// One restart cycle of at most cap <= cycle Arnoldi steps from the residual r
// (beta = ||r||): V_0 = r / beta, the WHILE graph, then x += Z y.  Writes the number of Arnoldi steps taken, the
// convergence flag and the residual estimates hist[0..k] (host, synchronous).
int irk_fgmres_graph_run(irk_ctx* ctx, irk_fgraph* fg, int cap, const double* r, double beta,
                         double target, double breakdown, double* x, int* k_host,
                         int* conv_host, double* hist_host) {
  IRK_REQUIRE(ctx && fg && r && x && k_host && conv_host && hist_host,
              "irk_fgmres_graph_run: NULL argument");
  IRK_REQUIRE(cap >= 1 && cap <= fg->cycle, "irk_fgmres_graph_run: 1 <= cap <= cycle");
  IRK_REQUIRE(fg->red == ctx->red,
              "irk_fgmres_graph_run: the context scratch moved since the graph was built");
  cudaStream_t s = ctx->stream;
  const int G = grid_for(ctx, fg->n, kBlock, 4);
  k_fg_start<<<G, kBlock, 0, s>>>(fg->n, fg->st, fg->g, fg->hist, fg->prm, fg->cycle, cap,
                                  beta, target, breakdown, r, fg->V, fg->vj);
  IRK_CHECK_LAUNCH(ctx);
  IRK_CUDA(cudaGraphLaunch(fg->exec, s));
  k_fg_backsub<<<1, 32, 0, s>>>(fg->st, fg->H, fg->cycle + 1, fg->g, fg->y);
  IRK_CHECK_LAUNCH(ctx);
  k_fg_lincomb<<<G, kBlock, 0, s>>>(fg->n, fg->st, fg->Z ? fg->Z : fg->V,
                                    fg->Z ? fg->ldz : fg->ldv, fg->y, x);
  IRK_CHECK_LAUNCH(ctx);
  IRK_TRY(ensure_pinned(ctx, 64 * sizeof(int) + (size_t)(fg->cycle + 1) * sizeof(double)));
  int* hs = reinterpret_cast<int*>(ctx->pinned);
  double* hh = reinterpret_cast<double*>(ctx->pinned + 64 * sizeof(int));
  IRK_CUDA(cudaMemcpyAsync(hs, fg->st, kFgInts * sizeof(int), cudaMemcpyDeviceToHost, s));
  IRK_CUDA(cudaMemcpyAsync(hh, fg->hist, (fg->cycle + 1) * sizeof(double), cudaMemcpyDeviceToHost,
                           s));
  IRK_CUDA(cudaStreamSynchronize(s));
  *k_host = hs[kFgK];
  *conv_host = hs[kFgConv];
  ctx->launches += (int64_t)hs[kFgK] * fg->pass_kernels;
  for (int i = 0; i <= hs[kFgK]; ++i) hist_host[i] = hh[i];
  return IRK_OK;
}

int irk_fgmres_graph_destroy(irk_fgraph* fg) {
  if (fg) {
    if (fg->exec) cudaGraphExecDestroy(fg->exec);
    delete fg;
  }
  return IRK_OK;
}

}  // extern "C"
