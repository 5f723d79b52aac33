// Device sparse matrices: CSR + SELL-32 storage, pattern algebra, P1/Q1
// assembly on the structured grid and the generic SpMV.
//
// Reference anchors (paths under /root/reference/pkg/src/implicitrk/):
//   SparseMatrix            sparsela.py:43-115
//   spmv                    sparsela.py:118-123
//   dirichlet_constrain     sparsela.py:126-146
//   StructuredGrid numbering problems.py:25-64 (x fastest, lexicographic)
//   _p1_matrices / assemble_heat  problems.py:67-99
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <vector>

#include "irk_internal.cuh"

namespace irk {

Pattern* pattern_new() { return new Pattern(); }
void pattern_retain(Pattern* p) { p->refs.fetch_add(1); }
void pattern_release(Pattern* p) {
  if (!p) return;
  if (p->refs.fetch_sub(1) == 1) {
    cudaFree(p->rowptr);
    cudaFree(p->col);
    cudaFree(p->slice_ptr);
    cudaFree(p->sell_col);
    cudaFree(p->csr2sell);
    cudaFree(p->diag_pos);
    cudaFree(p->colhdr);
    delete p;
  }
}

static int scan_exclusive(irk_ctx* ctx, const int* in, int* out, int64_t n) {
  size_t tmp = 0;
  IRK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, ctx->stream));
  void* d_tmp = nullptr;
  IRK_CUDA(cudaMalloc(&d_tmp, tmp + 16));
  cudaError_t e = cub::DeviceScan::ExclusiveSum(d_tmp, tmp, in, out, (int)n, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  cudaFree(d_tmp);
  IRK_CUDA(e);
  ctx->launches++;
  return IRK_OK;
}

// --------------------------------------------------------------- SELL build

__global__ void k_slice_sizes(int64_t nrows, int64_t nslices, const int* __restrict__ rowptr,
                              int* __restrict__ sizes) {
  int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (gw >= nslices) return;
  int64_t r = gw * kSlice + lane;
  int len = (r < nrows) ? rowptr[r + 1] - rowptr[r] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
  if (lane == 0) sizes[gw] = len * kSlice;
  if (gw == nslices - 1 && lane == 0) sizes[nslices] = 0;
}

// Rows whose columns all lie on the stencil r + stencil[k] (k < W == slice
// width) are stored stencil-aligned: entry with offset stencil[k] in slot k,
// absent neighbours as explicit zeros at column r + stencil[k] (or r when
// that is outside the matrix).  On structured grids this makes the slots of
// boundary-touching slices slot-uniform too.  Other rows are packed in CSR
// order and padded with column r.
__global__ void k_sell_fill(int64_t nrows, int64_t ncols, const int* __restrict__ rowptr,
                            const int* __restrict__ col, const int* __restrict__ slice_ptr,
                            int* __restrict__ sell_col, int* __restrict__ csr2sell,
                            int* __restrict__ diag_pos, int64_t nslices,
                            const int* __restrict__ stencil, int W) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t s = r / kSlice;
  if (s >= nslices) return;
  int lane = (int)(r % kSlice);
  int base = slice_ptr[s];
  int width = (slice_ptr[s + 1] - base) / kSlice;
  int pad = (int)(r < ncols ? r : 0);
  if (r >= nrows) {
    for (int k = 0; k < width; ++k) sell_col[base + k * kSlice + lane] = pad;
    return;
  }
  int p0 = rowptr[r], len = rowptr[r + 1] - p0;
  int dpos = -1;
  bool aligned = stencil != nullptr && W == width && len <= W;
  if (aligned) {
    unsigned used = 0;  // W <= 32
    for (int j = 0; j < len && aligned; ++j) {
      const int64_t d = (int64_t)col[p0 + j] - r;
      int k = 0;
      while (k < W && stencil[k] != d) ++k;
      if (k == W || ((used >> k) & 1u)) aligned = false;
      else used |= 1u << k;
    }
  }
  if (aligned) {
    for (int k = 0; k < W; ++k) {
      const int64_t c = r + stencil[k];
      sell_col[base + k * kSlice + lane] = (c >= 0 && c < ncols) ? (int)c : pad;
    }
    for (int j = 0; j < len; ++j) {
      const int c = col[p0 + j];
      int k = 0;
      while (stencil[k] != (int64_t)c - r) ++k;
      const int pos = base + k * kSlice + lane;
      csr2sell[p0 + j] = pos;
      if (c == r) dpos = pos;
    }
  } else {
    for (int k = 0; k < width; ++k) {
      int pos = base + k * kSlice + lane;
      if (k < len) {
        int c = col[p0 + k];
        sell_col[pos] = c;
        csr2sell[p0 + k] = pos;
        if (c == r) dpos = pos;
      } else {
        sell_col[pos] = pad;
      }
    }
  }
  diag_pos[r] = dpos;
}

// one warp per slice: slot-uniform column offsets
__global__ void k_colhdr(int64_t nrows, int64_t nslices, const int* __restrict__ slice_ptr,
                         const int* __restrict__ sell_col, int* __restrict__ colhdr) {
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  int base = slice_ptr[s], width = (slice_ptr[s + 1] - base) / kSlice;
  int64_t row = s * kSlice + lane;
  bool full = (s + 1) * kSlice <= nrows;
  for (int k = 0; k < width; ++k) {
    const int c = sell_col[base + k * kSlice + lane];
    int off = c - (int)row;
    int off0 = __shfl_sync(0xffffffffu, off, 0);
    bool uni = __all_sync(0xffffffffu, off == off0) && full;
    if (lane == 0) colhdr[base / kSlice + k] = uni ? off0 : kNonUniform;
  }
}

// one warp per slice: window rows of slot-uniform slices (max via atomicMax)
__global__ void k_win_rows(int64_t nslices, const int* __restrict__ slice_ptr,
                           const int* __restrict__ colhdr, int* __restrict__ out) {
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  int base = slice_ptr[s], width = (slice_ptr[s + 1] - base) / kSlice;
  if (width > 32) return;
  const int d = lane < width ? colhdr[base / kSlice + lane] : 0;
  if (!__all_sync(0xffffffffu, lane >= width || d != kNonUniform)) return;
  const WinLayout L = win_layout(d, width);
  if (lane == 0) atomicMax(out, L.total);
}

// one warp per slice: slot-uniform values (bitwise equality), else NaN
__global__ void k_valhdr(int64_t nrows, int64_t nslices, const int* __restrict__ slice_ptr,
                         const double* __restrict__ val, double* __restrict__ uval) {
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  int base = slice_ptr[s], width = (slice_ptr[s + 1] - base) / kSlice;
  bool full = (s + 1) * kSlice <= nrows;
  for (int k = 0; k < width; ++k) {
    unsigned long long b = __double_as_longlong(val[base + k * kSlice + lane]);
    unsigned long long b0 = __shfl_sync(0xffffffffu, b, 0);
    bool uni = __all_sync(0xffffffffu, b == b0) && full;
    if (lane == 0) uval[base / kSlice + k] = uni ? __longlong_as_double(b0) : __longlong_as_double(0x7ff8dead00000000ull);
  }
}

int mat_finalize(irk_ctx* ctx, irk_mat* A) {
  const Pattern* p = A->pat;
  if (p->nslices == 0) return IRK_OK;
  int64_t threads = p->nslices * 32;
  k_valhdr<<<(unsigned)((threads + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
      p->nrows, p->nslices, p->slice_ptr, A->val, A->uval);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int pattern_build_sell(irk_ctx* ctx, Pattern* p) {
  p->nslices = (p->nrows + kSlice - 1) / kSlice;
  int64_t ns = p->nslices;
  IRK_CUDA(cudaMalloc(&p->slice_ptr, (ns + 1) * sizeof(int)));
  int* sizes = nullptr;
  IRK_CUDA(cudaMalloc(&sizes, (ns + 1) * sizeof(int)));
  if (ns > 0) {
    int64_t threads = ns * 32;
    k_slice_sizes<<<(unsigned)((threads + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
        p->nrows, ns, p->rowptr, sizes);
    IRK_CHECK_LAUNCH(ctx);
    // Pad every slice to the widest one (ELL-32) when that costs <= 5% (or
    // the matrix is small): the slice offsets become arithmetic (32 * W * s),
    // so kernels need no dependent slice_ptr load before their first matrix
    // load.
    {
      std::vector<int> hs(ns);
      IRK_CUDA(cudaMemcpyAsync(hs.data(), sizes, ns * sizeof(int), cudaMemcpyDeviceToHost,
                               ctx->stream));
      IRK_CUDA(cudaStreamSynchronize(ctx->stream));
      int64_t tot = 0;
      int wmax = 0;
      for (int64_t q = 0; q < ns; ++q) {
        tot += hs[q];
        wmax = std::max(wmax, hs[q] / kSlice);
      }
      const int64_t padded = ns * (int64_t)kSlice * wmax;
      p->ellw = 0;
      // small matrices (the coarse multigrid levels): padding is cheap and
      // the arithmetic slice offsets / stencil path save a dependent load
      // in latency-bound kernels
      const bool small = p->nrows <= (1 << 17) && padded <= 2 * tot;
      if (wmax > 0 && (padded <= tot + tot / 20 || small) && padded < (int64_t)INT32_MAX / 2) {
        for (int64_t q = 0; q < ns; ++q) hs[q] = wmax * kSlice;
        IRK_CUDA(cudaMemcpyAsync(sizes, hs.data(), ns * sizeof(int), cudaMemcpyHostToDevice,
                                 ctx->stream));
        p->ellw = wmax;
      }
    }
    IRK_TRY(scan_exclusive(ctx, sizes, p->slice_ptr, ns + 1));
  } else {
    IRK_CUDA(cudaMemsetAsync(p->slice_ptr, 0, sizeof(int), ctx->stream));
  }
  int total = 0;
  IRK_CUDA(cudaMemcpyAsync(&total, p->slice_ptr + ns, sizeof(int), cudaMemcpyDeviceToHost,
                           ctx->stream));
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(sizes);
  p->sell_nnz = total;
  IRK_CUDA(cudaMalloc(&p->sell_col, ((size_t)total + 1) * sizeof(int)));
  IRK_CUDA(cudaMalloc(&p->csr2sell, ((size_t)p->nnz + 1) * sizeof(int)));
  IRK_CUDA(cudaMalloc(&p->diag_pos, ((size_t)p->nrows + 1) * sizeof(int)));
  if (ns > 0) {
    // stencil of ELL patterns: the offsets of a full-width row near the
    // middle of the matrix (an interior node on structured grids)
    int* d_stencil = nullptr;
    int W = 0;
    if (p->ellw > 0 && p->ellw <= 32) {
      const int64_t lo = p->nrows / 2, cnt = std::min<int64_t>(p->nrows - lo, 4096);
      std::vector<int> rp(cnt + 1);
      IRK_CUDA(cudaMemcpyAsync(rp.data(), p->rowptr + lo, (cnt + 1) * sizeof(int),
                               cudaMemcpyDeviceToHost, ctx->stream));
      IRK_CUDA(cudaStreamSynchronize(ctx->stream));
      for (int64_t q = 0; q < cnt; ++q) {
        if (rp[q + 1] - rp[q] != p->ellw) continue;
        std::vector<int> c(p->ellw);
        IRK_CUDA(cudaMemcpyAsync(c.data(), p->col + rp[q], p->ellw * sizeof(int),
                                 cudaMemcpyDeviceToHost, ctx->stream));
        IRK_CUDA(cudaStreamSynchronize(ctx->stream));
        std::vector<int> st(p->ellw);
        for (int k = 0; k < p->ellw; ++k) st[k] = c[k] - (int)(lo + q);
        std::sort(st.begin(), st.end());
        if (std::adjacent_find(st.begin(), st.end()) != st.end()) break;
        IRK_CUDA(cudaMalloc(&d_stencil, p->ellw * sizeof(int)));
        IRK_CUDA(cudaMemcpyAsync(d_stencil, st.data(), p->ellw * sizeof(int),
                                 cudaMemcpyHostToDevice, ctx->stream));
        W = p->ellw;
        p->stencil = st;
        break;
      }
    }
    int64_t threads = ns * kSlice;
    k_sell_fill<<<(unsigned)((threads + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
        p->nrows, p->ncols, p->rowptr, p->col, p->slice_ptr, p->sell_col, p->csr2sell,
        p->diag_pos, ns, d_stencil, W);
    IRK_CHECK_LAUNCH(ctx);
    if (d_stencil) {
      IRK_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(d_stencil);
    }
  }
  IRK_CUDA(cudaMalloc(&p->colhdr, ((size_t)total / kSlice + 1) * sizeof(int)));
  if (ns > 0) {
    int64_t threads = ns * 32;
    int* cm = nullptr;
    IRK_CUDA(cudaMalloc(&cm, sizeof(int)));
    k_colhdr<<<(unsigned)((threads + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
        p->nrows, ns, p->slice_ptr, p->sell_col, p->colhdr);
    IRK_CHECK_LAUNCH(ctx);
    IRK_CUDA(cudaMemsetAsync(cm, 0, sizeof(int), ctx->stream));
    k_win_rows<<<(unsigned)((threads + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
        ns, p->slice_ptr, p->colhdr, cm);
    IRK_CHECK_LAUNCH(ctx);
    IRK_CUDA(cudaMemcpyAsync(&p->win_rows, cm, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    IRK_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(cm);
    std::vector<int> sp(ns + 1);
    IRK_CUDA(cudaMemcpyAsync(sp.data(), p->slice_ptr, (ns + 1) * sizeof(int),
                             cudaMemcpyDeviceToHost, ctx->stream));
    IRK_CUDA(cudaStreamSynchronize(ctx->stream));
    int mw = 0;
    for (int64_t q = 0; q < ns; ++q) mw = std::max(mw, (sp[q + 1] - sp[q]) / kSlice);
    p->maxw = mw;
  }
  return IRK_OK;
}

int mat_alloc(irk_ctx* ctx, Pattern* p, irk_mat** out) {
  irk_mat* A = new irk_mat();
  A->pat = p;
  pattern_retain(p);
  cudaError_t e = cudaMalloc(&A->val, ((size_t)p->sell_nnz + 1) * sizeof(double));
  if (e != cudaSuccess) {
    pattern_release(p);
    delete A;
    set_error("mat_alloc: %s", cudaGetErrorString(e));
    return IRK_ECUDA;
  }
  IRK_CUDA(cudaMemsetAsync(A->val, 0, ((size_t)p->sell_nnz + 1) * sizeof(double), ctx->stream));
  IRK_CUDA(cudaMalloc(&A->uval, ((size_t)p->sell_nnz / kSlice + 1) * sizeof(double)));
  IRK_CUDA(cudaMemsetAsync(A->uval, 0, ((size_t)p->sell_nnz / kSlice + 1) * sizeof(double),
                           ctx->stream));
  *out = A;
  return IRK_OK;
}

__global__ void k_scatter_vals(int64_t nnz, const int* __restrict__ csr2sell,
                               const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x)
    dst[csr2sell[p]] = src[p];
}

__global__ void k_gather_vals(int64_t nnz, const int* __restrict__ csr2sell,
                              const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x)
    dst[p] = src[csr2sell[p]];
}

int mat_set_csr_values(irk_ctx* ctx, irk_mat* A, const double* csr_val_dev) {
  int64_t nnz = A->pat->nnz;
  if (nnz == 0) return IRK_OK;
  k_scatter_vals<<<grid_for(ctx, nnz), kBlock, 0, ctx->stream>>>(nnz, A->pat->csr2sell,
                                                                   csr_val_dev, A->val);
  IRK_CHECK_LAUNCH(ctx);
  return mat_finalize(ctx, A);
}

// ------------------------------------------------------------ P1 assembly
// One thread per vertex row.  The row is accumulated element by element in
// the global element order (cells ascending lexicographically, then the
// fixed simplex order inside a cell), i.e. the order a COO -> CSR
// sum-duplicates assembly over that element list produces.

struct Row27 {
  double m[27];
  double k[27];
  bool hit[27];
};

__device__ __forceinline__ int slot_of(int dx, int dy, int dz) {
  return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
}

// 2D: cell (ci, cj) holds T1 = (00, 10, 11) and T2 = (00, 11, 01).
__device__ void p1_row_2d(int64_t N, int64_t i, int64_t j, double h, Row27& R) {
  const int tv[2][3][2] = {{{0, 0}, {1, 0}, {1, 1}}, {{0, 0}, {1, 1}, {0, 1}}};
  const double kl[2][3][3] = {{{0.5, -0.5, 0.0}, {-0.5, 1.0, -0.5}, {0.0, -0.5, 0.5}},
                              {{0.5, 0.0, -0.5}, {0.0, 0.5, -0.5}, {-0.5, -0.5, 1.0}}};
  const double mf = h * h / 24.0;
  for (int q = 0; q < 27; ++q) {
    R.m[q] = 0.0;
    R.k[q] = 0.0;
    R.hit[q] = false;
  }
  for (int64_t cj = j - 1; cj <= j; ++cj) {
    if (cj < 0 || cj >= N) continue;
    for (int64_t ci = i - 1; ci <= i; ++ci) {
      if (ci < 0 || ci >= N) continue;
      int lx = (int)(i - ci), ly = (int)(j - cj);
      for (int t = 0; t < 2; ++t) {
        int a = -1;
        for (int q = 0; q < 3; ++q)
          if (tv[t][q][0] == lx && tv[t][q][1] == ly) a = q;
        if (a < 0) continue;
        for (int b = 0; b < 3; ++b) {
          int sl = slot_of(tv[t][b][0] - lx, tv[t][b][1] - ly, 0);
          R.m[sl] += mf * (a == b ? 2.0 : 1.0);
          R.k[sl] += kl[t][a][b];
          R.hit[sl] = true;
        }
      }
    }
  }
}

// 3D Kuhn split: tet p = (0, e_a, e_a + e_b, 1) for the permutation (a, b, c).
__device__ void p1_row_3d(int64_t N, int64_t i, int64_t j, int64_t k, double h, Row27& R) {
  const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  const double G[4][4] = {{1, -1, 0, 0}, {-1, 2, -1, 0}, {0, -1, 2, -1}, {0, 0, -1, 1}};
  const double mf = h * h * h / 120.0;
  const double kf = h / 6.0;
  for (int q = 0; q < 27; ++q) {
    R.m[q] = 0.0;
    R.k[q] = 0.0;
    R.hit[q] = false;
  }
  for (int64_t ck = k - 1; ck <= k; ++ck) {
    if (ck < 0 || ck >= N) continue;
    for (int64_t cj = j - 1; cj <= j; ++cj) {
      if (cj < 0 || cj >= N) continue;
      for (int64_t ci = i - 1; ci <= i; ++ci) {
        if (ci < 0 || ci >= N) continue;
        int l[3] = {(int)(i - ci), (int)(j - cj), (int)(k - ck)};
        for (int t = 0; t < 6; ++t) {
          int v[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {1, 1, 1}};
          v[1][perm[t][0]] = 1;
          v[2][perm[t][0]] = 1;
          v[2][perm[t][1]] = 1;
          int a = -1;
          for (int q = 0; q < 4; ++q)
            if (v[q][0] == l[0] && v[q][1] == l[1] && v[q][2] == l[2]) a = q;
          if (a < 0) continue;
          for (int b = 0; b < 4; ++b) {
            int sl = slot_of(v[b][0] - l[0], v[b][1] - l[1], v[b][2] - l[2]);
            R.m[sl] += mf * (a == b ? 2.0 : 1.0);
            R.k[sl] += kf * G[a][b];
            R.hit[sl] = true;
          }
        }
      }
    }
  }
}

// 1D P1 on intervals: element (h/6)[[2,1],[1,2]], (1/h)[[1,-1],[-1,1]].
__device__ void p1_row_1d(int64_t N, int64_t i, double h, Row27& R) {
  for (int q = 0; q < 27; ++q) {
    R.m[q] = 0.0;
    R.k[q] = 0.0;
    R.hit[q] = false;
  }
  const double mo = h / 6.0, md = 2.0 * h / 6.0, kd = 1.0 / h, ko = -1.0 / h;
  for (int64_t ci = i - 1; ci <= i; ++ci) {
    if (ci < 0 || ci >= N) continue;
    int a = (int)(i - ci);
    for (int b = 0; b < 2; ++b) {
      int sl = slot_of(b - a, 0, 0);
      R.m[sl] += (a == b) ? md : mo;
      R.k[sl] += (a == b) ? kd : ko;
      R.hit[sl] = true;
    }
  }
}

__device__ void p1_row(int dim, int64_t N, int64_t r, double h, Row27& R, int64_t* stride) {
  int64_t n1 = N + 1;
  stride[0] = 1;
  stride[1] = n1;
  stride[2] = n1 * n1;
  if (dim == 1) {
    p1_row_1d(N, r, h, R);
  } else if (dim == 2) {
    p1_row_2d(N, r % n1, r / n1, h, R);
  } else {
    p1_row_3d(N, r % n1, (r / n1) % n1, r / (n1 * n1), h, R);
  }
}

__global__ void k_p1_count(int dim, int64_t N, int64_t m, double h, int* __restrict__ counts) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) {
    if (r == m) counts[m] = 0;
    return;
  }
  Row27 R;
  int64_t st[3];
  p1_row(dim, N, r, h, R, st);
  int c = 0;
  for (int q = 0; q < 27; ++q) c += R.hit[q] ? 1 : 0;
  counts[r] = c;
}

__global__ void k_p1_fill(int dim, int64_t N, int64_t m, double h, const int* __restrict__ rowptr,
                          int* __restrict__ col, double* __restrict__ mval,
                          double* __restrict__ kval) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  Row27 R;
  int64_t st[3];
  p1_row(dim, N, r, h, R, st);
  int p = rowptr[r];
  // slot order (dz, dy, dx) ascending == column order for x-fastest numbering
  for (int q = 0; q < 27; ++q) {
    if (!R.hit[q]) continue;
    int dx = q % 3 - 1, dy = (q / 3) % 3 - 1, dz = q / 9 - 1;
    col[p] = (int)(r + dx * st[0] + dy * st[1] + dz * st[2]);
    mval[p] = R.m[q];
    kval[p] = R.k[q];
    ++p;
  }
}

// 2D Q1 operators of the reference: M = M1 (x) M1, K = K1 (x) M1 + M1 (x) K1
// (problems.py:93-95) with the 1D P1 entries of _p1_matrices
// (problems.py:67-77); y factor first.
__device__ __forceinline__ void p1_1d_entry(int64_t N, int64_t a, int64_t b, double h,
                                            double& mv, double& kv) {
  if (a == b) {
    bool end = (a == 0 || a == N);
    mv = end ? 2 * h / 6 : 4 * h / 6;
    kv = end ? 1.0 / h : 2.0 / h;
  } else {
    mv = h / 6;
    kv = -1.0 / h;
  }
}

// full_x: every x index of a neighbouring block row is stored (the
// block-sparse pattern the reference's K takes on grids with N <= 4, where
// scipy's kron switches to dense BSR blocks and keeps their explicit zeros).
__global__ void k_q1_count(int64_t N, int64_t m, int full_x, int* __restrict__ counts) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) {
    if (r == m) counts[m] = 0;
    return;
  }
  int64_t n1 = N + 1, i = r % n1, j = r / n1;
  int cx = full_x ? (int)n1 : 1 + (i > 0) + (i < N), cy = 1 + (j > 0) + (j < N);
  counts[r] = cx * cy;
}

__global__ void k_q1_fill(int64_t N, int64_t m, double h, int full_x,
                          const int* __restrict__ rowptr, int* __restrict__ col,
                          double* __restrict__ mval, double* __restrict__ kval) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  int64_t n1 = N + 1, i = r % n1, j = r / n1;
  int p = rowptr[r];
  for (int64_t jj = j - 1; jj <= j + 1; ++jj) {
    if (jj < 0 || jj > N) continue;
    double my, ky;
    p1_1d_entry(N, j, jj, h, my, ky);
    int64_t lo = full_x ? 0 : i - 1, hi = full_x ? N : i + 1;
    for (int64_t ii = lo; ii <= hi; ++ii) {
      if (ii < 0 || ii > N) continue;
      double mx = 0.0, kx = 0.0;
      if (ii >= i - 1 && ii <= i + 1) p1_1d_entry(N, i, ii, h, mx, kx);
      col[p] = (int)(jj * n1 + ii);
      if (mval) mval[p] = my * mx;
      kval[p] = ky * mx + my * kx;
      ++p;
    }
  }
}

// ------------------------------------------------------------ pattern union

__global__ void k_union_count(int64_t nrows, const int* __restrict__ ra, const int* __restrict__ ca,
                              const int* __restrict__ rb, const int* __restrict__ cb,
                              int* __restrict__ counts) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) {
    if (r == nrows) counts[nrows] = 0;
    return;
  }
  int pa = ra[r], ea = ra[r + 1], pb = rb[r], eb = rb[r + 1], c = 0;
  while (pa < ea || pb < eb) {
    int x = pa < ea ? ca[pa] : INT_MAX, y = pb < eb ? cb[pb] : INT_MAX;
    if (x <= y) ++pa;
    if (y <= x) ++pb;
    ++c;
  }
  counts[r] = c;
}

__global__ void k_union_fill(int64_t nrows, const int* __restrict__ ra, const int* __restrict__ ca,
                             const int* __restrict__ rb, const int* __restrict__ cb,
                             const int* __restrict__ ru, int* __restrict__ cu,
                             int* __restrict__ mapa, int* __restrict__ mapb) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int pa = ra[r], ea = ra[r + 1], pb = rb[r], eb = rb[r + 1], q = ru[r];
  while (pa < ea || pb < eb) {
    int x = pa < ea ? ca[pa] : INT_MAX, y = pb < eb ? cb[pb] : INT_MAX;
    int c = x < y ? x : y;
    cu[q] = c;
    if (x == c) mapa[pa++] = q;
    if (y == c) mapb[pb++] = q;
    ++q;
  }
}

__global__ void k_remap_vals(int64_t nnz, const int* __restrict__ old_csr2sell,
                             const double* __restrict__ old_val, const int* __restrict__ map,
                             const int* __restrict__ new_csr2sell, double* __restrict__ new_val) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x)
    new_val[new_csr2sell[map[p]]] = old_val[old_csr2sell[p]];
}

// position of each X entry inside T's row (both rows sorted); -1 if absent
__global__ void k_on_pattern_map(int64_t nrows, const int* __restrict__ rx, const int* __restrict__ cx,
                                 const int* __restrict__ rt, const int* __restrict__ ct,
                                 int* __restrict__ map, int* __restrict__ missing) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int q = rt[r], e = rt[r + 1];
  for (int p = rx[r]; p < rx[r + 1]; ++p) {
    int c = cx[p];
    while (q < e && ct[q] < c) ++q;
    if (q < e && ct[q] == c) {
      map[p] = q;
    } else {
      map[p] = -1;
      atomicAdd(missing, 1);
    }
  }
}

__global__ void k_semi_jac(int64_t nrows, const int* __restrict__ slice_ptr,
                           const int* __restrict__ sell_col, const double* __restrict__ mv,
                           const double* __restrict__ kv, double kscale,
                           const double* __restrict__ d, int64_t ld, int64_t off,
                           double* __restrict__ out) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int64_t s = r / kSlice;
  int lane = (int)(r % kSlice);
  int base = slice_ptr[s], width = (slice_ptr[s + 1] - base) / kSlice;
  for (int k = 0; k < width; ++k) {
    int pos = base + k * kSlice + lane;
    int c = sell_col[pos];
    out[pos] = kscale * kv[pos] + mv[pos] * d[(int64_t)c * ld + off];
  }
}

// ------------------------------------------------- elementwise matrix ops

__global__ void k_combine(int64_t n, double alpha, const double* __restrict__ a, double beta,
                          const double* __restrict__ b, double* __restrict__ c) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    c[p] = alpha * a[p] + beta * b[p];
}

__global__ void k_constrain(int64_t nrows, int64_t nslices, const int* __restrict__ slice_ptr,
                            const int* __restrict__ sell_col, const int* __restrict__ diag_pos,
                            const uint8_t* __restrict__ mask, double diag_value,
                            double* __restrict__ val, int* __restrict__ missing) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int64_t s = r / kSlice;
  int lane = (int)(r % kSlice);
  int base = slice_ptr[s], width = (slice_ptr[s + 1] - base) / kSlice;
  bool rowc = mask[r] != 0;
  int dpos = diag_pos[r];
  for (int k = 0; k < width; ++k) {
    int pos = base + k * kSlice + lane;
    int c = sell_col[pos];
    if (rowc || mask[c]) val[pos] = 0.0;
  }
  if (rowc) {
    if (dpos >= 0)
      val[dpos] = diag_value;
    else if (diag_value != 0.0)
      atomicAdd(missing, 1);
  }
}

__global__ void k_diag(int64_t nrows, const int* __restrict__ diag_pos,
                       const double* __restrict__ val, double* __restrict__ d) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int p = diag_pos[r];
  d[r] = p >= 0 ? val[p] : 0.0;
}

__global__ void k_rowsum(int64_t nrows, const int* __restrict__ slice_ptr,
                         const double* __restrict__ val, double* __restrict__ out) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int64_t s = r / kSlice;
  int lane = (int)(r % kSlice);
  int base = slice_ptr[s], width = (slice_ptr[s + 1] - base) / kSlice;
  double acc = 0.0;
  for (int k = 0; k < width; ++k) acc += val[base + k * kSlice + lane];
  out[r] = acc;
}

// Gershgorin data of D^-1 A: out[r] = sum_c |A[r,c]| (padding entries are 0)
__global__ void k_absrowsum(int64_t nrows, const int* __restrict__ slice_ptr,
                            const double* __restrict__ val, double* __restrict__ out) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int64_t s = r / kSlice;
  int lane = (int)(r % kSlice);
  int base = slice_ptr[s], width = (slice_ptr[s + 1] - base) / kSlice;
  double acc = 0.0;
  for (int k = 0; k < width; ++k) acc += fabs(val[base + k * kSlice + lane]);
  out[r] = acc;
}

// dense row-major copy (dense zeroed by the caller): one thread per CSR entry
__global__ void k_to_dense(int64_t nrows, const int* __restrict__ rowptr,
                           const int* __restrict__ col, const int* __restrict__ csr2sell,
                           const double* __restrict__ val, double* __restrict__ dense) {
  int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (r >= nrows) return;
  for (int p = rowptr[r] + (threadIdx.x & 31); p < rowptr[r + 1]; p += 32)
    dense[r * nrows + col[p]] = val[csr2sell[p]];
}

// ----------------------------------------------------------------- SpMV
// y[r*K + j] = sum_c A[r,c] x[c*K + j]; one thread per row on SELL-32.
template <int K>
__global__ void __launch_bounds__(kBlock) k_spmv(int64_t nrows, const int* __restrict__ slice_ptr,
                                                 const int* __restrict__ sell_col,
                                                 const double* __restrict__ val,
                                                 const double* __restrict__ x,
                                                 double* __restrict__ y) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int64_t s = r / kSlice;
  int lane = (int)(r % kSlice);
  int base = __ldg(slice_ptr + s), width = (__ldg(slice_ptr + s + 1) - base) / kSlice;
  double acc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = 0.0;
  for (int k = 0; k < width; ++k) {
    int pos = base + k * kSlice + lane;
    int c = __ldg(sell_col + pos);
    double a = __ldg(val + pos);
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] += a * __ldg(x + (int64_t)c * K + j);
  }
#pragma unroll
  for (int j = 0; j < K; ++j) y[r * K + j] = acc[j];
}

}  // namespace irk

using namespace irk;

// ------------------------------------------------------------------ C ABI
extern "C" {

int irk_mat_from_csr(irk_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz,
                     const int64_t* row_offsets_host, const int64_t* col_indices_host,
                     const double* values_host, irk_mat** out) {
  IRK_REQUIRE(ctx && out, "irk_mat_from_csr: NULL argument");
  IRK_REQUIRE(nrows >= 0 && ncols >= 0 && nnz >= 0, "irk_mat_from_csr: negative size");
  IRK_REQUIRE(nnz < (int64_t)INT32_MAX / 2 && nrows < (int64_t)INT32_MAX / 2 &&
                  ncols < (int64_t)INT32_MAX / 2,
              "irk_mat_from_csr: sizes exceed int32 device indexing");
  IRK_REQUIRE(row_offsets_host[0] == 0 && row_offsets_host[nrows] == nnz,
              "irk_mat_from_csr: row_offsets endpoints inconsistent with nnz");
  std::vector<int> rp(nrows + 1), ci(nnz > 0 ? nnz : 1);
  for (int64_t r = 0; r <= nrows; ++r) rp[r] = (int)row_offsets_host[r];
  for (int64_t p = 0; p < nnz; ++p) {
    int64_t c = col_indices_host[p];
    IRK_REQUIRE(c >= 0 && c < ncols, "irk_mat_from_csr: column index out of range");
    ci[p] = (int)c;
  }
  Pattern* P = pattern_new();
  P->nrows = nrows;
  P->ncols = ncols;
  P->nnz = nnz;
  IRK_CUDA(cudaMalloc(&P->rowptr, (nrows + 1) * sizeof(int)));
  IRK_CUDA(cudaMalloc(&P->col, (nnz + 1) * sizeof(int)));
  IRK_CUDA(cudaMemcpyAsync(P->rowptr, rp.data(), (nrows + 1) * sizeof(int),
                           cudaMemcpyHostToDevice, ctx->stream));
  if (nnz)
    IRK_CUDA(cudaMemcpyAsync(P->col, ci.data(), nnz * sizeof(int), cudaMemcpyHostToDevice,
                             ctx->stream));
  IRK_TRY(pattern_build_sell(ctx, P));
  irk_mat* A = nullptr;
  int st = mat_alloc(ctx, P, &A);
  pattern_release(P);
  IRK_TRY(st);
  if (nnz) {
    double* tmp = nullptr;
    IRK_CUDA(cudaMalloc(&tmp, nnz * sizeof(double)));
    IRK_CUDA(cudaMemcpyAsync(tmp, values_host, nnz * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    IRK_TRY(mat_set_csr_values(ctx, A, tmp));
    IRK_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(tmp);
  } else {
    IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  *out = A;
  return IRK_OK;
}

static int assemble_common(irk_ctx* ctx, int64_t m, int64_t N, int dim, bool q1, irk_mat** Mo,
                           irk_mat** Ko, int full_x = 0) {
  Pattern* P = pattern_new();
  P->nrows = P->ncols = m;
  IRK_CUDA(cudaMalloc(&P->rowptr, (m + 1) * sizeof(int)));
  int* counts = nullptr;
  IRK_CUDA(cudaMalloc(&counts, (m + 1) * sizeof(int)));
  unsigned g = (unsigned)((m + 1 + kBlock - 1) / kBlock);
  double h = 1.0 / (double)N;
  if (q1)
    k_q1_count<<<g, kBlock, 0, ctx->stream>>>(N, m, full_x, counts);
  else
    k_p1_count<<<g, kBlock, 0, ctx->stream>>>(dim, N, m, h, counts);
  IRK_CHECK_LAUNCH(ctx);
  IRK_TRY(scan_exclusive(ctx, counts, P->rowptr, m + 1));
  cudaFree(counts);
  int nnz = 0;
  IRK_CUDA(cudaMemcpy(&nnz, P->rowptr + m, sizeof(int), cudaMemcpyDeviceToHost));
  P->nnz = nnz;
  IRK_CUDA(cudaMalloc(&P->col, ((size_t)nnz + 1) * sizeof(int)));
  double *mv = nullptr, *kv = nullptr;
  IRK_CUDA(cudaMalloc(&mv, ((size_t)nnz + 1) * sizeof(double)));
  IRK_CUDA(cudaMalloc(&kv, ((size_t)nnz + 1) * sizeof(double)));
  if (q1)
    k_q1_fill<<<g, kBlock, 0, ctx->stream>>>(N, m, h, full_x, P->rowptr, P->col, mv, kv);
  else
    k_p1_fill<<<g, kBlock, 0, ctx->stream>>>(dim, N, m, h, P->rowptr, P->col, mv, kv);
  IRK_CHECK_LAUNCH(ctx);
  IRK_TRY(pattern_build_sell(ctx, P));
  irk_mat *M = nullptr, *K = nullptr;
  IRK_TRY(mat_alloc(ctx, P, &M));
  IRK_TRY(mat_alloc(ctx, P, &K));
  pattern_release(P);
  IRK_TRY(mat_set_csr_values(ctx, M, mv));
  IRK_TRY(mat_set_csr_values(ctx, K, kv));
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(mv);
  cudaFree(kv);
  *Mo = M;
  *Ko = K;
  return IRK_OK;
}

int irk_mat_assemble_p1(irk_ctx* ctx, int dim, int64_t N, irk_mat** M, irk_mat** K) {
  IRK_REQUIRE(ctx && M && K, "irk_mat_assemble_p1: NULL argument");
  IRK_REQUIRE(dim >= 1 && dim <= 3, "irk_mat_assemble_p1: dim must be 1, 2 or 3");
  IRK_REQUIRE(N >= 1, "irk_mat_assemble_p1: need N >= 1");
  int64_t m = 1;
  for (int d = 0; d < dim; ++d) m *= (N + 1);
  IRK_REQUIRE(m * (dim == 3 ? 15 : 7) < (int64_t)INT32_MAX / 2,
              "irk_mat_assemble_p1: grid too large for int32 indexing");
  return assemble_common(ctx, m, N, dim, false, M, K);
}

int irk_mat_assemble_q1(irk_ctx* ctx, int64_t N, irk_mat** M, irk_mat** K) {
  IRK_REQUIRE(ctx && M && K, "irk_mat_assemble_q1: NULL argument");
  IRK_REQUIRE(N >= 1, "irk_mat_assemble_q1: need N >= 1");
  int64_t m = (N + 1) * (N + 1);
  IRK_REQUIRE(m * 9 < (int64_t)INT32_MAX / 2, "irk_mat_assemble_q1: grid too large");
  IRK_TRY(assemble_common(ctx, m, N, 2, true, M, K));
  // scipy.sparse.kron (format=None) returns dense BSR blocks when the 1D
  // factor is at least half full, 2 (3N+1) >= (N+1)^2, i.e. N <= 4; the
  // reference's K then stores those blocks' explicit zeros.
  if (2 * (3 * N + 1) >= (N + 1) * (N + 1)) {
    irk_mat *Mb = nullptr, *Kb = nullptr;
    IRK_TRY(assemble_common(ctx, m, N, 2, true, &Mb, &Kb, 1));
    irk_mat_destroy(Mb);
    irk_mat_destroy(*K);
    *K = Kb;
  }
  return IRK_OK;
}

int irk_mat_info(const irk_mat* A, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
  IRK_REQUIRE(A, "irk_mat_info: NULL matrix");
  if (nrows) *nrows = A->pat->nrows;
  if (ncols) *ncols = A->pat->ncols;
  if (nnz) *nnz = A->pat->nnz;
  return IRK_OK;
}

int irk_mat_same_pattern(const irk_mat* A, const irk_mat* B) {
  return (A && B && A->pat == B->pat) ? 1 : 0;
}

int irk_mat_download(irk_ctx* ctx, const irk_mat* A, int64_t* row_offsets_host,
                     int64_t* col_indices_host, double* values_host) {
  IRK_REQUIRE(ctx && A, "irk_mat_download: NULL argument");
  const Pattern* P = A->pat;
  std::vector<int> rp(P->nrows + 1), ci(P->nnz + 1);
  IRK_CUDA(cudaMemcpyAsync(rp.data(), P->rowptr, (P->nrows + 1) * sizeof(int),
                           cudaMemcpyDeviceToHost, ctx->stream));
  if (P->nnz)
    IRK_CUDA(cudaMemcpyAsync(ci.data(), P->col, P->nnz * sizeof(int), cudaMemcpyDeviceToHost,
                             ctx->stream));
  double* tmp = nullptr;
  if (values_host && P->nnz) {
    IRK_CUDA(cudaMalloc(&tmp, P->nnz * sizeof(double)));
    k_gather_vals<<<grid_for(ctx, P->nnz), kBlock, 0, ctx->stream>>>(P->nnz, P->csr2sell, A->val,
                                                                     tmp);
    IRK_CHECK_LAUNCH(ctx);
    IRK_CUDA(cudaMemcpyAsync(values_host, tmp, P->nnz * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
  }
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (tmp) cudaFree(tmp);
  if (row_offsets_host)
    for (int64_t r = 0; r <= P->nrows; ++r) row_offsets_host[r] = rp[r];
  if (col_indices_host)
    for (int64_t p = 0; p < P->nnz; ++p) col_indices_host[p] = ci[p];
  return IRK_OK;
}

int irk_mat_destroy(irk_mat* A) {
  if (!A) return IRK_OK;
  cudaFree(A->val);
  cudaFree(A->uval);
  pattern_release(A->pat);
  delete A;
  return IRK_OK;
}

int irk_mat_union(irk_ctx* ctx, const irk_mat* A, const irk_mat* B, irk_mat** A_out,
                  irk_mat** B_out) {
  IRK_REQUIRE(ctx && A && B && A_out && B_out, "irk_mat_union: NULL argument");
  const Pattern *pa = A->pat, *pb = B->pat;
  IRK_REQUIRE(pa->nrows == pb->nrows && pa->ncols == pb->ncols, "irk_mat_union: shape mismatch");
  int64_t n = pa->nrows;
  Pattern* U = pattern_new();
  U->nrows = n;
  U->ncols = pa->ncols;
  IRK_CUDA(cudaMalloc(&U->rowptr, (n + 1) * sizeof(int)));
  int* counts = nullptr;
  IRK_CUDA(cudaMalloc(&counts, (n + 1) * sizeof(int)));
  unsigned g = (unsigned)((n + 1 + kBlock - 1) / kBlock);
  k_union_count<<<g, kBlock, 0, ctx->stream>>>(n, pa->rowptr, pa->col, pb->rowptr, pb->col,
                                                counts);
  IRK_CHECK_LAUNCH(ctx);
  IRK_TRY(scan_exclusive(ctx, counts, U->rowptr, n + 1));
  cudaFree(counts);
  int nnz = 0;
  IRK_CUDA(cudaMemcpy(&nnz, U->rowptr + n, sizeof(int), cudaMemcpyDeviceToHost));
  U->nnz = nnz;
  IRK_CUDA(cudaMalloc(&U->col, ((size_t)nnz + 1) * sizeof(int)));
  int *mapa = nullptr, *mapb = nullptr;
  IRK_CUDA(cudaMalloc(&mapa, ((size_t)pa->nnz + 1) * sizeof(int)));
  IRK_CUDA(cudaMalloc(&mapb, ((size_t)pb->nnz + 1) * sizeof(int)));
  k_union_fill<<<g, kBlock, 0, ctx->stream>>>(n, pa->rowptr, pa->col, pb->rowptr, pb->col,
                                               U->rowptr, U->col, mapa, mapb);
  IRK_CHECK_LAUNCH(ctx);
  IRK_TRY(pattern_build_sell(ctx, U));
  irk_mat *A2 = nullptr, *B2 = nullptr;
  IRK_TRY(mat_alloc(ctx, U, &A2));
  IRK_TRY(mat_alloc(ctx, U, &B2));
  pattern_release(U);
  if (pa->nnz)
    k_remap_vals<<<grid_for(ctx, pa->nnz), kBlock, 0, ctx->stream>>>(
        pa->nnz, pa->csr2sell, A->val, mapa, U->csr2sell, A2->val);
  IRK_CHECK_LAUNCH(ctx);
  if (pb->nnz)
    k_remap_vals<<<grid_for(ctx, pb->nnz), kBlock, 0, ctx->stream>>>(
        pb->nnz, pb->csr2sell, B->val, mapb, U->csr2sell, B2->val);
  IRK_CHECK_LAUNCH(ctx);
  IRK_TRY(mat_finalize(ctx, A2));
  IRK_TRY(mat_finalize(ctx, B2));
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(mapa);
  cudaFree(mapb);
  *A_out = A2;
  *B_out = B2;
  return IRK_OK;
}

int irk_mat_combine(irk_ctx* ctx, double alpha, const irk_mat* A, double beta, const irk_mat* B,
                    irk_mat** C) {
  IRK_REQUIRE(ctx && A && B && C, "irk_mat_combine: NULL argument");
  IRK_REQUIRE(A->pat == B->pat, "irk_mat_combine: operands must share one pattern");
  irk_mat* out = nullptr;
  IRK_TRY(mat_alloc(ctx, A->pat, &out));
  int64_t n = A->pat->sell_nnz;
  if (n)
    k_combine<<<grid_for(ctx, n), kBlock, 0, ctx->stream>>>(n, alpha, A->val, beta, B->val,
                                                           out->val);
  IRK_CHECK_LAUNCH(ctx);
  IRK_TRY(mat_finalize(ctx, out));
  *C = out;
  return IRK_OK;
}

int irk_mat_constrain(irk_ctx* ctx, const irk_mat* A, const uint8_t* mask_dev, double diag_value,
                      irk_mat** out) {
  IRK_REQUIRE(ctx && A && mask_dev && out, "irk_mat_constrain: NULL argument");
  const Pattern* P = A->pat;
  IRK_REQUIRE(P->nrows == P->ncols, "irk_mat_constrain: square matrix required");
  irk_mat* C = nullptr;
  IRK_TRY(mat_alloc(ctx, A->pat, &C));
  IRK_CUDA(cudaMemcpyAsync(C->val, A->val, P->sell_nnz * sizeof(double), cudaMemcpyDeviceToDevice,
                           ctx->stream));
  int* missing = (int*)ctx->counters + (kNumCounters - 1);
  IRK_CUDA(cudaMemsetAsync(missing, 0, sizeof(int), ctx->stream));
  if (P->nrows)
    k_constrain<<<(unsigned)((P->nrows + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
        P->nrows, P->nslices, P->slice_ptr, P->sell_col, P->diag_pos, mask_dev, diag_value,
        C->val, missing);
  IRK_CHECK_LAUNCH(ctx);
  IRK_TRY(mat_finalize(ctx, C));
  int h_missing = 0;
  IRK_CUDA(cudaMemcpyAsync(&h_missing, missing, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h_missing) {
    irk_mat_destroy(C);
    set_error("irk_mat_constrain: %d constrained rows have no stored diagonal", h_missing);
    return IRK_EINVAL;
  }
  *out = C;
  return IRK_OK;
}

int irk_mat_on_pattern(irk_ctx* ctx, const irk_mat* X, const irk_mat* T, irk_mat** out) {
  IRK_REQUIRE(ctx && X && T && out, "irk_mat_on_pattern: NULL argument");
  const Pattern *px = X->pat, *pt = T->pat;
  IRK_REQUIRE(px->nrows == pt->nrows && px->ncols == pt->ncols, "irk_mat_on_pattern: shape mismatch");
  irk_mat* Y = nullptr;
  IRK_TRY(mat_alloc(ctx, T->pat, &Y));
  if (px == pt) {
    IRK_CUDA(cudaMemcpyAsync(Y->val, X->val, px->sell_nnz * sizeof(double),
                             cudaMemcpyDeviceToDevice, ctx->stream));
    IRK_TRY(mat_finalize(ctx, Y));
    *out = Y;
    return IRK_OK;
  }
  int* map = nullptr;
  IRK_CUDA(cudaMalloc(&map, ((size_t)px->nnz + 1) * sizeof(int)));
  int* missing = (int*)ctx->counters + (kNumCounters - 1);
  IRK_CUDA(cudaMemsetAsync(missing, 0, sizeof(int), ctx->stream));
  if (px->nrows)
    k_on_pattern_map<<<(unsigned)((px->nrows + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
        px->nrows, px->rowptr, px->col, pt->rowptr, pt->col, map, missing);
  IRK_CHECK_LAUNCH(ctx);
  int h_missing = 0;
  IRK_CUDA(cudaMemcpyAsync(&h_missing, missing, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h_missing) {
    cudaFree(map);
    irk_mat_destroy(Y);
    set_error("irk_mat_on_pattern: %d entries are not in the target pattern", h_missing);
    return IRK_EINVAL;
  }
  if (px->nnz)
    k_remap_vals<<<grid_for(ctx, px->nnz), kBlock, 0, ctx->stream>>>(px->nnz, px->csr2sell, X->val,
                                                                     map, pt->csr2sell, Y->val);
  IRK_CHECK_LAUNCH(ctx);
  IRK_TRY(mat_finalize(ctx, Y));
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(map);
  *out = Y;
  return IRK_OK;
}

int irk_mat_semilinear_jacobian(irk_ctx* ctx, const irk_mat* M, const irk_mat* K, double kscale,
                                const double* d_dev, int64_t ld, int64_t off, irk_mat** out) {
  IRK_REQUIRE(ctx && M && K && d_dev && out, "irk_mat_semilinear_jacobian: NULL argument");
  IRK_REQUIRE(M->pat == K->pat, "irk_mat_semilinear_jacobian: M and K must share a pattern");
  irk_mat* J = nullptr;
  IRK_TRY(mat_alloc(ctx, M->pat, &J));
  int64_t n = M->pat->nrows;
  if (n)
    k_semi_jac<<<(unsigned)((n + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
        n, M->pat->slice_ptr, M->pat->sell_col, M->val, K->val, kscale, d_dev, ld, off, J->val);
  IRK_CHECK_LAUNCH(ctx);
  IRK_TRY(mat_finalize(ctx, J));
  *out = J;
  return IRK_OK;
}

int irk_mat_diagonal(irk_ctx* ctx, const irk_mat* A, double* diag_dev) {
  IRK_REQUIRE(ctx && A && diag_dev, "irk_mat_diagonal: NULL argument");
  int64_t n = A->pat->nrows;
  if (n)
    k_diag<<<(unsigned)((n + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
        n, A->pat->diag_pos, A->val, diag_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_mat_absrowsum(irk_ctx* ctx, const irk_mat* A, double* out_dev) {
  IRK_REQUIRE(ctx && A && out_dev, "irk_mat_absrowsum: NULL argument");
  int64_t n = A->pat->nrows;
  if (n)
    k_absrowsum<<<(unsigned)((n + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
        n, A->pat->slice_ptr, A->val, out_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_mat_to_dense(irk_ctx* ctx, const irk_mat* A, double* dense_dev) {
  IRK_REQUIRE(ctx && A && dense_dev, "irk_mat_to_dense: NULL argument");
  IRK_REQUIRE(A->pat->nrows == A->pat->ncols, "irk_mat_to_dense: square matrices only");
  int64_t n = A->pat->nrows;
  if (!n) return IRK_OK;
  IRK_CUDA(cudaMemsetAsync(dense_dev, 0, (size_t)n * n * sizeof(double), ctx->stream));
  const int rows_per_block = kBlock / 32;
  k_to_dense<<<(unsigned)((n + rows_per_block - 1) / rows_per_block), kBlock, 0, ctx->stream>>>(
      n, A->pat->rowptr, A->pat->col, A->pat->csr2sell, A->val, dense_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_mat_rowsum(irk_ctx* ctx, const irk_mat* A, double* rowsum_dev) {
  IRK_REQUIRE(ctx && A && rowsum_dev, "irk_mat_rowsum: NULL argument");
  int64_t n = A->pat->nrows;
  if (n)
    k_rowsum<<<(unsigned)((n + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
        n, A->pat->slice_ptr, A->val, rowsum_dev);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

}  // extern "C"

namespace irk {
// y[r * ldy] = sum_c A[r, c] x[c * ldx] (A dense row-major n x n): one warp
// per row, lanes stride the row (coalesced), x from L1/L2
__global__ void __launch_bounds__(kBlock)
    k_dense_gemv(int64_t n, const double* __restrict__ A, const double* __restrict__ x,
                 int64_t ldx, double* __restrict__ y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (r >= n) return;
  const double* a = A + r * n;
  double acc = 0.0;
  for (int64_t c = lane; c < n; c += 32) acc += __ldg(a + c) * __ldg(x + c * ldx);
  acc = warp_sum(acc);
  if (lane == 0) y[r * ldy] = acc;
}
}  // namespace irk

extern "C" {

int irk_dense_gemv(irk_ctx* ctx, int64_t n, const double* A_dev, const double* x_dev,
                   int64_t ldx, double* y_dev, int64_t ldy) {
  IRK_REQUIRE(ctx && A_dev && x_dev && y_dev, "irk_dense_gemv: NULL argument");
  IRK_REQUIRE(n >= 0 && ldx >= 1 && ldy >= 1, "irk_dense_gemv: bad sizes");
  if (n == 0) return IRK_OK;
  const unsigned g = (unsigned)((n * 32 + kBlock - 1) / kBlock);
  k_dense_gemv<<<g, kBlock, 0, ctx->stream>>>(n, A_dev, x_dev, ldx, y_dev, ldy);
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

int irk_spmv(irk_ctx* ctx, const irk_mat* A, int k, const double* x_dev, double* y_dev) {
  IRK_REQUIRE(ctx && A && x_dev && y_dev, "irk_spmv: NULL argument");
  IRK_REQUIRE(k >= 1 && k <= 8, "irk_spmv: 1 <= k <= 8 right-hand sides");
  const Pattern* P = A->pat;
  int64_t n = P->nrows;
  if (n == 0) return IRK_OK;
  unsigned g = (unsigned)((n + kBlock - 1) / kBlock);
#define IRK_SPMV_CASE(KK)                                                                    \
  case KK:                                                                                   \
    k_spmv<KK><<<g, kBlock, 0, ctx->stream>>>(n, P->slice_ptr, P->sell_col, A->val, x_dev, \
                                              y_dev);                                        \
    break;
  switch (k) {
    IRK_SPMV_CASE(1)
    IRK_SPMV_CASE(2)
    IRK_SPMV_CASE(3)
    IRK_SPMV_CASE(4)
    IRK_SPMV_CASE(5)
    IRK_SPMV_CASE(6)
    IRK_SPMV_CASE(7)
    IRK_SPMV_CASE(8)
  }
#undef IRK_SPMV_CASE
  IRK_CHECK_LAUNCH(ctx);
  return IRK_OK;
}

}  // extern "C"
