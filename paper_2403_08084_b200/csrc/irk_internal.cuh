// Internal declarations shared by the libirk translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <climits>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <tuple>
#include <utility>
#include <utility>
#include <vector>

#include "../../include/irk.h"

namespace irk {

constexpr int kSlice = 32;          // SELL slice height == warp size
constexpr int kBlock = 256;         // default threads per block
constexpr int kMaxStages = 8;       // s <= 8 on every stage kernel
constexpr int kMaxBasis = 64;       // Krylov basis vectors per fused call

void set_error(const char* fmt, ...);

struct Pattern {
  std::atomic<int> refs{1};
  int64_t nrows = 0, ncols = 0, nnz = 0;
  // CSR (int32 on device)
  int* rowptr = nullptr;     // nrows + 1
  int* col = nullptr;        // nnz
  // SELL-32: slice s holds rows [32 s, 32 s + 32); entry k of lane l lives at
  // slice_ptr[s] + 32 k + l.  Padding entries carry col = own row (or 0) and
  // value 0.
  int64_t nslices = 0, sell_nnz = 0;
  int* slice_ptr = nullptr;  // nslices + 1
  int* sell_col = nullptr;   // sell_nnz
  int* csr2sell = nullptr;   // nnz: SELL position of CSR entry p
  int* diag_pos = nullptr;   // nrows: SELL position of (r, r) or -1
  int maxw = 0;              // widest slice (entries per row)
  int ellw = 0;              // > 0: every slice padded to this width (ELL-32)
  // Slot-uniform column compression (a CSR-DU-style delta code for SELL):
  // slot q = slice_ptr[s]/32 + k covers entry k of the 32 rows of slice s.
  // colhdr[q] = d when every lane's column is row + d, else kNonUniform
  // (read sell_col[pos]).
  int* colhdr = nullptr;     // sell_nnz / 32
  // max over slot-uniform slices of the window rows (win_layout); 0 if none
  int win_rows = 0;
  // stencil-aligned ELL patterns: the ellw column offsets of every full row
  // (slot k of a stencil row holds column row + stencil[k]); else empty
  std::vector<int> stencil;
};

constexpr int kNonUniform = INT_MIN;

}  // namespace irk

struct irk_mat {
  irk::Pattern* pat = nullptr;
  double* val = nullptr;   // SELL order, sell_nnz entries
  // Slot-uniform value compression (CSR-VI-style): uval[q] = the common
  // value of slot q when all 32 lanes agree bit for bit, else NaN (read
  // val[pos]).
  double* uval = nullptr;  // sell_nnz / 32
};

struct irk_ctx {
  int device = 0;
  cudaStream_t stream = 0;
  int num_sms = 148;
  int64_t launches = 0;
  // reduction scratch: block partials and last-block counters
  double* red = nullptr;
  size_t red_cap = 0;  // doubles
  unsigned int* counters = nullptr;  // kNumCounters
  // generic device workspace
  char* work = nullptr;
  size_t work_cap = 0;
  // pinned host mirror for small status blocks
  char* pinned = nullptr;
  size_t pinned_cap = 0;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  // CUDA-graph cache for fixed launch sequences (inner-solver chunks): a
  // graph is a pure function of its key (kernels + every launch argument),
  // captured on a private stream and replayed on `stream`.
  struct GraphEntry {
    std::string key;
    cudaGraphExec_t exec;
    int64_t kernels;          // per launch (straight-line part)
    int64_t body_kernels = 0;  // per pass of a conditional WHILE body
    // kernel nodes whose arguments change from launch to launch (updated
    // with cudaGraphExecKernelNodeSetParams before every replay); their
    // handles belong to `graph`, which is kept alive for them
    cudaGraph_t graph = nullptr;
    cudaGraphNode_t unode[4] = {};
    int n_unode = 0;
  };
  std::vector<GraphEntry> graphs;
  cudaStream_t cap_stream = nullptr;
  // Deferred solve status (irk_ctx_log_enable): inner solves called with
  // NULL its/relres do not synchronise; each appends (iterations, code,
  // loop passes, kernels per pass) to this device log, read back in one copy
  // by irk_ctx_log_take.
  int log_on = 0;
  int* solve_log = nullptr;  // 4 ints per entry
  int log_cap = 0;
  int64_t log_n = 0;
  // Independent inner solves run concurrently (irk::run_forked): system
  // k >= 1 on auxiliary context aux[k-1] (own stream, workspace, reduction
  // scratch and graph cache), forked from and joined into `stream`.
  std::vector<irk_ctx*> aux;
  cudaStream_t own_stream = nullptr;  // created by and owned by this context
  cudaEvent_t fork_ev = nullptr;
  cudaEvent_t join_ev = nullptr;
};

namespace irk {

constexpr int kNumCounters = 16;

// error plumbing -----------------------------------------------------------
#define IRK_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ::irk::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                       cudaGetErrorString(_e));                               \
      return IRK_ECUDA;                                                       \
    }                                                                         \
  } while (0)

#define IRK_CHECK_LAUNCH(ctx)                                                 \
  do {                                                                        \
    (ctx)->launches++;                                                        \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess) {                                                  \
      ::irk::set_error("%s:%d kernel launch: %s", __FILE__, __LINE__,         \
                       cudaGetErrorString(_e));                               \
      return IRK_ECUDA;                                                       \
    }                                                                         \
  } while (0)

#define IRK_REQUIRE(cond, ...)                                                \
  do {                                                                        \
    if (!(cond)) {                                                            \
      ::irk::set_error(__VA_ARGS__);                                          \
      return IRK_EINVAL;                                                      \
    }                                                                         \
  } while (0)

#define IRK_TRY(expr)                                                         \
  do {                                                                        \
    int _st = (expr);                                                         \
    if (_st != IRK_OK) return _st;                                            \
  } while (0)

// context helpers ------------------------------------------------------------
int ensure_red(irk_ctx* ctx, size_t doubles);
int ensure_work(irk_ctx* ctx, size_t bytes);
int ensure_pinned(irk_ctx* ctx, size_t bytes);
int log_reserve(irk_ctx* ctx, int n = 1);
// auxiliary context k (lazily created, own non-blocking stream)
int aux_ctx(irk_ctx* ctx, int k, irk_ctx** out);

// Run fn(k, c) for the n independent systems k = 0..n-1.  Concurrent when
// `concurrent` (deferred solves: no host round trip inside fn) and the
// stream is not being captured: system k >= 1 runs on auxiliary context
// k-1, whose stream waits on an event of ctx->stream and is joined back
// into it; system 0 runs on ctx.  The latency-bound coarse levels of one
// system's V-cycles then overlap with the other systems' kernels.  Deferred
// log entries land in ctx's log in system order, launches are counted on
// ctx.  Sequential otherwise.
template <typename F>
int run_forked(irk_ctx* ctx, int n, bool concurrent, F&& fn) {
  static const bool fork_off = getenv("IRK_NO_FORK") != nullptr;  // A/B: one by one
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (fork_off) concurrent = false;
  if (concurrent && n > 1) {
    if (cudaStreamIsCapturing(ctx->stream, &cap) != cudaSuccess) cap = cudaStreamCaptureStatusActive;
  }
  if (!concurrent || n <= 1 || cap != cudaStreamCaptureStatusNone) {
    for (int k = 0; k < n; ++k) IRK_TRY(fn(k, ctx));
    return IRK_OK;
  }
  if (ctx->log_on) IRK_TRY(log_reserve(ctx, n));
  irk_ctx* a = nullptr;
  IRK_TRY(aux_ctx(ctx, n - 2, &a));
  IRK_CUDA(cudaEventRecord(ctx->fork_ev, ctx->stream));
  const int64_t base = ctx->log_n;
  int status = IRK_OK;
  int forked = 0;
  for (int k = 1; k < n && status == IRK_OK; ++k, ++forked) {
    a = ctx->aux[k - 1];
    IRK_CUDA(cudaStreamWaitEvent(a->stream, ctx->fork_ev, 0));
    a->log_on = ctx->log_on;
    a->solve_log = ctx->solve_log;
    a->log_cap = ctx->log_cap;
    a->log_n = base + k;
    const int64_t l0 = a->launches;
    status = fn(k, a);
    ctx->launches += a->launches - l0;
    a->solve_log = nullptr;
    a->log_on = 0;
    a->log_n = 0;
    IRK_CUDA(cudaEventRecord(a->join_ev, a->stream));
  }
  if (status == IRK_OK) {
    ctx->log_n = base;
    status = fn(0, ctx);
    ctx->log_n = base + n;
  }
  for (int k = 0; k < forked; ++k)
    IRK_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux[k]->join_ev, 0));
  return status;
}
// Byte-string key builder for the graph cache.
struct GraphKey {
  std::string k;
  template <class V>
  GraphKey& add(const V& v) {
    k.append(reinterpret_cast<const char*>(&v), sizeof(V));
    return *this;
  }
};

// Replay the cached graph for `key`, or capture `body(stream)` (a fixed
// kernel sequence that must not synchronise) into one, then replay it on
// ctx->stream.  IRK_NO_GRAPH=1 runs body directly on ctx->stream.
template <class F>
int graph_launch(irk_ctx* ctx, const std::string& key, F&& body) {
  static const bool off = getenv("IRK_NO_GRAPH") != nullptr;
  if (off) return body(ctx->stream);
  for (auto& g : ctx->graphs) {
    if (g.key == key) {
      IRK_CUDA(cudaGraphLaunch(g.exec, ctx->stream));
      ctx->launches += g.kernels;
      return IRK_OK;
    }
  }
  if (!ctx->cap_stream)
    IRK_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
  const int64_t l0 = ctx->launches;
  IRK_CUDA(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
  const int rc = body(ctx->cap_stream);
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(ctx->cap_stream, &graph);
  if (rc != IRK_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  IRK_CUDA(e);
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  IRK_CUDA(ei);
  if (ctx->graphs.size() >= 64) {
    cudaGraphExecDestroy(ctx->graphs.front().exec);
    if (ctx->graphs.front().graph) cudaGraphDestroy(ctx->graphs.front().graph);
    ctx->graphs.erase(ctx->graphs.begin());
  }
  ctx->graphs.push_back({key, exec, ctx->launches - l0});
  IRK_CUDA(cudaGraphLaunch(exec, ctx->stream));
  return IRK_OK;
}

// Graph-resident loop: a graph holding one conditional WHILE node whose
// body is `body(stream, handle)` (captured; the body sets the condition
// with cudaGraphSetConditional, default 1 at every launch).  Cached like
// graph_launch; replayed on ctx->stream.
// *body_kernels (optional) receives the kernel count of one body pass.
template <class F>
int graph_launch_while(irk_ctx* ctx, const std::string& key, F&& body,
                       int64_t* body_kernels = nullptr) {
  for (auto& g : ctx->graphs) {
    if (g.key == key) {
      IRK_CUDA(cudaGraphLaunch(g.exec, ctx->stream));
      if (body_kernels) *body_kernels = g.kernels;
      return IRK_OK;
    }
  }
  if (!ctx->cap_stream)
    IRK_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
  cudaGraph_t graph = nullptr;
  IRK_CUDA(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  if (e == cudaSuccess) e = cudaGraphAddNode(&node, graph, nullptr, 0, &np);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    IRK_CUDA(e);
  }
  cudaGraph_t bodyg = np.conditional.phGraph_out[0];
  const int64_t l0 = ctx->launches;
  e = cudaStreamBeginCaptureToGraph(ctx->cap_stream, bodyg, nullptr, nullptr, 0,
                                    cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    IRK_CUDA(e);
  }
  const int rc = body(ctx->cap_stream, h);
  cudaGraph_t got = nullptr;
  e = cudaStreamEndCapture(ctx->cap_stream, &got);
  if (rc != IRK_OK || e != cudaSuccess) {
    cudaGraphDestroy(graph);
    if (rc != IRK_OK) return rc;
    IRK_CUDA(e);
  }
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  IRK_CUDA(e);
  if (ctx->graphs.size() >= 64) {
    cudaGraphExecDestroy(ctx->graphs.front().exec);
    if (ctx->graphs.front().graph) cudaGraphDestroy(ctx->graphs.front().graph);
    ctx->graphs.erase(ctx->graphs.begin());
  }
  ctx->graphs.push_back({key, exec, ctx->launches - l0});
  ctx->launches = l0;  // counted per executed body pass by the caller
  if (body_kernels) *body_kernels = ctx->graphs.back().kernels;
  IRK_CUDA(cudaGraphLaunch(exec, ctx->stream));
  return IRK_OK;
}

// One graph = a straight-line prefix `pre(stream)` followed by a conditional
// WHILE node whose body is `body(stream, handle)`.  Replaces a prefix graph
// launch + a separate WHILE-graph launch: measured on B200 inside the
// multigrid-PCG solves, the second launch cost ~150 us of GPU idle per solve
// (profiles/r02), a sequence in one graph costs a few us.  Cached like
// graph_launch; the prefix kernels are counted per launch, *body_kernels
// receives the kernel count of one body pass.  `pre(stream, handle)` may
// launch a kernel that sets the loop condition (default 1 at every launch).
// The kernel node a capturing stream ends in (the kernel just captured).
inline cudaGraphNode_t capture_tail(cudaStream_t s) {
  cudaStreamCaptureStatus st;
  const cudaGraphNode_t* deps = nullptr;
  size_t n = 0;
  if (cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &n) != cudaSuccess || n != 1)
    return nullptr;
  return deps[0];
}

struct NoPost {
  int operator()(cudaStream_t) const { return IRK_OK; }
};
struct NoUpdate {
  int operator()(cudaGraphExec_t, const cudaGraphNode_t*) const { return IRK_OK; }
};

// `post(stream)` (optional) is captured after the WHILE node.  `unodes`
// (optional, n_unodes <= 4 handles recorded by pre / post with
// capture_tail) are kernel nodes whose arguments differ between launches:
// `update(exec, nodes)` sets them before every replay of the cached graph
// (the first launch runs with the captured arguments).
template <class F, class B, class Pst = NoPost, class U = NoUpdate>
int graph_launch_prefix_while(irk_ctx* ctx, const std::string& key, F&& pre, B&& body,
                              int64_t* body_kernels, Pst&& post = NoPost{},
                              const cudaGraphNode_t* unodes = nullptr, int n_unodes = 0,
                              U&& update = NoUpdate{}) {
  for (auto& g : ctx->graphs) {
    if (g.key == key) {
      if (g.n_unode) IRK_TRY(update(g.exec, g.unode));
      IRK_CUDA(cudaGraphLaunch(g.exec, ctx->stream));
      ctx->launches += g.kernels;
      *body_kernels = g.body_kernels;
      return IRK_OK;
    }
  }
  if (!ctx->cap_stream)
    IRK_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
  cudaGraph_t graph = nullptr;
  IRK_CUDA(cudaGraphCreate(&graph, 0));
  const int64_t l0 = ctx->launches;
  cudaError_t e = cudaStreamBeginCaptureToGraph(ctx->cap_stream, graph, nullptr, nullptr, 0,
                                                cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    IRK_CUDA(e);
  }
  // the handle exists before the prefix is captured: its last kernel may
  // clear the condition (a solve that finished inside the prefix)
  cudaGraphConditionalHandle h{};
  e = cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault);
  int rc = e == cudaSuccess ? pre(ctx->cap_stream, h) : IRK_ECUDA;
  // the conditional node joins the capture after the prefix's sink nodes
  cudaGraphNode_t node = nullptr;
  cudaGraph_t bodyg = nullptr;
  if (rc == IRK_OK) {
    cudaStreamCaptureStatus cst;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    e = cudaStreamGetCaptureInfo(ctx->cap_stream, &cst, nullptr, nullptr, &deps, &ndeps);
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    if (e == cudaSuccess) e = cudaGraphAddNode(&node, graph, deps, ndeps, &np);
    if (e == cudaSuccess) {
      bodyg = np.conditional.phGraph_out[0];
      e = cudaStreamUpdateCaptureDependencies(ctx->cap_stream, &node, 1,
                                              cudaStreamSetCaptureDependencies);
    }
    if (e == cudaSuccess) rc = post(ctx->cap_stream);
  }
  cudaGraph_t got = nullptr;
  const cudaError_t ee = cudaStreamEndCapture(ctx->cap_stream, &got);
  if (rc != IRK_OK || e != cudaSuccess || ee != cudaSuccess) {
    cudaGraphDestroy(graph);
    if (rc != IRK_OK) return rc;
    IRK_CUDA(e != cudaSuccess ? e : ee);
  }
  const int64_t pre_kernels = ctx->launches - l0;
  e = cudaStreamBeginCaptureToGraph(ctx->cap_stream, bodyg, nullptr, nullptr, 0,
                                    cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    IRK_CUDA(e);
  }
  rc = body(ctx->cap_stream, h);
  e = cudaStreamEndCapture(ctx->cap_stream, &got);
  if (rc != IRK_OK || e != cudaSuccess) {
    cudaGraphDestroy(graph);
    if (rc != IRK_OK) return rc;
    IRK_CUDA(e);
  }
  const int64_t bk = ctx->launches - l0 - pre_kernels;
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  bool keep = n_unodes > 0 && n_unodes <= 4 && e == cudaSuccess;
  for (int i = 0; keep && i < n_unodes; ++i) keep = unodes[i] != nullptr;
  if (n_unodes > 0 && !keep && e == cudaSuccess) {
    // the caller's arguments cannot be updated in this graph: not cacheable
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    set_error("graph_launch_prefix_while: updatable kernel nodes not recorded");
    return IRK_ECUDA;
  }
  if (!keep) cudaGraphDestroy(graph);
  IRK_CUDA(e);
  if (ctx->graphs.size() >= 64) {
    cudaGraphExecDestroy(ctx->graphs.front().exec);
    if (ctx->graphs.front().graph) cudaGraphDestroy(ctx->graphs.front().graph);
    ctx->graphs.erase(ctx->graphs.begin());
  }
  ctx->graphs.push_back({key, exec, pre_kernels, bk});
  ctx->launches = l0 + pre_kernels;  // body passes are counted by the caller
  *body_kernels = bk;
  if (keep) {
    auto& ge = ctx->graphs.back();
    ge.graph = graph;
    ge.n_unode = n_unodes;
    for (int i = 0; i < n_unodes; ++i) ge.unode[i] = unodes[i];
    // arguments that were not known at capture time (the body's kernel count)
    IRK_TRY(update(ge.exec, ge.unode));
  }
  ctx->launches = l0 + pre_kernels;  // body passes are counted by the caller
  *body_kernels = bk;
  IRK_CUDA(cudaGraphLaunch(exec, ctx->stream));
  return IRK_OK;
}

// Programmatic dependent launch (PDL): kernels of the inner-solver loops are
// launched with programmatic stream serialisation, so a kernel's CTAs are
// scheduled while its predecessor drains and only wait (griddepcontrol.wait)
// for the predecessor's completion and memory before touching data; each
// kernel immediately allows its own dependents to launch.  Every kernel
// launched through irk::launch() must start with IRK_PDL_ENTER() (a no-op
// when launched without the attribute).  Env IRK_NO_PDL disables it.
#define IRK_PDL_ENTER()                                    \
  do {                                                     \
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   \
    asm volatile("griddepcontrol.launch_dependents;\n");   \
  } while (0)

inline bool pdl_on() {
  static const bool on = getenv("IRK_NO_PDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// Launch without the programmatic-serialisation attribute (a kernel whose
// predecessor in a captured graph is not a kernel node).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_plain(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s,
                                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// New arguments for a kernel node of an instantiated graph (same kernel,
// grid and block as captured; arguments converted to the kernel's types).
template <typename Tup, size_t... I>
inline void tuple_ptrs(Tup& t, void** out, std::index_sequence<I...>) {
  ((out[I] = (void*)&std::get<I>(t)), ...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t exec_set_kernel_args(cudaGraphExec_t exec, cudaGraphNode_t node,
                                        void (*k)(KArgs...), dim3 g, dim3 b, Args&&... args) {
  static_assert(sizeof...(KArgs) == sizeof...(Args), "exec_set_kernel_args: argument count");
  std::tuple<std::remove_cv_t<KArgs>...> vals(std::forward<Args>(args)...);
  void* ptrs[sizeof...(KArgs)];
  tuple_ptrs(vals, ptrs, std::index_sequence_for<KArgs...>{});
  cudaKernelNodeParams kp = {};
  kp.func = (void*)k;
  kp.gridDim = g;
  kp.blockDim = b;
  kp.sharedMemBytes = 0;
  kp.kernelParams = ptrs;
  kp.extra = nullptr;
  return cudaGraphExecKernelNodeSetParams(exec, node, &kp);
}

inline int grid_for(const irk_ctx* ctx, int64_t work_items, int per_block = kBlock,
                    int blocks_per_sm = 8) {
  int64_t g = (work_items + per_block - 1) / per_block;
  int64_t cap = (int64_t)ctx->num_sms * blocks_per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// pattern / matrix helpers ---------------------------------------------------
Pattern* pattern_new();
void pattern_retain(Pattern* p);
void pattern_release(Pattern* p);
// Build SELL arrays for a pattern whose CSR arrays are already on device.
int pattern_build_sell(irk_ctx* ctx, Pattern* p);
// Allocate a matrix on pattern p (retains p) with zeroed SELL values.
int mat_alloc(irk_ctx* ctx, Pattern* p, irk_mat** out);
// Scatter CSR-ordered device values into the SELL array of A.
int mat_set_csr_values(irk_ctx* ctx, irk_mat* A, const double* csr_val_dev);
// Recompute the slot-uniform value headers after A->val changed.
int mat_finalize(irk_ctx* ctx, irk_mat* A);

// Read entry k of row `row` (lane `lane` of slice `s`, slot base `q0`,
// position base `base`) through the slot-uniform headers.
__device__ __forceinline__ int sell_col_at(const int* __restrict__ colhdr,
                                          const int* __restrict__ sell_col, int q, int pos,
                                          int64_t row) {
  int h = __ldg(colhdr + q);
  return h != kNonUniform ? (int)(row + h) : __ldg(sell_col + pos);
}
__device__ __forceinline__ double sell_val_at(const double* __restrict__ uval,
                                              const double* __restrict__ val, int q, int pos) {
  double u = __ldg(uval + q);
  return isnan(u) ? __ldg(val + pos) : u;
}

// Window layout of a slot-uniform slice (all lanes of the warp call this;
// lane k < width holds the slot offset d_k = colhdr[q0 + k]).  Offsets are
// grouped into windows of stage-block rows: a new window starts at slot 0,
// at a decreasing offset (ELL padding) or after a gap of more than kWinGap
// rows; window w covers rows [r0 + dfirst_w, r0 + d_last_w + 32).  Returns
// the total number of window rows; per lane: `row` = buffer row of slot
// `lane` for lane 0 of the slice, and on window-end lanes (bit set in
// `ends`) `rows`, `dfirst` and `wbase` (buffer row of the window start).
constexpr int kWinGap = 8;
struct WinLayout {
  int total, row, rows, dfirst, wbase;
  unsigned ends;
};
__device__ __forceinline__ WinLayout win_layout(int d, int width) {
  const int lane = threadIdx.x & 31;
  const int dprev = __shfl_up_sync(0xffffffffu, d, 1);
  const bool start = lane < width && (lane == 0 || d < dprev || d - dprev > kWinGap);
  const unsigned sb = __ballot_sync(0xffffffffu, start);
  const unsigned upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
  const int first_lane = 31 - __clz(sb & upto);
  const int dfirst = __shfl_sync(0xffffffffu, d, first_lane & 31);
  const bool next_start = lane < 31 && ((sb >> (lane + 1)) & 1u);
  const bool is_end = lane < width && (lane == width - 1 || next_start);
  const int rows = is_end ? d - dfirst + 32 : 0;
  int incl = rows;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  WinLayout L;
  L.total = __shfl_sync(0xffffffffu, incl, 31);
  L.ends = __ballot_sync(0xffffffffu, is_end);
  const unsigned from = lane == 0 ? 0xffffffffu : ~((1u << lane) - 1u);
  const int end_lane = __ffs(L.ends & from) - 1;
  L.wbase = incl - rows;
  L.row = __shfl_sync(0xffffffffu, L.wbase, end_lane & 31) + (d - dfirst);
  L.rows = rows;
  L.dfirst = dfirst;
  return L;
}

// warp / block reductions ----------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction of NV values per thread into red_smem[0..NV).
// Requires blockDim.x == kBlock.  Result valid in all threads after return.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem /* >= 8*NV */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) smem[warp * NV + j] = v[j];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double t = (lane < (kBlock / 32)) ? smem[lane * NV + j] : 0.0;
      t = warp_sum(t);
      v[j] = t;
    }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < NV; ++j) smem[j] = v[j];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = smem[j];
  __syncthreads();
}

}  // namespace irk
