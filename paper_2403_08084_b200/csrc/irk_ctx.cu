// Context lifetime, error reporting and workspace management.
#include <cstdarg>
#include <cstring>

#include <algorithm>

#include "irk_internal.cuh"

namespace irk {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int ensure_red(irk_ctx* ctx, size_t doubles) {
  if (doubles <= ctx->red_cap) return IRK_OK;
  size_t cap = doubles < 4096 ? 4096 : doubles * 2;
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->red) IRK_CUDA(cudaFree(ctx->red));
  ctx->red = nullptr;
  IRK_CUDA(cudaMalloc(&ctx->red, cap * sizeof(double)));
  ctx->red_cap = cap;
  return IRK_OK;
}

int ensure_work(irk_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->work_cap) return IRK_OK;
  size_t cap = bytes + bytes / 4 + (1 << 20);
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->work) IRK_CUDA(cudaFree(ctx->work));
  ctx->work = nullptr;
  IRK_CUDA(cudaMalloc(&ctx->work, cap));
  ctx->work_cap = cap;
  return IRK_OK;
}

int ensure_pinned(irk_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->pinned_cap) return IRK_OK;
  size_t cap = bytes < 65536 ? 65536 : bytes * 2;
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->pinned) IRK_CUDA(cudaFreeHost(ctx->pinned));
  ctx->pinned = nullptr;
  IRK_CUDA(cudaHostAlloc((void**)&ctx->pinned, cap, cudaHostAllocDefault));
  ctx->pinned_cap = cap;
  return IRK_OK;
}

}  // namespace irk

using namespace irk;

extern "C" {

const char* irk_last_error(void) { return g_last_error.c_str(); }

const char* irk_version(void) { return "libirk 0.1.0 sm_100a"; }

int irk_ctx_create(int device, irk_ctx** out) {
  IRK_REQUIRE(out != nullptr, "irk_ctx_create: out is NULL");
  int ndev = 0;
  IRK_CUDA(cudaGetDeviceCount(&ndev));
  IRK_REQUIRE(device >= 0 && device < ndev, "irk_ctx_create: device %d of %d", device, ndev);
  IRK_CUDA(cudaSetDevice(device));
  irk_ctx* c = new irk_ctx();
  c->device = device;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) c->num_sms = prop.multiProcessorCount;
  if (cudaMalloc(&c->counters, kNumCounters * sizeof(unsigned int)) != cudaSuccess ||
      cudaMemset(c->counters, 0, kNumCounters * sizeof(unsigned int)) != cudaSuccess) {
    set_error("irk_ctx_create: counter allocation failed");
    delete c;
    return IRK_ECUDA;
  }
  for (auto& e : c->ev) {
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      set_error("irk_ctx_create: event creation failed");
      return IRK_ECUDA;
    }
  }
  int st = ensure_red(c, 1 << 16);
  if (st != IRK_OK) return st;
  st = ensure_pinned(c, 1 << 16);
  if (st != IRK_OK) return st;
  *out = c;
  return IRK_OK;
}

int irk_ctx_destroy(irk_ctx* ctx) {
  if (!ctx) return IRK_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->red) cudaFree(ctx->red);
  if (ctx->counters) cudaFree(ctx->counters);
  if (ctx->work) cudaFree(ctx->work);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& g : ctx->graphs) {
    cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
  }
  for (irk_ctx* a : ctx->aux) irk_ctx_destroy(a);
  if (ctx->solve_log) cudaFree(ctx->solve_log);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
  delete ctx;
  return IRK_OK;
}

int irk_ctx_set_stream(irk_ctx* ctx, void* stream) {
  IRK_REQUIRE(ctx, "irk_ctx_set_stream: NULL context");
  ctx->stream = (cudaStream_t)stream;
  return IRK_OK;
}

int irk_ctx_synchronize(irk_ctx* ctx) {
  IRK_REQUIRE(ctx, "irk_ctx_synchronize: NULL context");
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  return IRK_OK;
}

int64_t irk_ctx_launch_count(const irk_ctx* ctx) { return ctx ? ctx->launches : -1; }

}  // extern "C"

namespace irk {
// Room for n more deferred-solve entries: the log doubles when full (a rare,
// synchronous event; entries already written are carried over in order).
int log_reserve(irk_ctx* ctx, int n) {
  if (ctx->log_n + n <= ctx->log_cap) return IRK_OK;
  int cap = ctx->log_cap * 2;
  while (ctx->log_n + n > cap) cap *= 2;
  int* fresh = nullptr;
  IRK_CUDA(cudaMalloc(&fresh, (size_t)cap * 4 * sizeof(int)));
  IRK_CUDA(cudaMemcpyAsync(fresh, ctx->solve_log, (size_t)ctx->log_n * 4 * sizeof(int),
                           cudaMemcpyDeviceToDevice, ctx->stream));
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  IRK_CUDA(cudaFree(ctx->solve_log));
  ctx->solve_log = fresh;
  ctx->log_cap = cap;
  return IRK_OK;
}

int aux_ctx(irk_ctx* ctx, int k, irk_ctx** out) {
  while ((int)ctx->aux.size() <= k) {
    irk_ctx* a = nullptr;
    IRK_TRY(irk_ctx_create(ctx->device, &a));
    if (cudaStreamCreateWithFlags(&a->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&a->join_ev, cudaEventDisableTiming) != cudaSuccess) {
      irk_ctx_destroy(a);
      set_error("aux_ctx: stream/event creation failed");
      return IRK_ECUDA;
    }
    a->stream = a->own_stream;
    ctx->aux.push_back(a);
  }
  if (!ctx->fork_ev) IRK_CUDA(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
  *out = ctx->aux[k];
  return IRK_OK;
}
}  // namespace irk

extern "C" {

int irk_ctx_log_enable(irk_ctx* ctx, int on) {
  IRK_REQUIRE(ctx, "irk_ctx_log_enable: NULL context");
  if (on && !ctx->solve_log) {
    ctx->log_cap = 4096;
    IRK_CUDA(cudaMalloc(&ctx->solve_log, (size_t)ctx->log_cap * 4 * sizeof(int)));
  }
  ctx->log_on = on ? 1 : 0;
  ctx->log_n = 0;
  return IRK_OK;
}

int irk_ctx_log_size(const irk_ctx* ctx, int64_t* n_out) {
  IRK_REQUIRE(ctx && n_out, "irk_ctx_log_size: NULL argument");
  *n_out = ctx->log_n;
  return IRK_OK;
}

int irk_ctx_log_take(irk_ctx* ctx, int* out_host, int max_entries, int* n_out) {
  IRK_REQUIRE(ctx && n_out, "irk_ctx_log_take: NULL argument");
  const int n = (int)std::min<int64_t>(ctx->log_n, max_entries);
  if (n > 0) {
    IRK_REQUIRE(out_host, "irk_ctx_log_take: NULL output");
    IRK_CUDA(cudaMemcpyAsync(out_host, ctx->solve_log, (size_t)n * 4 * sizeof(int),
                             cudaMemcpyDeviceToHost, ctx->stream));
  }
  IRK_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < n; ++i) {
    // kernels executed by graph-resident loops: kernels per pass x passes
    ctx->launches += (int64_t)out_host[4 * i + 3] * out_host[4 * i + 2];
  }
  *n_out = n;
  ctx->log_n = 0;
  return IRK_OK;
}

}  // extern "C"
