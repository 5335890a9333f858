// context.cu -- C-ABI: contexts, memory, timing, aggregates, NCCL.
#include <dlfcn.h>

#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>

#include <condition_variable>
#include <exception>
#include <functional>
#include <thread>

#include "common.cuh"
#include "internal.hpp"

using namespace scendp_host;

namespace scendp_host {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

// ---- NCCL, loaded at run time ----------------------------------------------
// Minimal ABI of nccl.h (2.x): opaque comm, 128-byte unique id, enums.
typedef struct { char internal[SCENDP_NCCL_UNIQUE_ID_BYTES]; } NcclUniqueId;
typedef int NcclResult;
struct NcclApi {
  void* handle = nullptr;
  NcclResult (*GetUniqueId)(NcclUniqueId*) = nullptr;
  NcclResult (*CommInitRank)(void**, int, NcclUniqueId, int) = nullptr;
  NcclResult (*CommInitAll)(void**, int, const int*) = nullptr;
  NcclResult (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  NcclResult (*CommDestroy)(void*) = nullptr;
  const char* (*GetErrorString)(NcclResult) = nullptr;
};
constexpr int kNcclUint64 = 5, kNcclSum = 0;

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      api.handle = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.handle) break;
    }
    if (!api.handle) return;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.handle, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.handle, "ncclCommInitRank"));
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(dlsym(api.handle, "ncclCommInitAll"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(api.handle, "ncclAllReduce"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.handle, "ncclCommDestroy"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.handle, "ncclGetErrorString"));
  });
  if (!api.handle || !api.AllReduce)
    fail(SCENDP_ERR_NCCL, "NCCL not available (dlopen libnccl.so.2 failed)");
  return api;
}

static void nccl_check(NcclResult r, const char* what) {
  if (r == 0) return;
  fail(SCENDP_ERR_NCCL, std::string(what) + ": " +
                            (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
}

// ---- exact aggregate finalization -----------------------------------------
// The device accumulates 32-bit digits d[j] (weight 2^(32j-192)) in u64
// words.  Carry-propagate into 32-bit words and round once to the nearest
// double (ties to even) -> the correctly rounded sum.
static double digits_to_double(const unsigned __int128* dsum) {
  uint32_t w[18] = {};
  unsigned __int128 carry = 0;
  for (int j = 0; j < 18; ++j) {
    unsigned __int128 t = carry + (j < SCENDP_AGG_DIGITS ? dsum[j] : 0);
    w[j] = static_cast<uint32_t>(t);
    carry = t >> 32;
  }
  int J = 17;
  while (J >= 0 && w[J] == 0) --J;
  if (J < 0) return 0.0;
  unsigned __int128 T = 0;
  int base = J - 2;  // word index of T's lowest word
  for (int j = J; j >= J - 2; --j) T = (T << 32) | (j >= 0 ? w[j] : 0u);
  bool sticky = false;
  for (int j = 0; j < base; ++j) sticky |= (w[j] != 0);
  int nbits = 0;
  for (unsigned __int128 x = T; x; x >>= 1) ++nbits;
  uint64_t mant;
  int shift = 0;
  if (nbits <= 53) {
    mant = static_cast<uint64_t>(T);
  } else {
    shift = nbits - 53;
    mant = static_cast<uint64_t>(T >> shift);
    const unsigned __int128 rem = T & ((static_cast<unsigned __int128>(1) << shift) - 1);
    const unsigned __int128 half = static_cast<unsigned __int128>(1) << (shift - 1);
    const bool up = rem > half || (rem == half && (sticky || (mant & 1)));
    if (up) {
      ++mant;
      if (mant == (1ULL << 53)) { mant >>= 1; ++shift; }
    }
  }
  return std::ldexp(static_cast<double>(mant), shift + 32 * base - 192);
}

void finalize_agg(const scendp_agg_raw* raw, uint32_t n, uint32_t k,
                  scendp_agg* out) {
  for (uint32_t c = 0; c < k; ++c) {
    unsigned __int128 d[SCENDP_AGG_DIGITS] = {};
    scendp_agg a{};
    for (uint32_t r = 0; r < n; ++r) {
      const scendp_agg_raw& x = raw[static_cast<uint64_t>(r) * k + c];
      for (int j = 0; j < SCENDP_AGG_DIGITS; ++j) d[j] += x.digits[j];
      a.finite_count += x.finite_count;
      a.infeasible_count += x.infeasible_count;
      a.error_count += x.error_count;
      a.range_errors += x.range_errors;
    }
    a.sum = digits_to_double(d);
    a.mean = a.finite_count ? a.sum / static_cast<double>(a.finite_count)
                            : std::numeric_limits<double>::quiet_NaN();
    out[c] = a;
  }
}

void* mapped_host_alias(void* host) {
  if (!host) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
    (void)cudaGetLastError();  // unregistered pageable pointer
    return nullptr;
  }
  if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
  return at.devicePointer;
}

}  // namespace scendp_host

// ---- host worker pool ----------------------------------------------------------
namespace scendp_host {
namespace {
struct HostPool {
  std::mutex use;  // one job at a time
  std::mutex mu;
  std::condition_variable cv, done_cv;
  std::vector<std::thread> workers;
  const std::function<void(int)>* job = nullptr;
  int parts = 0, next = 1, remaining = 0;
  uint64_t gen = 0;
  std::exception_ptr err;

  explicit HostPool(int n) {
    for (int w = 0; w < n; ++w) workers.emplace_back([this] { loop(); });
  }
  void take_parts() {  // with mu held on entry and exit
    while (job && next < parts) {
      const int p = next++;
      const std::function<void(int)>* f = job;
      mu.unlock();
      std::exception_ptr e;
      try {
        (*f)(p);
      } catch (...) {
        e = std::current_exception();
      }
      mu.lock();
      if (e && !err) err = e;
      if (--remaining == 0) done_cv.notify_all();
    }
  }
  void loop() {
    std::unique_lock<std::mutex> lk(mu);
    uint64_t seen = 0;
    for (;;) {
      cv.wait(lk, [&] { return gen != seen; });
      seen = gen;
      take_parts();
    }
  }
};

HostPool& host_pool() {
  // leaked on purpose: workers must outlive every static destructor that
  // could still stage data
  static HostPool* pool = new HostPool(
      static_cast<int>(std::min(16u, std::max(1u, std::thread::hardware_concurrency()))) - 1);
  return *pool;
}
}  // namespace

void parallel_parts(int parts, const std::function<void(int)>& fn) {
  if (parts <= 1) {
    if (parts == 1) fn(0);
    return;
  }
  HostPool& pool = host_pool();
  std::unique_lock<std::mutex> use(pool.use, std::try_to_lock);
  if (!use.owns_lock() || pool.workers.empty()) {
    std::vector<std::thread> th;
    std::vector<std::exception_ptr> errs(parts);
    for (int p = 1; p < parts; ++p)
      th.emplace_back([&, p] {
        try {
          fn(p);
        } catch (...) {
          errs[p] = std::current_exception();
        }
      });
    try {
      fn(0);
    } catch (...) {
      errs[0] = std::current_exception();
    }
    for (auto& t : th) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    return;
  }
  std::exception_ptr first;
  {
    std::lock_guard<std::mutex> g(pool.mu);
    pool.job = &fn;
    pool.parts = parts;
    pool.next = 1;
    pool.remaining = parts - 1;
    pool.err = nullptr;
    ++pool.gen;
  }
  pool.cv.notify_all();
  try {
    fn(0);
  } catch (...) {
    first = std::current_exception();
  }
  std::unique_lock<std::mutex> lk(pool.mu);
  pool.take_parts();  // help with whatever is left
  pool.done_cv.wait(lk, [&] { return pool.remaining == 0; });
  pool.job = nullptr;
  if (!first) first = pool.err;
  lk.unlock();
  if (first) std::rethrow_exception(first);
}
}  // namespace scendp_host

// ---- scendp_ctx members ------------------------------------------------------
void* scendp_ctx::scratch_get(int slot, uint64_t bytes) {
  if (bytes == 0) bytes = 256;
  if (scratch_bytes[slot] >= bytes) return scratch[slot];
  scratch_free(slot);
  const uint64_t want = (bytes + (bytes >> 3) + 4095) & ~uint64_t{4095};
  const cudaError_t e = cudaMalloc(&scratch[slot], want);
  if (e != cudaSuccess) {
    scratch[slot] = nullptr;
    (void)cudaGetLastError();  // not sticky: clear it for the caller's retry
    CUDA_CHECK(e);
  }
  scratch_bytes[slot] = want;
  ++scratch_gen[slot];
  scratch_total += want;
  scratch_peak = std::max(scratch_peak, scratch_total);
  return scratch[slot];
}

void scendp_ctx::scratch_free(int slot) {
  if (slot == scendp_host::kScrCustomers) dsirp_key.clear();  // tables move
  if (slot == scendp_host::kScrTours) tours_dev = nullptr;
  if (!scratch[slot]) return;
  CUDA_CHECK(cudaStreamSynchronize(stream));
  CUDA_CHECK(cudaFree(scratch[slot]));
  scratch[slot] = nullptr;
  scratch_total -= scratch_bytes[slot];
  scratch_bytes[slot] = 0;
}

uint64_t scendp_ctx::wave_for_model(uint64_t m, uint64_t fixed, uint64_t per_scenario,
                                    uint64_t* budget_out) {
  uint64_t w = ((std::max<uint64_t>(m, 1) + 31) / 32) * 32;
  if (opts.max_batch) w = std::min(w, (opts.max_batch + 31) & ~uint64_t{31});
  uint64_t budget = opts.scratch_limit;
  if (!budget) {
    if (fixed + per_scenario * w <= scratch_total) {
      // fits what is already held: one wave, no driver query
      if (budget_out) *budget_out = scratch_total;
      return w;
    }
    size_t fr = 0, tot = 0;
    CUDA_CHECK(cudaMemGetInfo(&fr, &tot));
    budget = scratch_total + fr - fr / 16;
  }
  if (budget_out) *budget_out = budget;
  if (per_scenario) {
    // the model counts requested bytes; scratch_get allocates 1/8 more (and
    // rounds each block to 4 KB), so the budget is applied to that
    const uint64_t fixed_alloc = fixed + fixed / 8 + (uint64_t{64} << 10);
    const uint64_t per_alloc = per_scenario + per_scenario / 8 + 1;
    const uint64_t room = budget > fixed_alloc ? budget - fixed_alloc : 0;
    w = std::min(w, std::max<uint64_t>(32, (room / per_alloc) & ~uint64_t{31}));
  }
  return w;
}

void* scendp_ctx::pinned_agg(uint64_t bytes) {
  if (agg_pinned_bytes >= bytes) return agg_pinned;
  if (agg_pinned) CUDA_CHECK(cudaFreeHost(agg_pinned));
  agg_pinned = nullptr;
  CUDA_CHECK(cudaMallocHost(&agg_pinned, bytes));
  agg_pinned_bytes = bytes;
  return agg_pinned;
}

void* scendp_ctx::pinned_stage(int idx, uint64_t bytes) {
  if (stage_pinned_bytes[idx] >= bytes) return stage_pinned[idx];
  if (stage_pinned[idx]) {
    CUDA_CHECK(cudaStreamSynchronize(stream));
    CUDA_CHECK(cudaFreeHost(stage_pinned[idx]));
  }
  stage_pinned[idx] = nullptr;
  stage_pinned_bytes[idx] = 0;
  CUDA_CHECK(cudaMallocHost(&stage_pinned[idx], bytes));
  stage_pinned_bytes[idx] = bytes;
  return stage_pinned[idx];
}

void* scendp_ctx::pinned_tables(uint64_t bytes) {
  if (tables_done) CUDA_CHECK(cudaEventSynchronize(tables_done));
  if (tables_pinned_bytes >= bytes) return tables_pinned;
  if (tables_pinned) CUDA_CHECK(cudaFreeHost(tables_pinned));
  tables_pinned = nullptr;
  tables_pinned_bytes = 0;
  const uint64_t want = std::max<uint64_t>(bytes, 64 << 10);
  CUDA_CHECK(cudaMallocHost(&tables_pinned, want));
  tables_pinned_bytes = want;
  return tables_pinned;
}

void scendp_ctx::tables_uploaded() {
  if (!tables_done) CUDA_CHECK(cudaEventCreateWithFlags(&tables_done, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventRecord(tables_done, stream));
}

int scendp_ctx::timing_begin(int kind) {
  if (!(opts.flags & SCENDP_CTX_KERNEL_TIMING)) return -1;
  const int idx = static_cast<int>(pending.size());
  if (idx >= static_cast<int>(event_pool.size())) {
    cudaEvent_t a, b;
    CUDA_CHECK(cudaEventCreate(&a));
    CUDA_CHECK(cudaEventCreate(&b));
    event_pool.emplace_back(a, b);
  }
  CUDA_CHECK(cudaEventRecord(event_pool[idx].first, stream));
  pending.push_back({idx, kind});
  return idx;
}

void scendp_ctx::timing_end(int token) {
  if (token < 0) return;
  CUDA_CHECK(cudaEventRecord(event_pool[token].second, stream));
}

void scendp_ctx::timing_resolve() {
  for (const Pending& p : pending) {
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, event_pool[p.pool_index].first,
                                    event_pool[p.pool_index].second));
    if (p.kind == 0) {
      stats.dp_launches += 1;
      stats.dp_ms += ms;
    } else {
      stats.gen_launches += 1;
      stats.gen_ms += ms;
    }
  }
  pending.clear();
}

void scendp_ctx::sync() {
  CUDA_CHECK(cudaStreamSynchronize(stream));
  if (comm_pending) {
    CUDA_CHECK(cudaStreamSynchronize(comm_stream));
    comm_pending = false;
  }
  timing_resolve();
}

void* scendp_ctx::agg_buffer(uint64_t bytes) {
  if (!overlapped()) return scratch_get(scendp_host::kScrAgg, bytes);
  if (!comm_stream) {
    CUDA_CHECK(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreateWithFlags(&ev_dp, cudaEventDisableTiming));
    for (auto& e : ev_ar) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  agg_slot ^= 1;
  if (agg_bufs_bytes < bytes) {
    CUDA_CHECK(cudaStreamSynchronize(comm_stream));
    CUDA_CHECK(cudaStreamSynchronize(stream));
    for (auto& b : agg_bufs) {
      if (b) CUDA_CHECK(cudaFree(b));
      b = nullptr;
    }
    const uint64_t want = (bytes + 4095) & ~uint64_t{4095};
    for (auto& b : agg_bufs) CUDA_CHECK(cudaMalloc(&b, want));
    agg_bufs_bytes = want;
    ev_ar_used[0] = ev_ar_used[1] = false;
  }
  // the all-reduce that last read this buffer (two calls ago) must be done
  // before the kernels of this call clear and fill it
  if (ev_ar_used[agg_slot]) CUDA_CHECK(cudaStreamWaitEvent(stream, ev_ar[agg_slot], 0));
  return agg_bufs[agg_slot];
}

void scendp_ctx::allreduce_agg(void* dev_raw, uint64_t words) {
  if (!overlapped()) return;
  CUDA_CHECK(cudaEventRecord(ev_dp, stream));
  CUDA_CHECK(cudaStreamWaitEvent(comm_stream, ev_dp, 0));
  nccl_check(nccl().AllReduce(dev_raw, dev_raw, words, kNcclUint64, kNcclSum,
                              nccl_comm, comm_stream),
             "ncclAllReduce");
  CUDA_CHECK(cudaEventRecord(ev_ar[agg_slot], comm_stream));
  ev_ar_used[agg_slot] = true;
  comm_pending = true;
}

void scendp_ctx::agg_readback(void* host, const void* dev, uint64_t bytes) {
  if (overlapped()) {
    // read the reduced buffer after the all-reduce, on the comm stream
    scendp_host::cuda_check(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, comm_stream),
                            "cudaMemcpyAsync");
    stats.d2h_bytes += bytes;
    comm_pending = true;
  } else {
    copy(host, dev, bytes, cudaMemcpyDeviceToHost);
  }
}

// One host thread per context (the NCCL contract for a single-process
// group): each evaluates its own shard; the first failure is reported.
static scendp_status run_per_context(int32_t n,
                                     const std::function<scendp_status(int32_t)>& call) {
  return guard([&] {
    if (n < 1) fail(SCENDP_ERR_INVALID_ARGUMENT, "need at least one context");
    std::vector<scendp_status> st(static_cast<size_t>(n), SCENDP_OK);
    std::vector<std::string> msg(static_cast<size_t>(n));
    std::vector<std::thread> th;
    th.reserve(static_cast<size_t>(n));
    for (int32_t i = 0; i < n; ++i)
      th.emplace_back([&, i] {
        st[i] = call(i);
        if (st[i] != SCENDP_OK) msg[i] = scendp_last_error();  // thread-local
      });
    for (auto& t : th) t.join();
    for (int32_t i = 0; i < n; ++i)
      if (st[i] != SCENDP_OK) fail(st[i], "context " + std::to_string(i) + ": " + msg[i]);
  });
}

// ---- C-ABI -------------------------------------------------------------------
extern "C" {

const char* scendp_last_error(void) { return g_last_error.c_str(); }

int32_t scendp_abi_version(void) { return SCENDP_ABI_VERSION; }

scendp_status scendp_ctx_create(const scendp_opts* opts, scendp_ctx** out) {
  return guard([&] {
    if (!out) fail(SCENDP_ERR_INVALID_ARGUMENT, "out is null");
    *out = nullptr;
    int ndev = 0;
    const cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
      fail(SCENDP_ERR_NO_DEVICE,
           std::string("no CUDA device available (the engine has no CPU fallback): ") +
               cudaGetErrorString(e));
    scendp_opts o{};
    o.device = -1;
    if (opts) o = *opts;
    int dev = o.device;
    if (dev < 0) CUDA_CHECK(cudaGetDevice(&dev));
    if (dev >= ndev) fail(SCENDP_ERR_INVALID_ARGUMENT, "device ordinal out of range");
    CUDA_CHECK(cudaSetDevice(dev));
    cudaDeviceProp prop{};
    CUDA_CHECK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major < 10)
      fail(SCENDP_ERR_NO_DEVICE, "this build targets sm_100a (B200); device is sm_" +
                                     std::to_string(prop.major * 10 + prop.minor));
    auto* ctx = new scendp_ctx();
    ctx->device = dev;
    ctx->sm_count = prop.multiProcessorCount;
    ctx->opts = o;
    ctx->opts.device = dev;
    CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreate(&ctx->t0));
    CUDA_CHECK(cudaEventCreate(&ctx->t1));
    *out = ctx;
  });
}

void scendp_ctx_destroy(scendp_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->nccl_comm) scendp_comm_destroy(ctx);
  for (int s = 0; s < kScrCount; ++s)
    if (ctx->scratch[s]) cudaFree(ctx->scratch[s]);
  if (ctx->agg_pinned) cudaFreeHost(ctx->agg_pinned);
  for (void* p : ctx->stage_pinned)
    if (p) cudaFreeHost(p);
  if (ctx->tables_pinned) cudaFreeHost(ctx->tables_pinned);
  if (ctx->tables_done) cudaEventDestroy(ctx->tables_done);
  if (ctx->comm_stream) {
    cudaStreamSynchronize(ctx->comm_stream);
    cudaStreamDestroy(ctx->comm_stream);
  }
  if (ctx->ev_dp) cudaEventDestroy(ctx->ev_dp);
  for (auto& e : ctx->ev_ar)
    if (e) cudaEventDestroy(e);
  for (void* b : ctx->agg_bufs)
    if (b) cudaFree(b);
  for (auto& p : ctx->event_pool) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  cudaEventDestroy(ctx->t0);
  cudaEventDestroy(ctx->t1);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

scendp_status scendp_ctx_info(scendp_ctx* ctx, int32_t* device, int32_t* sm_count,
                              void** cuda_stream) {
  return guard([&] {
    if (!ctx) fail(SCENDP_ERR_INVALID_ARGUMENT, "ctx is null");
    if (device) *device = ctx->device;
    if (sm_count) *sm_count = ctx->sm_count;
    if (cuda_stream) *cuda_stream = ctx->stream;
  });
}

scendp_status scendp_ctx_sync(scendp_ctx* ctx) {
  return guard([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    ctx->sync();
  });
}

scendp_status scendp_ctx_set_max_batch(scendp_ctx* ctx, uint64_t max_batch) {
  return guard([&] {
    if (!ctx) fail(SCENDP_ERR_INVALID_ARGUMENT, "ctx is null");
    ctx->opts.max_batch = max_batch;
  });
}

scendp_status scendp_device_alloc(scendp_ctx* ctx, uint64_t bytes, void** ptr) {
  return guard([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    CUDA_CHECK(cudaMalloc(ptr, bytes ? bytes : 1));
  });
}

scendp_status scendp_device_free(scendp_ctx* ctx, void* ptr) {
  return guard([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    CUDA_CHECK(cudaFree(ptr));
  });
}

scendp_status scendp_host_alloc_pinned(uint64_t bytes, void** ptr) {
  return guard([&] { CUDA_CHECK(cudaMallocHost(ptr, bytes ? bytes : 1)); });
}

scendp_status scendp_host_free_pinned(void* ptr) {
  return guard([&] { CUDA_CHECK(cudaFreeHost(ptr)); });
}

scendp_status scendp_memcpy(scendp_ctx* ctx, void* dst, const void* src,
                            uint64_t bytes, int32_t kind, uint32_t flags) {
  return guard([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    const cudaMemcpyKind k = kind == 0   ? cudaMemcpyHostToDevice
                             : kind == 1 ? cudaMemcpyDeviceToHost
                                         : cudaMemcpyDeviceToDevice;
    if (k == cudaMemcpyDeviceToHost && !(flags & SCENDP_ASYNC))
      download(ctx, dst, src, bytes);  // pipelined when large and pageable
    else
      ctx->copy(dst, src, bytes, k);
    if (!(flags & SCENDP_ASYNC)) ctx->sync();
  });
}

scendp_status scendp_memset(scendp_ctx* ctx, void* dst, int32_t value, uint64_t bytes) {
  return guard([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    CUDA_CHECK(cudaMemsetAsync(dst, value, bytes, ctx->stream));
  });
}

scendp_status scendp_ctx_memory(scendp_ctx* ctx, scendp_memory_info* info) {
  return guard([&] {
    if (!ctx || !info) fail(SCENDP_ERR_INVALID_ARGUMENT, "null argument");
    CUDA_CHECK(cudaSetDevice(ctx->device));
    size_t fr = 0, tot = 0;
    CUDA_CHECK(cudaMemGetInfo(&fr, &tot));
    info->scratch_bytes = ctx->scratch_total;
    info->scratch_peak = ctx->scratch_peak;
    info->device_free = fr;
    info->device_total = tot;
    info->oom_retries = ctx->oom_retries;
    info->last_wave = ctx->last_wave;
    info->tnormal_host_columns = ctx->tnormal_host_columns;
  });
}

scendp_status scendp_agg_finalize(const scendp_agg_raw* raw, uint32_t n, uint32_t k,
                                  scendp_agg* out) {
  return guard([&] {
    if (!raw || !out) fail(SCENDP_ERR_INVALID_ARGUMENT, "null aggregate pointer");
    finalize_agg(raw, n, k, out);
  });
}

int64_t scendp_best_candidate(const scendp_agg* agg, uint32_t k) {
  int64_t best = -1;
  double bv = std::numeric_limits<double>::infinity();
  for (uint32_t c = 0; c < k; ++c) {
    if (agg[c].finite_count == 0) continue;
    if (agg[c].mean < bv) {
      bv = agg[c].mean;
      best = c;
    }
  }
  return best;
}

scendp_status scendp_nccl_unique_id(uint8_t out[SCENDP_NCCL_UNIQUE_ID_BYTES]) {
  return guard([&] {
    NcclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, SCENDP_NCCL_UNIQUE_ID_BYTES);
  });
}

scendp_status scendp_comm_init_rank(scendp_ctx* ctx,
                                    const uint8_t id[SCENDP_NCCL_UNIQUE_ID_BYTES],
                                    int32_t nranks, int32_t rank) {
  return guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks)
      fail(SCENDP_ERR_INVALID_ARGUMENT, "bad rank / nranks");
    CUDA_CHECK(cudaSetDevice(ctx->device));
    NcclUniqueId uid;
    std::memcpy(uid.internal, id, SCENDP_NCCL_UNIQUE_ID_BYTES);
    void* comm = nullptr;
    nccl_check(nccl().CommInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
    ctx->nccl_comm = comm;
    ctx->nranks = nranks;
    ctx->force_overlap = std::getenv("SCENDP_OVERLAP_ALLREDUCE") != nullptr;
    ctx->rank = rank;
  });
}

scendp_status scendp_comm_init_all(scendp_ctx** ctxs, int32_t n) {
  return guard([&] {
    if (n < 1) fail(SCENDP_ERR_INVALID_ARGUMENT, "need at least one context");
    std::vector<int> devs(n);
    for (int i = 0; i < n; ++i) devs[i] = ctxs[i]->device;
    std::vector<void*> comms(n, nullptr);
    nccl_check(nccl().CommInitAll(comms.data(), n, devs.data()), "ncclCommInitAll");
    for (int i = 0; i < n; ++i) {
      ctxs[i]->nccl_comm = comms[i];
      ctxs[i]->nranks = n;
      ctxs[i]->force_overlap = std::getenv("SCENDP_OVERLAP_ALLREDUCE") != nullptr;
      ctxs[i]->rank = i;
    }
  });
}

scendp_status scendp_split_eval_multi(scendp_ctx** ctxs, int32_t n, const scendp_routing* inst,
                                      const int32_t* tours, uint32_t k_tours,
                                      const scendp_scenarios* sc, uint32_t flags,
                                      const scendp_split_out* out) {
  if (!ctxs || !sc || !out) {
    set_last_error("null contexts / scenarios / outputs");
    return SCENDP_ERR_INVALID_ARGUMENT;
  }
  return run_per_context(n, [&](int32_t i) {
    return scendp_split_eval(ctxs[i], inst, tours, k_tours, sc + i, flags, out + i);
  });
}

scendp_status scendp_dsirp_eval_multi(scendp_ctx** ctxs, int32_t n,
                                      const scendp_customer* customers, uint32_t n_customers,
                                      const scendp_scenarios* sc, uint32_t flags,
                                      const scendp_dsirp_out* out) {
  if (!ctxs || !sc || !out) {
    set_last_error("null contexts / scenarios / outputs");
    return SCENDP_ERR_INVALID_ARGUMENT;
  }
  return run_per_context(n, [&](int32_t i) {
    return scendp_dsirp_eval(ctxs[i], customers, n_customers, sc + i, flags, out + i);
  });
}

scendp_status scendp_comm_destroy(scendp_ctx* ctx) {
  return guard([&] {
    ctx->sync();
    if (ctx->nccl_comm) nccl().CommDestroy(ctx->nccl_comm);
    ctx->nccl_comm = nullptr;
    ctx->nranks = 1;
    ctx->rank = 0;
  });
}

scendp_status scendp_timer_start(scendp_ctx* ctx) {
  return guard([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    CUDA_CHECK(cudaEventRecord(ctx->t0, ctx->stream));
  });
}

scendp_status scendp_timer_stop(scendp_ctx* ctx, double* ms) {
  return guard([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    // the timed region ends after the last all-reduce as well
    if (ctx->comm_pending && ctx->ev_ar_used[ctx->agg_slot])
      CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, ctx->ev_ar[ctx->agg_slot], 0));
    CUDA_CHECK(cudaEventRecord(ctx->t1, ctx->stream));
    ctx->sync();
    float f = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&f, ctx->t0, ctx->t1));
    *ms = f;
  });
}

scendp_status scendp_kernel_stats_get(scendp_ctx* ctx, scendp_kernel_stats* s,
                                      int32_t reset) {
  return guard([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    ctx->sync();
    if (s) *s = ctx->stats;
    if (reset) ctx->stats = scendp_kernel_stats{};
  });
}

}  // extern "C"

// L2 flush: overwrite a buffer twice the L2 size.
__global__ void scendp_flush_kernel(uint4* buf, uint64_t n16, uint32_t salt) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n16;
       i += uint64_t(gridDim.x) * blockDim.x)
    buf[i] = make_uint4(salt, static_cast<uint32_t>(i), 0u, 0u);
}

extern "C" scendp_status scendp_flush_l2(scendp_ctx* ctx) {
  return guard([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    const uint64_t bytes = uint64_t{256} << 20;
    void* p = ctx->scratch_get(kScrFlush, bytes);
    static uint32_t salt = 1;
    scendp_flush_kernel<<<ctx->sm_count * 4, 512, 0, ctx->stream>>>(
        static_cast<uint4*>(p), bytes / 16, salt++);
    CUDA_CHECK(cudaGetLastError());
  });
}
