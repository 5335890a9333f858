// internal.hpp -- host-side context shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "scendp_cuda.h"

// NVTX (header-only v3; a no-op unless a profiler attaches): one range per
// C-ABI call, so nsys/ncu timelines show the engine's phases by name.
#include <nvtx3/nvToolsExt.h>

namespace scendp_host {

struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Thrown inside the library, converted to a status at the C-ABI boundary.
struct Error {
  scendp_status status;
  std::string msg;
};

[[noreturn]] inline void fail(scendp_status s, std::string msg) {
  throw Error{s, std::move(msg)};
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation)
    fail(SCENDP_ERR_OUT_OF_MEMORY, std::string(what) + ": " + cudaGetErrorString(e));
  fail(SCENDP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CUDA_CHECK(x) ::scendp_host::cuda_check((x), #x)

void set_last_error(const std::string& msg);

// fn(part) for part in [0, parts) on a persistent process-wide pool of host
// threads (the caller runs part 0 and waits for the rest).  Replaces a
// thread spawn per staging chunk.  A call made while another call holds the
// pool runs its parts on freshly spawned threads instead.  Exceptions from
// parts are rethrown (the first one).
void parallel_parts(int parts, const std::function<void(int)>& fn);

// Named, growable device scratch buffers owned by a context.
enum ScratchSlot {
  kScrScenarios = 0,   // tiled scenarios (converted or generated)
  kScrStaging,         // reference-layout staging for host/device inputs
  kScrTours,           // per-tour position tables
  kScrAgg,             // raw aggregates [k]
  kScrTotals,          // per-scenario totals when the caller wants host copies
  kScrOut1, kScrOut2, kScrOut3, kScrOut4, kScrOut5, kScrOut6,
  kScrOut7, kScrOut8, kScrOut9,
  kScrOverflow,        // general staging (DSIRP reference-layout outputs)
  kScrHandoff,         // split hand-off bitmap + list: owned by split_eval
                       // only (the bitmap must stay all-zero at rest)
  kScrLongHorizon,     // DSIRP dense fallback (H > 32): per-thread frontiers
  kScrFallback,        // overflow-path deques
  kScrCdf,             // poisson table
  kScrCustomers,       // dsirp customer records
  kScrFlush,           // L2 flush buffer
  kScrCount
};

struct NcclApi;

}  // namespace scendp_host

struct scendp_ctx {
  int device = 0;
  int sm_count = 0;
  // split overflow bitmap: allocation generation it lives in, bytes known
  // all-zero (reset on reallocation -- a new block may reuse the address --
  // and while a call that may set bits is in flight)
  uint64_t ovf_gen = ~uint64_t{0};
  uint64_t ovf_clean = 0;
  cudaStream_t stream = nullptr;
  scendp_opts opts{};
  void* scratch[scendp_host::kScrCount] = {};
  uint64_t scratch_bytes[scendp_host::kScrCount] = {};
  uint64_t scratch_gen[scendp_host::kScrCount] = {};  // bumped on every (re)allocation
  void* agg_pinned = nullptr;       // pinned staging for raw aggregates
  uint64_t agg_pinned_bytes = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  // kernel timing
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> event_pool;
  struct Pending { int pool_index; int kind; };  // kind 0 = dp, 1 = gen
  std::vector<Pending> pending;
  scendp_kernel_stats stats{};
  // multi-GPU
  void* nccl_comm = nullptr;
  int nranks = 1, rank = 0;

  void* scratch_get(int slot, uint64_t bytes);
  void scratch_free(int slot);
  uint64_t scratch_total = 0;  // device bytes held in scratch blocks
  uint64_t scratch_peak = 0;   // high-water mark of scratch_total
  uint64_t oom_retries = 0;    // waves halved after cudaErrorMemoryAllocation
  uint64_t last_wave = 0;      // wave size of the last split / DSIRP call
  uint64_t tnormal_host_columns = 0;  // tnormal columns resolved on the host
  // Scenarios per wave from the device footprint model: fixed + per_scenario
  // x wave must fit the budget -- scratch_limit if set, else the scratch
  // already held plus the free device memory (less 1/16 headroom); also
  // capped by max_batch.  Tile-aligned, at least one tile.
  uint64_t wave_for_model(uint64_t m, uint64_t fixed, uint64_t per_scenario,
                          uint64_t* budget_out);
  // kernel timing helpers (no-ops unless SCENDP_CTX_KERNEL_TIMING)
  int timing_begin(int kind);
  void timing_end(int token);
  void timing_resolve();  // after a stream sync
  void count_launch(uint64_t n = 1) { stats.launches += n; }
  // scenarios per launch wave: max_batch (tile-aligned), further capped so
  // the wave's staged scenario copy (stage_bytes per scenario) stays within
  // scratch_limit; 0 / unset = the whole call
  uint64_t wave_for(uint64_t m, uint64_t stage_bytes) const {
    uint64_t w = opts.max_batch ? ((opts.max_batch + 31) & ~uint64_t{31}) : m;
    if (opts.scratch_limit && stage_bytes)
      w = std::min<uint64_t>(w, std::max<uint64_t>(32, (opts.scratch_limit / stage_bytes) & ~uint64_t{31}));
    return w;
  }
  // stream-ordered copy with H2D / D2H byte accounting (bench e2e bytes)
  void copy(void* dst, const void* src, uint64_t bytes, cudaMemcpyKind kind) {
    if (bytes == 0) return;
    scendp_host::cuda_check(cudaMemcpyAsync(dst, src, bytes, kind, stream), "cudaMemcpyAsync");
    if (kind == cudaMemcpyHostToDevice) stats.h2d_bytes += bytes;
    else if (kind == cudaMemcpyDeviceToHost) stats.d2h_bytes += bytes;
  }
  void sync();
  // Multi-GPU aggregates.  With a communicator of > 1 rank the raw
  // aggregates alternate between two device buffers and the all-reduce runs
  // on comm_stream after the DP kernels (event-ordered), so it overlaps the
  // next call's kernels; a call waits for the all-reduce only when it reads
  // the aggregate back (agg_readback) or reuses the buffer two calls later.
  void* agg_buffer(uint64_t bytes);      // this call's aggregate buffer
  void allreduce_agg(void* dev_raw, uint64_t words);  // NCCL, if attached
  void agg_readback(void* host, const void* dev, uint64_t bytes);  // after the all-reduce
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_dp = nullptr;
  cudaEvent_t ev_ar[2] = {nullptr, nullptr};
  bool ev_ar_used[2] = {false, false};
  void* agg_bufs[2] = {nullptr, nullptr};
  uint64_t agg_bufs_bytes = 0;
  int agg_slot = 0;
  bool comm_pending = false;  // an all-reduce is queued on comm_stream
  // SCENDP_OVERLAP_ALLREDUCE=1 at communicator creation forces the
  // overlapped path for a 1-rank communicator too (tests on one GPU)
  bool force_overlap = false;
  bool overlapped() const { return nccl_comm != nullptr && (nranks > 1 || force_overlap); }
  void* pinned_agg(uint64_t bytes);
  // DSIRP customer tables resident in kScrCustomers: the serialized customer
  // set they were built from (calls with an identical set skip the host
  // preparation and the upload)
  std::vector<char> dsirp_key;
  bool dsirp_int_path = false;
  int dsirp_maxR = 1;
  bool dsirp_fast_fp64 = false;
  size_t dsirp_o_pool = 0, dsirp_o_ipool = 0;  // offsets inside kScrCustomers
  // page-locked staging buffers (SCNB ingestion double buffering)
  void* stage_pinned[2] = {nullptr, nullptr};
  uint64_t stage_pinned_bytes[2] = {0, 0};
  void* pinned_stage(int idx, uint64_t bytes);
  // pinned staging of per-call tables (split tour tables); the event marks
  // the last upload from it, so the next call waits only if it is pending
  void* tables_pinned = nullptr;
  uint64_t tables_pinned_bytes = 0;
  cudaEvent_t tables_done = nullptr;
  void* pinned_tables(uint64_t bytes);
  std::vector<char> tours_blob;  // split tour tables resident at tours_dev
  std::vector<double> valid_costs;  // last cost matrix that passed validation
  const double* last_costs_ptr = nullptr;  // where the last validated matrix was
  // the Poisson CDF resident in kScrCdf (make_gen_params)
  double cdf_mean = -1.0;
  int64_t cdf_hi = -1;
  const double* cdf_dev = nullptr;
  uint64_t cdf_gen = 0;
  void* tours_dev = nullptr;
  void tables_uploaded();
};

namespace scendp_host {

// Finalize raw aggregates (host): combine n shard records per candidate.
void finalize_agg(const scendp_agg_raw* raw, uint32_t n, uint32_t k,
                  scendp_agg* out);

// Device -> host copy of a large result into pageable memory: whole chunks
// go D2H into two page-locked buffers (alternating) and are copied out by
// host threads while the next chunk transfers.  Small or page-locked
// destinations take one plain async copy.  Returns after the data is in
// `dst` for the pipelined form (the caller synchronises the stream anyway).
void download(scendp_ctx* ctx, void* dst, const void* src, uint64_t bytes);

// Device alias of a page-locked, UVA-mapped host buffer (cudaMallocHost /
// cudaHostAlloc / cudaHostRegister), or nullptr for pageable memory.  Per-
// scenario totals bound for such a buffer are stored by the DP kernels
// straight over PCIe while they run, instead of a D2H copy after them.
void* mapped_host_alias(void* host);

// C-ABI wrapper: run `f`, translate exceptions to a status.
template <typename F>
scendp_status guard(F&& f) {
  try {
    f();
    return SCENDP_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.status;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SCENDP_ERR_RUNTIME;
  }
}

// Make the scenario source available on the device in the tiled layout (or
// report that the kernel generates it).  Returns the tiled device pointer or
// nullptr for fused generation; fills `gen` for GENERATED sources.
struct GenParamsHost;
const uint32_t* stage_scenarios(scendp_ctx* ctx, const scendp_scenarios* sc,
                                bool allow_fused, void* gen_params_out,
                                bool* fused);

// Device bytes stage_scenarios needs for `sc` (allow_fused = true): per
// scenario of a wave (returned) and independent of the wave (*fixed).
uint64_t stage_footprint(const scendp_scenarios* sc, uint64_t* fixed);
// Reserve stage_scenarios' scratch for a wave of `mw` scenarios of `sc`.
void reserve_stage(scendp_ctx* ctx, const scendp_scenarios* sc, uint64_t mw);
// Free the per-wave scratch blocks (out-of-memory retry with a smaller wave).
void release_wave_scratch(scendp_ctx* ctx);

}  // namespace scendp_host
