// runtime.hpp -- internal glue between the C++ drop-in facade and the C-ABI.
#pragma once

#include <cstdint>
#include <functional>
#include <mutex>
#include <vector>

#include "scendp/engine.hpp"
#include "scendp/scenario.hpp"
#include "scendp_cuda.h"

namespace scendp::detail {

// Map a C-ABI status to the reference's exception types (invalid_argument,
// logic_error, runtime_error; OOM -> std::bad_alloc).
void check(scendp_status s);

// Lazily created, cached context per CUDA device (+ its call mutex).
struct DeviceSlot {
  scendp_ctx* ctx = nullptr;
  std::mutex mu;
  // page-locked staging for per-scenario totals (the kernels store into it
  // directly); grown on demand, used under `mu`
  void* pinned = nullptr;
  std::size_t pinned_bytes = 0;
  double* pinned_totals(std::size_t count);
  // two page-locked chunk buffers for pipelined result downloads
  void* chunk[2] = {nullptr, nullptr};
  std::size_t chunk_bytes = 0;
  void* pinned_chunk(int which, std::size_t bytes);
};
DeviceSlot& device_slot(int device);

std::vector<int> devices_of(const BackendConfig& cfg);

struct Shard {
  std::size_t lo = 0, hi = 0;
  int device = 0;
};

// Contiguous scenario ranges [g*m/G, (g+1)*m/G) per device.
std::vector<Shard> make_shards(std::size_t m, const std::vector<int>& devs);

// Run fn(shard, ctx) on every shard, one host thread per device, holding the
// device's call mutex.  Rethrows the first exception.
void run_shards(const std::vector<Shard>& shards,
                const std::function<void(const Shard&, scendp_ctx*)>& fn);

// The reference's run_batched batches (engine.hpp:150-192) on the GPU: every
// device shard is cut into waves of `wave` scenarios (in scenario order), one
// C-ABI call per wave, each timed.  run_waves runs fn(index, wave, ctx) for
// every wave -- one host thread per device, its waves in order under the
// device's call mutex -- and appends one BatchTiming per wave to `timings`
// (batch index = wave index, bytes = size x per_scenario_bytes), in scenario
// order like the reference's.
std::vector<Shard> make_waves(const std::vector<Shard>& shards, std::size_t wave);
void run_waves(const std::vector<Shard>& waves, std::uint64_t per_scenario_bytes,
               std::vector<BatchTiming>* timings,
               const std::function<void(std::size_t, const Shard&, scendp_ctx*)>& fn);

// BackendConfig::batch_size / memory_budget -> per-call wave size
// (adjust_batch_size, engine.cpp:7-20); appends the reference's warning.
std::size_t wave_size(const BackendConfig& cfg, std::size_t count,
                      std::uint64_t per_scenario_bytes,
                      std::vector<std::string>* warnings);

scendp_dist to_c(const DistributionSpec& d);

// Fixed-order aggregate of run_batched (engine.hpp:195-211).
template <typename R, typename CostOf>
void sequential_aggregate(BatchResultSet<R>& out, CostOf cost_of) {
  double sum = 0.0;
  for (std::size_t w = 0; w < out.per_scenario.size(); ++w) {
    if (!out.evaluated[w]) continue;
    const double c = cost_of(out.per_scenario[w]);
    if (c < std::numeric_limits<double>::infinity()) {
      sum += c;
      ++out.finite_count;
    } else {
      ++out.infeasible_count;
    }
  }
  if (out.finite_count > 0) out.mean_cost = sum / static_cast<double>(out.finite_count);
}

ExactAggregate to_exact(const scendp_agg& a);

// fn(lo, hi) over [0, count) split across up to `threads` host threads
// (result objects of the batched evaluators are built in parallel, like the
// reference's worker threads build theirs).
void parallel_for(std::size_t count, const std::function<void(std::size_t, std::size_t)>& fn,
                  unsigned threads = 0, std::size_t min_per_thread = 4096);

// While alive, heap growth steps are `pad` bytes instead of glibc's 128 KB
// (M_TOP_PAD), restored afterwards.  Building millions of small result
// vectors on many threads otherwise serializes on the kernel's address-space
// lock (one heap-growth mprotect per 128 KB): measured 2.4x on
// batched_expected_split at C2.  No-op outside glibc.
class MallocPadScope {
 public:
  explicit MallocPadScope(std::size_t pad);
  ~MallocPadScope();
  MallocPadScope(const MallocPadScope&) = delete;
  MallocPadScope& operator=(const MallocPadScope&) = delete;
};

// Transparent huge pages for a large block about to be filled (advisory):
// a vector's value-initialization then takes ~1/512 of the page faults.
void advise_huge_pages(void* p, std::size_t bytes);

double ms_since(std::uint64_t t0_ns);
std::uint64_t now_ns();

}  // namespace scendp::detail
