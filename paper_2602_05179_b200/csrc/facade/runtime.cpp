// runtime.cpp -- device registry, sharding and error mapping for the facade;
// engine.hpp host utilities (adjust_batch_size / memory_footprint,
// proj/src/engine.cpp:7-30) and ValueFrontier::initial (minplus.cpp:8-21).
#include "runtime.hpp"

#include <cstdlib>
#ifdef __GLIBC__
#include <malloc.h>
#endif
#ifdef __linux__
#include <sys/mman.h>
#endif

#include <algorithm>
#include <chrono>
#include <exception>
#include <limits>
#include <map>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>

#include "scendp/minplus.hpp"

namespace scendp {

std::size_t adjust_batch_size(std::size_t requested, std::uint64_t budget_bytes,
                              std::uint64_t per_scenario_bytes, bool* undersized) {
  if (undersized) *undersized = false;
  if (per_scenario_bytes == 0) return requested < 1 ? 1 : requested;
  const std::uint64_t fit = budget_bytes / per_scenario_bytes;
  if (fit == 0) {
    if (undersized) *undersized = true;
    return 1;
  }
  const std::uint64_t capped = fit < requested ? fit : requested;
  return static_cast<std::size_t>(capped < 1 ? 1 : capped);
}

FootprintEstimate memory_footprint(const FootprintModel& model, std::uint64_t scenario_count) {
  constexpr std::uint64_t kMax = std::numeric_limits<std::uint64_t>::max();
  if (model.per_scenario_bytes != 0 &&
      scenario_count > (kMax - model.fixed_bytes) / model.per_scenario_bytes)
    return {kMax, true};
  return {model.fixed_bytes + scenario_count * model.per_scenario_bytes, false};
}

ValueFrontier ValueFrontier::initial(int stage, std::size_t state_count,
                                     std::size_t start_state) {
  if (start_state >= state_count)
    throw std::invalid_argument("initial frontier: start state " + std::to_string(start_state) +
                                " outside state space of size " + std::to_string(state_count));
  ValueFrontier f;
  f.stage = stage;
  f.values.assign(state_count, ExtendedCost::infinity());
  f.values[start_state] = ExtendedCost::zero();
  return f;
}

namespace detail {

void parallel_for(std::size_t count, const std::function<void(std::size_t, std::size_t)>& fn,
                  unsigned threads, std::size_t min_per_thread) {
  if (threads == 0) threads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const std::size_t parts = std::max<std::size_t>(
      1, std::min<std::size_t>(threads, count / std::max<std::size_t>(1, min_per_thread)));
  if (parts <= 1) {
    fn(0, count);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(parts);
  for (std::size_t p = 0; p < parts; ++p)
    pool.emplace_back([&, p] {
      try {
        fn(count * p / parts, count * (p + 1) / parts);
      } catch (...) {
        errs[p] = std::current_exception();
      }
    });
  for (auto& t : pool) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

void check(scendp_status s) {
  if (s == SCENDP_OK) return;
  const std::string msg = scendp_last_error();
  switch (s) {
    case SCENDP_ERR_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case SCENDP_ERR_LOGIC:
      throw std::logic_error(msg);
    case SCENDP_ERR_OUT_OF_MEMORY:
      throw std::runtime_error("scendp: out of device memory: " + msg);
    default:
      throw std::runtime_error("scendp: " + msg);
  }
}

#ifdef __GLIBC__
namespace {
// glibc's top pad: DEFAULT_TOP_PAD (128 KB) unless MALLOC_TOP_PAD_ set it
std::size_t default_top_pad() {
  const char* e = std::getenv("MALLOC_TOP_PAD_");
  return e ? static_cast<std::size_t>(std::strtoull(e, nullptr, 10)) : std::size_t{128} << 10;
}
std::mutex g_pad_mu;
int g_pad_users = 0;
}  // namespace

MallocPadScope::MallocPadScope(std::size_t pad) {
  std::lock_guard<std::mutex> g(g_pad_mu);
  if (g_pad_users++ == 0) mallopt(M_TOP_PAD, static_cast<int>(std::min<std::size_t>(pad, 1u << 30)));
}
MallocPadScope::~MallocPadScope() {
  std::lock_guard<std::mutex> g(g_pad_mu);
  if (--g_pad_users == 0) mallopt(M_TOP_PAD, static_cast<int>(default_top_pad()));
}
#else
MallocPadScope::MallocPadScope(std::size_t) {}
MallocPadScope::~MallocPadScope() {}
#endif

void advise_huge_pages(void* p, std::size_t bytes) {
#ifdef __linux__
  constexpr std::uintptr_t kHuge = std::uintptr_t{2} << 20;
  if (bytes < 4 * kHuge) return;
  const std::uintptr_t a = (reinterpret_cast<std::uintptr_t>(p) + kHuge - 1) & ~(kHuge - 1);
  const std::uintptr_t e = (reinterpret_cast<std::uintptr_t>(p) + bytes) & ~(kHuge - 1);
  if (e > a) (void)madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
#else
  (void)p;
  (void)bytes;
#endif
}

double* DeviceSlot::pinned_totals(std::size_t count) {
  const std::size_t bytes = std::max<std::size_t>(count, 1) * sizeof(double);
  if (pinned_bytes < bytes) {
    if (pinned) check(scendp_host_free_pinned(pinned));
    pinned = nullptr;
    pinned_bytes = 0;
    check(scendp_host_alloc_pinned(bytes, &pinned));
    pinned_bytes = bytes;
  }
  return static_cast<double*>(pinned);
}

void* DeviceSlot::pinned_chunk(int which, std::size_t bytes) {
  if (chunk_bytes < bytes) {
    for (auto& c : chunk) {
      if (c) check(scendp_host_free_pinned(c));
      c = nullptr;
    }
    chunk_bytes = 0;
    for (auto& c : chunk) check(scendp_host_alloc_pinned(bytes, &c));
    chunk_bytes = bytes;
  }
  return chunk[which];
}

DeviceSlot& device_slot(int device) {
  static std::mutex reg_mu;
  static std::map<int, std::unique_ptr<DeviceSlot>> reg;
  std::lock_guard<std::mutex> g(reg_mu);
  auto& p = reg[device];
  if (!p) {
    p = std::make_unique<DeviceSlot>();
    scendp_opts o{};
    o.device = device;
    check(scendp_ctx_create(&o, &p->ctx));
  }
  return *p;
}

std::vector<int> devices_of(const BackendConfig& cfg) {
  if (!cfg.devices.empty()) return cfg.devices;
  return {-1};
}

std::vector<Shard> make_shards(std::size_t m, const std::vector<int>& devs) {
  std::vector<Shard> out;
  const std::size_t G = devs.size();
  for (std::size_t g = 0; g < G; ++g) {
    Shard s;
    s.lo = g * m / G;
    s.hi = (g + 1) * m / G;
    s.device = devs[g];
    if (s.hi > s.lo || (m == 0 && g == 0)) out.push_back(s);
  }
  if (out.empty()) out.push_back(Shard{0, 0, devs.front()});
  return out;
}

void run_shards(const std::vector<Shard>& shards,
                const std::function<void(const Shard&, scendp_ctx*)>& fn) {
  auto run_one = [&](const Shard& s) {
    DeviceSlot& slot = device_slot(s.device);
    std::lock_guard<std::mutex> g(slot.mu);
    fn(s, slot.ctx);
  };
  if (shards.size() == 1) {
    run_one(shards[0]);
    return;
  }
  std::vector<std::exception_ptr> errs(shards.size());
  std::vector<std::thread> pool;
  for (std::size_t i = 0; i < shards.size(); ++i)
    pool.emplace_back([&, i] {
      try {
        run_one(shards[i]);
      } catch (...) {
        errs[i] = std::current_exception();
      }
    });
  for (auto& t : pool) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

std::vector<Shard> make_waves(const std::vector<Shard>& shards, std::size_t wave) {
  std::vector<Shard> out;
  const std::size_t w = std::max<std::size_t>(wave, 1);
  for (const Shard& s : shards) {
    if (s.hi == s.lo) {
      out.push_back(s);
      continue;
    }
    for (std::size_t lo = s.lo; lo < s.hi; lo += w)
      out.push_back(Shard{lo, std::min(s.hi, lo + w), s.device});
  }
  return out;
}

void run_waves(const std::vector<Shard>& waves, std::uint64_t per_scenario_bytes,
               std::vector<BatchTiming>* timings,
               const std::function<void(std::size_t, const Shard&, scendp_ctx*)>& fn) {
  std::vector<double> ms(waves.size(), 0.0);
  // per device: the indices of its waves (contiguous, in scenario order)
  std::vector<std::pair<int, std::vector<std::size_t>>> groups;
  for (std::size_t i = 0; i < waves.size(); ++i) {
    if (groups.empty() || groups.back().first != waves[i].device)
      groups.push_back({waves[i].device, {}});
    groups.back().second.push_back(i);
  }
  auto run_group = [&](const std::vector<std::size_t>& idx, int device) {
    DeviceSlot& slot = device_slot(device);
    std::lock_guard<std::mutex> g(slot.mu);
    for (std::size_t i : idx) {
      const std::uint64_t t0 = now_ns();
      fn(i, waves[i], slot.ctx);
      ms[i] = ms_since(t0);
    }
  };
  if (groups.size() == 1) {
    run_group(groups[0].second, groups[0].first);
  } else {
    std::vector<std::exception_ptr> errs(groups.size());
    std::vector<std::thread> pool;
    for (std::size_t gi = 0; gi < groups.size(); ++gi)
      pool.emplace_back([&, gi] {
        try {
          run_group(groups[gi].second, groups[gi].first);
        } catch (...) {
          errs[gi] = std::current_exception();
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }
  if (timings)
    for (std::size_t i = 0; i < waves.size(); ++i) {
      const std::size_t size = waves[i].hi - waves[i].lo;
      timings->push_back({i, size, ms[i], static_cast<std::uint64_t>(size) * per_scenario_bytes});
    }
}

std::size_t wave_size(const BackendConfig& cfg, std::size_t count,
                      std::uint64_t per_scenario_bytes, std::vector<std::string>* warnings) {
  cfg.validate();
  bool undersized = false;
  const std::size_t b = adjust_batch_size(count < cfg.batch_size ? count : cfg.batch_size,
                                          cfg.memory_budget, per_scenario_bytes, &undersized);
  if (undersized && warnings)
    warnings->push_back("memory budget below one scenario's footprint; running batches of 1");
  return b;
}

scendp_dist to_c(const DistributionSpec& d) {
  scendp_dist c{};
  c.kind = d.kind == DistributionSpec::Kind::kUniformInt        ? SCENDP_DIST_UNIFORM
           : d.kind == DistributionSpec::Kind::kTruncatedNormal ? SCENDP_DIST_TNORMAL
                                                                : SCENDP_DIST_POISSON;
  c.lo = d.lo;
  c.hi = d.hi;
  c.mean = d.mean;
  c.stddev = d.stddev;
  c.seed = d.seed;
  return c;
}

ExactAggregate to_exact(const scendp_agg& a) {
  ExactAggregate e;
  e.sum = a.sum;
  if (a.finite_count > 0) e.mean_cost = a.mean;
  e.finite_count = a.finite_count;
  e.infeasible_count = a.infeasible_count;
  e.error_count = a.error_count;
  return e;
}

std::uint64_t now_ns() {
  return static_cast<std::uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                        std::chrono::steady_clock::now().time_since_epoch())
                                        .count());
}

double ms_since(std::uint64_t t0_ns) { return static_cast<double>(now_ns() - t0_ns) * 1e-6; }

}  // namespace detail
}  // namespace scendp
