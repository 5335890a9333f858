// run_batched_probe.hpp -- TEST INFRASTRUCTURE: one run_batched workload
// (engine.hpp:120-212 contract) compiled against either the reference's
// headers (oracle/ref_shim.cpp) or this repository's drop-in headers
// (tests/cpp/facade_main.cpp); both print the same summary line, which
// tests/test_gpu_facade.py compares.  Non-integral per-scenario costs, +inf
// slots and throwing slots exercise the fixed-order mean, the infeasible
// count and the per-slot error map.
#pragma once

#include <cstdint>
#include <cstdio>
#include <limits>
#include <stdexcept>
#include <string>

inline std::string run_batched_probe(std::size_t count, std::size_t batch, unsigned threads,
                                     std::uint64_t budget, std::uint64_t per_bytes) {
  using namespace scendp;
  BackendConfig cfg = threads > 1 ? BackendConfig::multi_thread(threads) : BackendConfig::single_thread();
  cfg.batch_size = batch;
  cfg.memory_budget = budget;
  std::size_t before = 0, after = 0, covered = 0;
  BatchHooks hooks;
  hooks.before = [&](std::size_t, std::size_t lo, std::size_t hi) { ++before; covered += hi - lo; };
  hooks.after = [&](std::size_t, std::size_t, std::size_t) { ++after; };
  auto res = run_batched<ExtendedCost>(
      count,
      [](unsigned) {
        return [](std::size_t w) {
          if (w % 97 == 5) throw std::runtime_error("slot " + std::to_string(w));
          if (w % 13 == 0) return ExtendedCost{std::numeric_limits<double>::infinity()};
          return ExtendedCost{static_cast<double>(w % 17) * 0.1 + 1e-3 * static_cast<double>(w)};
        };
      },
      cfg, per_bytes, &hooks);
  std::size_t ev = 0;
  for (auto e : res.evaluated) ev += e;
  char buf[512];
  std::snprintf(buf, sizeof(buf),
                "mean %.17g finite %zu infeasible %zu errors %zu first_error %s evaluated %zu "
                "batches %zu before %zu after %zu covered %zu warnings %zu",
                res.mean_cost ? *res.mean_cost : -1.0, res.finite_count, res.infeasible_count,
                res.errors.size(), res.errors.empty() ? "-" : res.errors.begin()->second.c_str(), ev,
                res.timings.size(), before, after, covered, res.warnings.size());
  return buf;
}
