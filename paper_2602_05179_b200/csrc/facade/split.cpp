// split.cpp -- the split evaluators of the drop-in facade
// (reference: proj/src/split.cpp).  Validation and prefix helpers run on the
// host; every DP runs on the GPU through scendp_split_eval.
#include "scendp/split.hpp"

#include <algorithm>
#include <thread>
#include <cstdlib>
#include <cstdio>
#include <atomic>
#include <cmath>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>

#include "runtime.hpp"

namespace scendp {

namespace {

scendp_routing to_c(const RoutingInstance& inst) {
  scendp_routing r{};
  r.n = inst.n;
  r.capacity = inst.capacity;
  r.hard = inst.hard ? 1 : 0;
  r.penalty_beta = inst.penalty_beta;
  r.costs = inst.costs.data();
  return r;
}

void check_inputs(const RoutingInstance& inst, const GiantTour& tour, std::size_t demand_size) {
  inst.validate();
  tour.validate(inst.n);
  if (demand_size != static_cast<std::size_t>(inst.n))
    throw std::invalid_argument("demand column has " + std::to_string(demand_size) +
                                " entries, instance has " + std::to_string(inst.n) +
                                " customers");
}

// Cost-only totals for scenarios given by `make_sc(range)`, sharded over the
// config's devices and cut into the reference's batches (one call and one
// BatchTiming per wave, detail::run_waves).
template <typename MakeSc>
BatchResultSet<ExtendedCost> costs_impl(const RoutingInstance& inst, const GiantTour& tour,
                                        std::size_t count, MakeSc make_sc,
                                        const BackendConfig& cfg) {
  BatchResultSet<ExtendedCost> out;
  const std::size_t wave = detail::wave_size(cfg, count, sizeof(ExtendedCost), &out.warnings);
  out.per_scenario.resize(count);
  out.evaluated.assign(count, 1);
  if (count == 0) {
    out.evaluated.clear();
    return out;
  }
  const scendp_routing r = to_c(inst);
  const auto waves = detail::make_waves(detail::make_shards(count, detail::devices_of(cfg)), wave);
  std::vector<scendp_agg_raw> raws(waves.size());
  // the reference's mean is a sequential fp64 sum (engine.hpp:195-211); when
  // every finite total is an integer and count * max|total| < 2^53, no
  // partial sum rounds, so it equals the engine's exact aggregate
  std::atomic<bool> integral{true};
  std::atomic<double> max_abs{0.0};
  detail::run_waves(waves, sizeof(ExtendedCost), &out.timings,
                    [&](std::size_t wi, const detail::Shard& s, scendp_ctx* ctx) {
    detail::check(scendp_ctx_set_max_batch(ctx, wave));
    scendp_scenarios sc = make_sc(s);
    // totals land in the device slot's page-locked buffer (stored by the
    // kernels over PCIe, no copy), then become the result objects
    double* tot = detail::device_slot(s.device).pinned_totals(s.hi - s.lo);
    scendp_split_out o{};
    o.mem_kind = SCENDP_MEM_HOST;
    o.totals = tot;
    o.agg_raw = &raws[wi];
    detail::check(scendp_split_eval(ctx, &r, tour.order.data(), 1, &sc, SCENDP_SPLIT_COST_ONLY, &o));
    detail::parallel_for(s.hi - s.lo, [&](std::size_t a, std::size_t b) {
      bool whole = true;
      double mx = 0.0;
      for (std::size_t w = a; w < b; ++w) {
        const double v = tot[w];
        out.per_scenario[s.lo + w] = ExtendedCost{v};
        if (v < std::numeric_limits<double>::infinity()) {
          whole &= std::fabs(v) >= 4503599627370496.0 ||
                   v == static_cast<double>(static_cast<std::int64_t>(v));
          mx = std::max(mx, std::fabs(v));
        }
      }
      if (!whole) integral = false;
      double cur = max_abs.load();
      while (mx > cur && !max_abs.compare_exchange_weak(cur, mx)) {
      }
    });
  });
  scendp_agg agg{};
  detail::check(scendp_agg_finalize(raws.data(), static_cast<std::uint32_t>(raws.size()), 1, &agg));
  if (integral && agg.range_errors == 0 &&
      max_abs.load() * static_cast<double>(count) < 9007199254740992.0) {
    out.finite_count = agg.finite_count;
    out.infeasible_count = agg.infeasible_count;
    if (agg.finite_count > 0) out.mean_cost = agg.mean;
  } else {
    detail::sequential_aggregate(out, [](const ExtendedCost& c) { return c.value; });
  }
  return out;
}

// Full solutions for host columns [lo, hi) of `scen` on one context.  The
// evaluator leaves V and cuts on the device (reference layout); they come
// back in chunks of scenarios through two page-locked buffers, a helper
// thread copying chunk k+1 while the host threads turn chunk k into
// SplitSolution objects -- no full-size pageable intermediate.  Object
// construction runs under MallocPadScope (see runtime.hpp).
void full_impl(scendp_ctx* ctx, const scendp_routing& r, const GiantTour& tour,
               const std::uint32_t* data, std::size_t count, bool quadratic,
               SplitSolution* dst, detail::DeviceSlot& slot) {
  const int n = r.n;
  const std::size_t n1 = static_cast<std::size_t>(n) + 1;
  struct DevBuf {
    scendp_ctx* ctx;
    void* p = nullptr;
    DevBuf(scendp_ctx* c, std::size_t bytes) : ctx(c) {
      detail::check(scendp_device_alloc(ctx, std::max<std::size_t>(bytes, 1), &p));
    }
    ~DevBuf() { scendp_device_free(ctx, p); }
  };
  DevBuf dV(ctx, count * n1 * 8), dC(ctx, count * n1 * 4), dT(ctx, count * 8), dR(ctx, count * 4),
      dF(ctx, count);
  scendp_scenarios sc{};
  sc.mem_kind = SCENDP_MEM_HOST;
  sc.data = data;
  sc.rows = static_cast<std::uint64_t>(n);
  sc.count = count;
  scendp_split_out o{};
  o.mem_kind = SCENDP_MEM_DEVICE;
  o.totals = static_cast<double*>(dT.p);
  o.values = static_cast<double*>(dV.p);
  o.cuts = static_cast<std::int32_t*>(dC.p);
  o.route_count = static_cast<std::int32_t*>(dR.p);
  o.feasible = static_cast<std::uint8_t*>(dF.p);
  const std::uint64_t t0 = detail::now_ns();
  detail::check(scendp_split_eval(ctx, &r, tour.order.data(), 1, &sc,
                                  SCENDP_SPLIT_FULL | (quadratic ? SCENDP_QUADRATIC : 0u), &o));
  std::unique_ptr<double[]> totals(new double[std::max<std::size_t>(count, 1)]);
  std::unique_ptr<std::int32_t[]> rc(new std::int32_t[std::max<std::size_t>(count, 1)]);
  std::unique_ptr<std::uint8_t[]> feas(new std::uint8_t[std::max<std::size_t>(count, 1)]);
  detail::check(scendp_memcpy(ctx, totals.get(), dT.p, count * 8, 1, 0));
  detail::check(scendp_memcpy(ctx, rc.get(), dR.p, count * 4, 1, 0));
  detail::check(scendp_memcpy(ctx, feas.get(), dF.p, count, 1, 0));
  const double eval_ms = detail::ms_since(t0);

  const std::size_t chunk = std::max<std::size_t>(1, std::min<std::size_t>(count, (48u << 20) / (n1 * 12)));
  const std::size_t vbytes = chunk * n1 * 8;
  char* buf[2] = {static_cast<char*>(slot.pinned_chunk(0, chunk * n1 * 12)),
                  static_cast<char*>(slot.pinned_chunk(1, chunk * n1 * 12))};
  auto fetch = [&](std::size_t lo, char* b) -> scendp_status {
    const std::size_t c = std::min(chunk, count - lo);
    scendp_status s = scendp_memcpy(ctx, b, static_cast<const char*>(dV.p) + lo * n1 * 8,
                                    c * n1 * 8, 1, 0);
    if (s == SCENDP_OK)
      s = scendp_memcpy(ctx, b + vbytes, static_cast<const char*>(dC.p) + lo * n1 * 4, c * n1 * 4,
                        1, 0);
    return s;
  };
  detail::MallocPadScope pad(std::size_t{64} << 20);
  if (count > 0) detail::check(fetch(0, buf[0]));
  for (std::size_t lo = 0, k = 0; lo < count; lo += chunk, k ^= 1) {
    const std::size_t next = lo + chunk;
    scendp_status ns = SCENDP_OK;
    std::thread copier;
    if (next < count) copier = std::thread([&, next] { ns = fetch(next, buf[k ^ 1]); });
    const double* V = reinterpret_cast<const double*>(buf[k]);
    const std::int32_t* C = reinterpret_cast<const std::int32_t*>(buf[k] + vbytes);
    try {
      detail::parallel_for(std::min(chunk, count - lo), [&](std::size_t a, std::size_t e) {
        for (std::size_t j = a; j < e; ++j) {
          SplitSolution& s = dst[lo + j];
          s.values.stage = 1;
          s.values.values.resize(n1);
          const double* v = V + j * n1;
          for (std::size_t i = 0; i < n1; ++i) s.values.values[i] = ExtendedCost{v[i]};
          s.cuts.assign(C + j * n1, C + (j + 1) * n1);
          s.total = ExtendedCost{totals[lo + j]};
          s.route_count = rc[lo + j];
          s.feasible = feas[lo + j] != 0;
        }
      }, 0, 1024);
    } catch (...) {
      if (copier.joinable()) copier.join();
      throw;
    }
    if (copier.joinable()) copier.join();
    detail::check(ns);
  }
  if (std::getenv("SCENDP_HOST_TRACE"))
    std::fprintf(stderr, "facade full: evaluate %.1f ms, download + result objects %.1f ms\n",
                 eval_ms, detail::ms_since(t0) - eval_ms);
}

SplitSolution single_scenario(const RoutingInstance& inst, const GiantTour& tour,
                              std::span<const std::uint32_t> demand, bool quadratic) {
  check_inputs(inst, tour, demand.size());
  SplitSolution s;
  const scendp_routing r = to_c(inst);
  detail::DeviceSlot& slot = detail::device_slot(-1);
  std::lock_guard<std::mutex> g(slot.mu);
  detail::check(scendp_ctx_set_max_batch(slot.ctx, 0));
  full_impl(slot.ctx, r, tour, demand.data(), 1, quadratic, &s, slot);
  return s;
}

}  // namespace

void RoutingInstance::validate() const {
  if (n < 1) throw std::invalid_argument("instance needs at least one customer");
  if (capacity <= 0) throw std::invalid_argument("capacity Q must be > 0");
  const std::size_t side = static_cast<std::size_t>(n) + 2;
  if (costs.size() != side * side) throw std::invalid_argument("cost matrix must be (n+2) x (n+2)");
  for (std::size_t a = 0; a < side; ++a)
    for (std::size_t b = 0; b < side; ++b) {
      const double c = costs[a * side + b];
      if (!std::isfinite(c) || c < 0.0)
        throw std::invalid_argument("cost matrix entries must be finite and >= 0");
      if (a == b && c != 0.0) throw std::invalid_argument("cost matrix diagonal must be 0");
    }
  if (!hard && !(penalty_beta >= 0.0)) throw std::invalid_argument("penalty beta must be >= 0");
}

void GiantTour::validate(int n) const {
  if (order.size() != static_cast<std::size_t>(n))
    throw std::invalid_argument("tour must visit all " + std::to_string(n) + " customers");
  std::vector<char> seen(static_cast<std::size_t>(n) + 1, 0);
  for (int c : order) {
    if (c < 1 || c > n || seen[c])
      throw std::invalid_argument("tour is not a permutation of 1.." + std::to_string(n));
    seen[c] = 1;
  }
}

// fill_prefixes (split.cpp:24-39) for callers that inspect the prefixes.
SplitPrefixes build_split_inputs(const RoutingInstance& inst, const GiantTour& tour,
                                 std::span<const std::uint32_t> demand) {
  check_inputs(inst, tour, demand.size());
  const int n = inst.n;
  SplitPrefixes pre;
  pre.dist.assign(n + 1, 0.0);
  pre.load.assign(n + 1, 0);
  for (int i = 1; i <= n; ++i) {
    pre.load[i] = pre.load[i - 1] + demand[tour.order[i - 1] - 1];
    if (i >= 2) pre.dist[i] = pre.dist[i - 1] + inst.cost(tour.order[i - 2], tour.order[i - 1]);
  }
  return pre;
}

double subroute_cost(const RoutingInstance& inst, const GiantTour& tour, const SplitPrefixes& pre,
                     int p, int i) {
  return inst.cost(0, tour.order[p]) + pre.dist[i] - pre.dist[p + 1] +
         inst.cost(tour.order[i - 1], inst.depot_in());
}

std::vector<std::pair<int, int>> recover_routes(const SplitSolution& solution) {
  std::vector<std::pair<int, int>> routes;
  if (!solution.feasible) return routes;
  const int n = static_cast<int>(solution.cuts.size()) - 1;
  for (int i = n; i > 0;) {
    const int p = solution.cuts[i];
    routes.emplace_back(p, i);
    i = p;
  }
  std::reverse(routes.begin(), routes.end());
  return routes;
}

SplitSolution split_scenario_quadratic(const RoutingInstance& inst, const GiantTour& tour,
                                       std::span<const std::uint32_t> demand) {
  return single_scenario(inst, tour, demand, true);
}

SplitSolution split_scenario_linear(const RoutingInstance& inst, const GiantTour& tour,
                                    std::span<const std::uint32_t> demand) {
  if (!inst.hard)
    throw std::invalid_argument(
        "linear split handles hard capacities only; use the quadratic form for penalized "
        "instances");
  return single_scenario(inst, tour, demand, false);
}

ExtendedCost brute_force_split(const RoutingInstance& inst, const GiantTour& tour,
                               std::span<const std::uint32_t> demand) {
  check_inputs(inst, tour, demand.size());
  const int n = inst.n;
  if (n > 20) throw std::invalid_argument("brute-force split is limited to n <= 20");
  double best = std::numeric_limits<double>::infinity();
  // bit p-1 of `cuts` set: a route ends after tour position p (p < n)
  for (std::uint64_t cuts = 0; cuts < (std::uint64_t{1} << (n - 1)); ++cuts) {
    double total = 0.0;
    bool feasible = true;
    for (int first = 1; first <= n && feasible;) {
      int last = first;
      while (last < n && !((cuts >> (last - 1)) & 1)) ++last;
      double c = inst.cost(0, tour.order[first - 1]);
      std::int64_t load = 0;
      for (int k = first; k <= last; ++k) {
        load += demand[tour.order[k - 1] - 1];
        if (k > first) c += inst.cost(tour.order[k - 2], tour.order[k - 1]);
      }
      c += inst.cost(tour.order[last - 1], inst.depot_in());
      if (load > inst.capacity) {
        if (inst.hard) feasible = false;
        else c += inst.penalty_beta * static_cast<double>(load - inst.capacity);
      }
      total += c;
      first = last + 1;
    }
    if (feasible && total < best) best = total;
  }
  return ExtendedCost{best};
}

std::uint64_t split_per_scenario_bytes(int n) {
  const std::uint64_t states = static_cast<std::uint64_t>(n) + 1;
  return states * sizeof(ExtendedCost) + states * sizeof(std::int32_t) +
         static_cast<std::uint64_t>(n) * sizeof(std::uint32_t) + 96;
}

FootprintModel split_footprint_model(const RoutingInstance& instance) {
  const std::uint64_t side = static_cast<std::uint64_t>(instance.n) + 2;
  FootprintModel m;
  m.fixed_bytes = side * side * sizeof(double) + (std::uint64_t{1} << 20);
  m.per_scenario_bytes = split_per_scenario_bytes(instance.n);
  return m;
}

BatchResultSet<SplitSolution> batched_expected_split(const RoutingInstance& inst,
                                                     const GiantTour& tour,
                                                     const ScenarioBatch& scenarios,
                                                     const BackendConfig& cfg) {
  check_inputs(inst, tour, scenarios.rows);
  BatchResultSet<SplitSolution> out;
  const std::size_t m = scenarios.count;
  const std::size_t wave = detail::wave_size(cfg, m, split_per_scenario_bytes(inst.n), &out.warnings);
  out.per_scenario.reserve(m);
  detail::advise_huge_pages(out.per_scenario.data(), m * sizeof(SplitSolution));
  out.per_scenario.resize(m);
  out.evaluated.assign(m, 1);
  if (m == 0) {
    out.evaluated.clear();
    return out;
  }
  const scendp_routing r = to_c(inst);
  const auto waves = detail::make_waves(detail::make_shards(m, detail::devices_of(cfg)), wave);
  detail::run_waves(waves, split_per_scenario_bytes(inst.n), &out.timings,
                    [&](std::size_t, const detail::Shard& s, scendp_ctx* ctx) {
    detail::check(scendp_ctx_set_max_batch(ctx, wave));
    // hard -> linear deque, penalized -> quadratic (split.cpp:316-318)
    full_impl(ctx, r, tour, scenarios.data.data() + s.lo * scenarios.rows, s.hi - s.lo, false,
              out.per_scenario.data() + s.lo, detail::device_slot(s.device));
  });
  detail::sequential_aggregate(out, [](const SplitSolution& s) { return s.total.value; });
  return out;
}

BatchResultSet<ExtendedCost> batched_split_costs(const RoutingInstance& inst,
                                                 const GiantTour& tour,
                                                 const ScenarioBatch& scenarios,
                                                 const BackendConfig& cfg) {
  check_inputs(inst, tour, scenarios.rows);
  return costs_impl(inst, tour, scenarios.count,
                    [&](const detail::Shard& s) {
                      scendp_scenarios sc{};
                      sc.mem_kind = SCENDP_MEM_HOST;
                      sc.data = scenarios.data.data() + s.lo * scenarios.rows;
                      sc.rows = scenarios.rows;
                      sc.count = s.hi - s.lo;
                      sc.first_index = s.lo;
                      return sc;
                    },
                    cfg);
}

BatchResultSet<ExtendedCost> batched_split_costs_generated(const RoutingInstance& inst,
                                                           const GiantTour& tour,
                                                           const DistributionSpec& dist,
                                                           std::size_t count,
                                                           const BackendConfig& cfg) {
  inst.validate();
  tour.validate(inst.n);
  dist.validate();
  const scendp_dist cd = detail::to_c(dist);
  return costs_impl(inst, tour, count,
                    [&](const detail::Shard& s) {
                      scendp_scenarios sc{};
                      sc.mem_kind = SCENDP_MEM_GENERATED;
                      sc.rows = static_cast<std::uint64_t>(inst.n);
                      sc.count = s.hi - s.lo;
                      sc.first_index = s.lo;
                      sc.dist = &cd;
                      return sc;
                    },
                    cfg);
}

RoutingInstance make_random_instance(int n, std::uint64_t seed, std::int64_t capacity, bool hard,
                                     double penalty_beta) {
  RoutingInstance inst;
  inst.n = n;
  inst.capacity = capacity;
  inst.hard = hard;
  inst.penalty_beta = penalty_beta;
  const int side = n + 2;
  inst.costs.assign(static_cast<std::size_t>(side) * side, 0.0);
  SplitMix64 rng(derive_stream(seed, kStreamInstance, 0));
  for (int a = 0; a < side; ++a)
    for (int b = a + 1; b < side; ++b) {
      const double c = static_cast<double>(1 + rng.next_below(20));
      inst.costs[a * side + b] = c;
      inst.costs[b * side + a] = c;
    }
  return inst;
}

std::vector<ExactAggregate> batched_candidate_costs(const RoutingInstance& inst,
                                                    const std::vector<GiantTour>& tours,
                                                    const ScenarioBatch& scenarios,
                                                    const BackendConfig& cfg) {
  inst.validate();
  if (tours.empty()) return {};
  for (const GiantTour& t : tours) t.validate(inst.n);
  if (scenarios.rows != static_cast<std::size_t>(inst.n))
    throw std::invalid_argument("demand column has " + std::to_string(scenarios.rows) +
                                " entries, instance has " + std::to_string(inst.n) +
                                " customers");
  const std::uint32_t k = static_cast<std::uint32_t>(tours.size());
  std::vector<std::int32_t> flat(static_cast<std::size_t>(k) * inst.n);
  for (std::uint32_t q = 0; q < k; ++q)
    std::copy(tours[q].order.begin(), tours[q].order.end(), flat.begin() + q * inst.n);
  const scendp_routing r = to_c(inst);
  const auto shards = detail::make_shards(scenarios.count, detail::devices_of(cfg));
  std::vector<scendp_agg_raw> raw(shards.size() * k);
  detail::run_shards(shards, [&](const detail::Shard& s, scendp_ctx* ctx) {
    detail::check(scendp_ctx_set_max_batch(ctx, 0));
    scendp_scenarios sc{};
    sc.mem_kind = SCENDP_MEM_HOST;
    sc.data = scenarios.data.data() + s.lo * scenarios.rows;
    sc.rows = scenarios.rows;
    sc.count = s.hi - s.lo;
    scendp_split_out o{};
    o.mem_kind = SCENDP_MEM_HOST;
    o.agg_raw = raw.data() + (&s - shards.data()) * k;
    detail::check(scendp_split_eval(ctx, &r, flat.data(), k, &sc, SCENDP_SPLIT_COST_ONLY, &o));
  });
  std::vector<scendp_agg> agg(k);
  detail::check(scendp_agg_finalize(raw.data(), static_cast<std::uint32_t>(shards.size()), k,
                                    agg.data()));
  std::vector<ExactAggregate> out(k);
  for (std::uint32_t q = 0; q < k; ++q) out[q] = detail::to_exact(agg[q]);
  return out;
}

long best_candidate(const std::vector<ExactAggregate>& scores) {
  long best = -1;
  double bv = std::numeric_limits<double>::infinity();
  for (std::size_t c = 0; c < scores.size(); ++c)
    if (scores[c].mean_cost && *scores[c].mean_cost < bv) {
      bv = *scores[c].mean_cost;
      best = static_cast<long>(c);
    }
  return best;
}

}  // namespace scendp
