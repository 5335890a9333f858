// saa.cpp -- SAA first-stage search on the B200 evaluator (reference:
// proj/src/saa.cpp:19-189).
//
// The reference scores one candidate per batched_split_costs call.  Here the
// next K candidates of the reference's scan order (NN constructions, then
// 2-opt (i,j) and Or-opt (len,i,k) rescans) are scored in ONE launch against
// a training set uploaded once; they are then consumed in scan order with the
// reference's accept rule (v < best, strict), and everything after an
// accepted move is discarded (never counted), so the trajectory matches the
// reference's.  `v` is the reference's sequential-order mean: the exact device
// mean decides unless it lies within the sequential sum's rounding band
// (|seq - exact| <= (m+2) 2^-52 |mean|), in which case that candidate's totals
// are summed on the host in scenario order.
#include "scendp/saa.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>

#include "runtime.hpp"

namespace scendp {

namespace {

std::size_t g_candidate_batch = 256;

// saa.cpp:19-43
GiantTour nearest_neighbor_tour(const RoutingInstance& inst, int start) {
  const int n = inst.n;
  GiantTour tour;
  tour.order.reserve(n);
  std::vector<char> used(n + 1, 0);
  int current = start;
  tour.order.push_back(current);
  used[current] = 1;
  for (int step = 1; step < n; ++step) {
    int best = -1;
    double best_cost = std::numeric_limits<double>::infinity();
    for (int c = 1; c <= n; ++c) {
      if (used[c]) continue;
      const double d = inst.cost(current, c);
      if (d < best_cost) {
        best_cost = d;
        best = c;
      }
    }
    tour.order.push_back(best);
    used[best] = 1;
    current = best;
  }
  return tour;
}

// Position in the first-improvement scan (saa.cpp:157-186).
struct Scan {
  int phase = 0;  // 0: 2-opt, 1: or-opt, 2: exhausted
  int i = 0, j = 1;
  int len = 1, oi = 0, ok = 0;
};

void normalize(Scan& s, int n) {
  while (true) {
    if (s.phase == 0) {
      if (s.i + 1 >= n) {
        s.phase = 1;
        s.len = 1;
        s.oi = 0;
        s.ok = 0;
        continue;
      }
      if (s.j >= n) {
        ++s.i;
        s.j = s.i + 1;
        continue;
      }
      return;
    }
    if (s.phase == 1) {
      if (s.len > 3) {
        s.phase = 2;
        return;
      }
      if (s.oi + s.len > n) {
        ++s.len;
        s.oi = 0;
        s.ok = 0;
        continue;
      }
      if (s.ok > n - s.len) {
        ++s.oi;
        s.ok = 0;
        continue;
      }
      if (s.ok == s.oi) {
        ++s.ok;
        continue;
      }
      return;
    }
    return;
  }
}

void advance(Scan& s, int n) {
  if (s.phase == 0) ++s.j;
  else if (s.phase == 1) ++s.ok;
  normalize(s, n);
}

GiantTour apply_move(const GiantTour& cur, const Scan& s) {
  const int n = static_cast<int>(cur.order.size());
  GiantTour cand;
  if (s.phase == 0) {
    cand = cur;
    std::reverse(cand.order.begin() + s.i, cand.order.begin() + s.j + 1);
    return cand;
  }
  const auto& ord = cur.order;
  std::vector<int> rest;
  rest.reserve(n - s.len);
  for (int p = 0; p < n; ++p)
    if (p < s.oi || p >= s.oi + s.len) rest.push_back(ord[p]);
  cand.order.reserve(n);
  cand.order.assign(rest.begin(), rest.begin() + s.ok);
  cand.order.insert(cand.order.end(), ord.begin() + s.oi, ord.begin() + s.oi + s.len);
  cand.order.insert(cand.order.end(), rest.begin() + s.ok, rest.end());
  return cand;
}

// Scenario set resident on one device in the tiled layout.
struct DeviceSet {
  scendp_ctx* ctx = nullptr;
  void* tiled = nullptr;
  std::size_t rows = 0, count = 0;
  DeviceSet() = default;
  DeviceSet(const DeviceSet&) = delete;
  DeviceSet& operator=(const DeviceSet&) = delete;
  ~DeviceSet() {
    if (tiled) scendp_device_free(ctx, tiled);
  }
};
using DeviceTrain = DeviceSet;

// A host batch (reference layout) -> tiled device set.
void upload_set(scendp_ctx* ctx, const ScenarioBatch& b, DeviceSet& ds) {
  ds.ctx = ctx;
  ds.rows = b.rows;
  ds.count = b.count;
  void* ref = nullptr;
  const std::uint64_t bytes = static_cast<std::uint64_t>(b.rows) * b.count * 4;
  detail::check(scendp_device_alloc(ctx, bytes, &ref));
  scendp_status s = scendp_memcpy(ctx, ref, b.data.data(), bytes, 0, 0);
  if (s == SCENDP_OK) s = scendp_device_alloc(ctx, scendp_tiled_bytes(b.rows, b.count), &ds.tiled);
  if (s == SCENDP_OK)
    s = scendp_scenarios_to_tiled(ctx, static_cast<const std::uint32_t*>(ref), b.rows, b.count,
                                  static_cast<std::uint32_t*>(ds.tiled));
  scendp_device_free(ctx, ref);
  detail::check(s);
}

// generate_scenarios(dist, rows, 1, count) produced directly in HBM (K4,
// bit-identical to the host generator for uniform and poisson): the SAA
// experiments never materialize a training or evaluation batch on the host.
void generate_set(scendp_ctx* ctx, const DistributionSpec& dist, std::size_t rows,
                  std::size_t count, DeviceSet& ds) {
  dist.validate();
  ds.ctx = ctx;
  ds.rows = rows;
  ds.count = count;
  detail::check(scendp_device_alloc(ctx, std::max<std::uint64_t>(256, scendp_tiled_bytes(rows, count)),
                                    &ds.tiled));
  const scendp_dist cd = detail::to_c(dist);
  if (count)
    detail::check(scendp_gen_scenarios(ctx, &cd, rows, 0, count, SCENDP_MEM_DEVICE_TILED,
                                       static_cast<std::uint32_t*>(ds.tiled)));
}

std::vector<scendp_agg> score_batch(const DeviceTrain& dt, const RoutingInstance& inst,
                                    const std::vector<GiantTour>& cands) {
  const std::uint32_t k = static_cast<std::uint32_t>(cands.size());
  std::vector<std::int32_t> flat(static_cast<std::size_t>(k) * inst.n);
  for (std::uint32_t q = 0; q < k; ++q)
    std::copy(cands[q].order.begin(), cands[q].order.end(), flat.begin() + q * inst.n);
  scendp_routing r{inst.n, inst.capacity, inst.hard ? 1 : 0, inst.penalty_beta, inst.costs.data()};
  scendp_scenarios sc{};
  sc.mem_kind = SCENDP_MEM_DEVICE_TILED;
  sc.data = static_cast<const std::uint32_t*>(dt.tiled);
  sc.rows = dt.rows;
  sc.count = dt.count;
  std::vector<scendp_agg> agg(k);
  scendp_split_out o{};
  o.mem_kind = SCENDP_MEM_HOST;
  o.agg = agg.data();
  detail::check(scendp_split_eval(dt.ctx, &r, flat.data(), k, &sc, SCENDP_SPLIT_COST_ONLY, &o));
  return agg;
}

// Reference-order mean of one candidate (engine.hpp:195-211).
double sequential_mean(const DeviceTrain& dt, const RoutingInstance& inst, const GiantTour& t) {
  std::vector<double> totals(dt.count);
  scendp_routing r{inst.n, inst.capacity, inst.hard ? 1 : 0, inst.penalty_beta, inst.costs.data()};
  scendp_scenarios sc{};
  sc.mem_kind = SCENDP_MEM_DEVICE_TILED;
  sc.data = static_cast<const std::uint32_t*>(dt.tiled);
  sc.rows = dt.rows;
  sc.count = dt.count;
  scendp_split_out o{};
  o.mem_kind = SCENDP_MEM_HOST;
  o.totals = totals.data();
  detail::check(scendp_split_eval(dt.ctx, &r, t.order.data(), 1, &sc, SCENDP_SPLIT_COST_ONLY, &o));
  double sum = 0.0;
  std::size_t fc = 0;
  for (double v : totals)
    if (v < std::numeric_limits<double>::infinity()) {
      sum += v;
      ++fc;
    }
  if (fc == 0) throw std::runtime_error("evaluation produced no finite scenario cost");
  return sum / static_cast<double>(fc);
}

}  // namespace

void set_candidate_batch(std::size_t k) { g_candidate_batch = k < 1 ? 1 : k; }

std::string mode_label(const BackendConfig& backend) {
  if (backend.mode == BackendConfig::Mode::kSingleThread) return "single";
  if (backend.mode == BackendConfig::Mode::kGpu)
    return "gpu" + std::to_string(backend.devices.empty() ? 1 : backend.devices.size());
  return "multi" + std::to_string(backend.threads);
}

double least_squares_slope(std::span<const double> x, std::span<const double> y) {
  if (x.size() != y.size() || x.size() < 2) return std::numeric_limits<double>::quiet_NaN();
  const double n = static_cast<double>(x.size());
  double sx = 0.0, sy = 0.0, sxx = 0.0, sxy = 0.0;
  for (std::size_t k = 0; k < x.size(); ++k) {
    sx += x[k];
    sy += y[k];
    sxx += x[k] * x[k];
    sxy += x[k] * y[k];
  }
  return (n * sxy - sx * sy) / (n * sxx - sx * sx);
}

double out_of_sample_eval(const RoutingInstance& instance, const GiantTour& tour,
                          const ScenarioBatch& eval, const BackendConfig& backend) {
  const auto res = batched_split_costs(instance, tour, eval, backend);
  if (!res.mean_cost) throw std::runtime_error("evaluation produced no finite scenario cost");
  return *res.mean_cost;
}

namespace {

// The first-improvement search of improve_first_stage (saa.cpp:106-189) on a
// training set already resident in HBM.  `t0` is the caller's start time (the
// reference's clock starts after validation, saa.cpp:106-120).
SearchResult search_on(const RoutingInstance& instance, const DeviceSet& dt,
                       const SearchBudget& budget, std::uint64_t t0) {
  const int n = instance.n;
  const double band = (static_cast<double>(dt.count) + 2.0) * 0x1.0p-52;

  SearchResult out;
  auto over_budget = [&] {
    return out.evaluations >= budget.max_evaluations ||
           detail::ms_since(t0) >= budget.max_wall_seconds * 1000.0;
  };
  // consume one scored candidate exactly like attempt() (saa.cpp:132-142)
  auto consume = [&](GiantTour&& cand, const scendp_agg& a) {
    ++out.evaluations;
    bool better = false;
    double v = std::numeric_limits<double>::infinity();
    if (a.finite_count > 0) {
      const double e = a.mean;
      if (!(out.value < std::numeric_limits<double>::infinity())) {
        v = sequential_mean(dt, instance, cand);
        better = v < out.value;
      } else {
        const double tol = band * std::max(std::fabs(e), std::fabs(out.value));
        if (e < out.value - tol) {
          v = sequential_mean(dt, instance, cand);
          better = true;
        } else if (e <= out.value + tol) {
          v = sequential_mean(dt, instance, cand);
          better = v < out.value;
        }
      }
    }
    if (better) {
      out.tour = std::move(cand);
      out.value = v;
      out.best_found_at = out.evaluations;
    }
    out.trajectory.push_back({detail::ms_since(t0), out.evaluations, out.value});
    return better;
  };

  // constructions (saa.cpp:145-150): the first one is scored even under a
  // zero budget
  {
    const int starts = std::min(n, 8);
    std::vector<GiantTour> cands;
    for (int k = 0; k < starts; ++k) {
      if (k > 0 && static_cast<std::uint64_t>(k) >= budget.max_evaluations) break;
      cands.push_back(nearest_neighbor_tour(instance, 1 + (k * n) / starts));
    }
    const auto agg = score_batch(dt, instance, cands);
    for (std::size_t k = 0; k < cands.size(); ++k) {
      if (k > 0 && over_budget()) break;
      consume(std::move(cands[k]), agg[k]);
    }
  }

  // first-improvement local search, rescanning after each accepted move
  Scan scan;
  normalize(scan, n);
  while (scan.phase != 2) {
    if (over_budget()) return out;
    std::uint64_t room = budget.max_evaluations - out.evaluations;
    const std::size_t kmax = static_cast<std::size_t>(
        std::min<std::uint64_t>(g_candidate_batch, room));
    std::vector<GiantTour> cands;
    std::vector<Scan> where;
    Scan s = scan;
    while (cands.size() < kmax && s.phase != 2) {
      cands.push_back(apply_move(out.tour, s));
      where.push_back(s);
      advance(s, n);
    }
    if (cands.empty()) break;
    const auto agg = score_batch(dt, instance, cands);
    bool accepted = false;
    for (std::size_t c = 0; c < cands.size(); ++c) {
      if (over_budget()) return out;
      if (consume(std::move(cands[c]), agg[c])) {
        accepted = true;
        break;
      }
      scan = where[c];
      advance(scan, n);
    }
    if (accepted) {
      scan = Scan{};
      normalize(scan, n);
    }
  }
  return out;
}

void check_search_inputs(const RoutingInstance& instance, std::size_t rows, std::size_t count) {
  instance.validate();
  if (instance.hard)
    throw std::invalid_argument(
        "first-stage search scores candidates by expected penalized cost; run the instance in "
        "penalized mode");
  if (count == 0) throw std::invalid_argument("training batch is empty");
  if (rows != static_cast<std::size_t>(instance.n))
    throw std::invalid_argument("demand column has " + std::to_string(rows) +
                                " entries, instance has " + std::to_string(instance.n) +
                                " customers");
}

}  // namespace

SearchResult improve_first_stage(const RoutingInstance& instance, const ScenarioBatch& train,
                                 const BackendConfig& backend, const SearchBudget& budget) {
  check_search_inputs(instance, train.rows, train.count);
  backend.validate();
  // upload the training set once (tiled layout) on the first device
  detail::DeviceSlot& slot = detail::device_slot(detail::devices_of(backend).front());
  std::lock_guard<std::mutex> guard(slot.mu);
  detail::check(scendp_ctx_set_max_batch(slot.ctx, 0));
  DeviceSet dt;
  const std::uint64_t t0 = detail::now_ns();
  upload_set(slot.ctx, train, dt);
  return search_on(instance, dt, budget, t0);
}

// ---------------------------------------------------------------------------
// SAA experiments (saa.cpp:191-443).  Same seeds, streams, row order and
// statistics as the reference; every training, evaluation and reference set
// is generated directly in HBM, every search and out-of-sample evaluation
// runs on it, and only means cross back to the host.
namespace {

struct Stats {
  double mean = 0.0, se = 0.0, stddev = 0.0;
};

// sample mean, sample standard deviation (n-1) and standard error
Stats summarize(const std::vector<double>& xs) {
  Stats st;
  if (xs.empty()) return st;
  double sum = 0.0;
  for (double x : xs) sum += x;
  st.mean = sum / static_cast<double>(xs.size());
  if (xs.size() < 2) return st;
  double ss = 0.0;
  for (double x : xs) ss += (x - st.mean) * (x - st.mean);
  st.stddev = std::sqrt(ss / static_cast<double>(xs.size() - 1));
  st.se = st.stddev / std::sqrt(static_cast<double>(xs.size()));
  return st;
}

std::uint64_t rep_index(std::size_t mi, int rep) {
  return static_cast<std::uint64_t>(mi) * 1000003ULL + static_cast<std::uint64_t>(rep);
}

DistributionSpec reseeded(DistributionSpec d, std::uint64_t seed) {
  d.seed = seed;
  return d;
}

// One experiment session: the first device of the config, locked for the
// whole experiment.
struct Session {
  detail::DeviceSlot& slot;
  std::lock_guard<std::mutex> guard;
  explicit Session(const BackendConfig& b)
      : slot(detail::device_slot(detail::devices_of(b).front())), guard(slot.mu) {
    detail::check(scendp_ctx_set_max_batch(slot.ctx, 0));
  }
  scendp_ctx* ctx() const { return slot.ctx; }
};

// Train on a fresh set (stream index rep_index(mi, rep)) with the config's
// evaluation budget.
SearchResult train_and_search(Session& ss, const RoutingInstance& inst,
                              const DistributionSpec& demand, const ExperimentConfig& cfg,
                              std::size_t mi, int rep, std::size_t m) {
  DeviceSet train;
  generate_set(ss.ctx(), reseeded(demand, derive_stream(cfg.seed, kStreamExperiment, rep_index(mi, rep))),
               static_cast<std::size_t>(inst.n), m, train);
  check_search_inputs(inst, train.rows, train.count);
  const std::uint64_t t0 = detail::now_ns();
  return search_on(inst, train, {cfg.search_evaluations, std::numeric_limits<double>::infinity()},
                   t0);
}

ReportRow row(const std::string& exp, const ExperimentConfig& cfg, std::uint64_t m,
              std::int64_t rep, const std::string& metric, double value, double ms = 0.0) {
  return ReportRow{exp, cfg.instance_label, m, rep, metric, value, ms, cfg.seed};
}

}  // namespace

ExperimentReport run_bias_experiment(const RoutingInstance& instance,
                                     const DistributionSpec& demand,
                                     const std::vector<std::size_t>& m_list, int reps,
                                     std::size_t eval_size, std::size_t reference_size,
                                     const ExperimentConfig& config) {
  if (reps < 2) throw std::invalid_argument("bias experiment needs reps >= 2");
  const std::size_t n = static_cast<std::size_t>(instance.n);
  Session ss(config.backend);
  DeviceSet eval;
  generate_set(ss.ctx(), reseeded(demand, derive_stream(config.seed, kStreamEvaluation, 0)), n,
               eval_size, eval);
  ExperimentReport rep_out;
  const std::string exp = "saa_bias";
  double best_oos = std::numeric_limits<double>::infinity();
  GiantTour best_tour;
  for (std::size_t mi = 0; mi < m_list.size(); ++mi) {
    const std::size_t m = m_list[mi];
    std::vector<double> zs, oos;
    for (int rep = 0; rep < reps; ++rep) {
      const SearchResult sr = train_and_search(ss, instance, demand, config, mi, rep, m);
      const double o = sequential_mean(eval, instance, sr.tour);
      zs.push_back(sr.value);
      oos.push_back(o);
      if (o < best_oos) {
        best_oos = o;
        best_tour = sr.tour;
      }
      rep_out.rows.push_back(row(exp, config, m, rep, "in_sample", sr.value));
      rep_out.rows.push_back(row(exp, config, m, rep, "out_of_sample", o));
      rep_out.rows.push_back(row(exp, config, m, rep, "candidates", static_cast<double>(sr.evaluations)));
      rep_out.rows.push_back(row(exp, config, m, rep, "best_found_at", static_cast<double>(sr.best_found_at)));
    }
    const Stats z = summarize(zs), o = summarize(oos);
    rep_out.rows.push_back(row(exp, config, m, -1, "in_sample_mean", z.mean));
    rep_out.rows.push_back(row(exp, config, m, -1, "in_sample_se", z.se));
    rep_out.rows.push_back(row(exp, config, m, -1, "out_of_sample_mean", o.mean));
    rep_out.rows.push_back(row(exp, config, m, -1, "out_of_sample_se", o.se));
  }
  if (reference_size > 0 && !best_tour.order.empty()) {
    DeviceSet ref;
    generate_set(ss.ctx(), reseeded(demand, derive_stream(config.seed, kStreamEvaluation, 1)), n,
                 reference_size, ref);
    rep_out.rows.push_back(row(exp, config, 0, -1, "reference_value",
                               sequential_mean(ref, instance, best_tour)));
  }
  return rep_out;
}

ExperimentReport run_convergence_experiment(const RoutingInstance& instance,
                                            const DistributionSpec& demand,
                                            const std::vector<std::size_t>& m_list, int reps,
                                            const ExperimentConfig& config) {
  if (m_list.size() < 2 || m_list.back() < 100 * m_list.front())
    throw std::invalid_argument(
        "convergence experiment needs m values spanning at least two decades");
  Session ss(config.backend);
  ExperimentReport out;
  const std::string exp = "saa_convergence";
  std::vector<double> lx, ly;
  for (std::size_t mi = 0; mi < m_list.size(); ++mi) {
    const std::size_t m = m_list[mi];
    std::vector<double> zs;
    for (int rep = 0; rep < reps; ++rep) {
      const SearchResult sr = train_and_search(ss, instance, demand, config, mi, rep, m);
      zs.push_back(sr.value);
      out.rows.push_back(row(exp, config, m, rep, "in_sample", sr.value));
      out.rows.push_back(row(exp, config, m, rep, "candidates", static_cast<double>(sr.evaluations)));
    }
    const Stats z = summarize(zs);
    out.rows.push_back(row(exp, config, m, -1, "in_sample_mean", z.mean));
    out.rows.push_back(row(exp, config, m, -1, "in_sample_std", z.stddev));
    if (z.stddev > 0.0) {
      lx.push_back(std::log(static_cast<double>(m)));
      ly.push_back(std::log(z.stddev));
    }
  }
  out.rows.push_back(row(exp, config, 0, -1, "log_std_slope",
                         lx.size() >= 2 ? least_squares_slope(lx, ly) : 0.0));
  return out;
}

ExperimentReport run_quality_experiment(const RoutingInstance& instance,
                                        const DistributionSpec& demand,
                                        const std::vector<std::size_t>& m_list, int reps,
                                        std::size_t eval_size, const ExperimentConfig& config) {
  Session ss(config.backend);
  DeviceSet eval;
  generate_set(ss.ctx(), reseeded(demand, derive_stream(config.seed, kStreamEvaluation, 0)),
               static_cast<std::size_t>(instance.n), eval_size, eval);
  ExperimentReport out;
  const std::string exp = "quality_vs_scenarios";
  for (std::size_t mi = 0; mi < m_list.size(); ++mi) {
    const std::size_t m = m_list[mi];
    std::vector<double> oos;
    for (int rep = 0; rep < reps; ++rep) {
      const SearchResult sr = train_and_search(ss, instance, demand, config, mi, rep, m);
      const double o = sequential_mean(eval, instance, sr.tour);
      oos.push_back(o);
      out.rows.push_back(row(exp, config, m, rep, "out_of_sample", o));
    }
    const Stats o = summarize(oos);
    out.rows.push_back(row(exp, config, m, -1, "out_of_sample_mean", o.mean));
    out.rows.push_back(row(exp, config, m, -1, "out_of_sample_se", o.se));
  }
  return out;
}

ExperimentReport run_scaling_benchmark(const RoutingInstance& instance,
                                       const DistributionSpec& demand,
                                       const ScalingOptions& options,
                                       const ExperimentConfig& config) {
  ExperimentReport out;
  const std::string exp = "scaling";
  GiantTour tour;
  tour.order.resize(instance.n);
  std::iota(tour.order.begin(), tour.order.end(), 1);
  const DistributionSpec dist = reseeded(demand, derive_stream(config.seed, kStreamScenario, 1));
  for (const BackendConfig& mode : options.modes) {
    const std::string label = mode_label(mode);
    std::vector<double> lx, ly;
    // warm-up (context creation, first-launch costs) outside the timings
    batched_split_costs_generated(instance, tour, dist,
                                  std::min<std::size_t>(options.sizes.front(), 1000), mode);
    for (std::size_t size : options.sizes) {
      const std::size_t reps = std::max<std::size_t>(1, options.target_evaluations / size);
      const std::uint64_t t0 = detail::now_ns();
      for (std::size_t r = 0; r < reps; ++r)
        batched_split_costs_generated(instance, tour, dist, size, mode);
      const double ms = detail::ms_since(t0) / static_cast<double>(reps);
      out.rows.push_back(row(exp, config, size, -1, label + "_wall_ms", ms, ms));
      lx.push_back(std::log(static_cast<double>(size)));
      ly.push_back(std::log(ms));
    }
    out.rows.push_back(row(exp, config, 0, -1, label + "_loglog_slope", least_squares_slope(lx, ly)));
  }
  return out;
}

ExperimentReport run_time_budget_experiment(const RoutingInstance& instance,
                                            const DistributionSpec& demand,
                                            const TimeBudgetOptions& options,
                                            const ExperimentConfig& config) {
  if (options.budgets_seconds.empty() ||
      !std::is_sorted(options.budgets_seconds.begin(), options.budgets_seconds.end()))
    throw std::invalid_argument("budgets must be ascending and nonempty");
  ExperimentReport out;
  const std::string exp = "time_budget";
  const DistributionSpec tdist = reseeded(demand, derive_stream(config.seed, kStreamScenario, 0));
  for (const BackendConfig& mode : options.modes) {
    const std::string label = mode_label(mode);
    SearchResult sr;
    {
      Session ss(mode);
      DeviceSet train;
      generate_set(ss.ctx(), tdist, static_cast<std::size_t>(instance.n), options.train_size, train);
      check_search_inputs(instance, train.rows, train.count);
      const std::uint64_t t0 = detail::now_ns();
      SearchBudget budget;
      budget.max_wall_seconds = options.budgets_seconds.back();
      sr = search_on(instance, train, budget, t0);
    }
    for (std::size_t bi = 0; bi < options.budgets_seconds.size(); ++bi) {
      const double limit = options.budgets_seconds[bi] * 1000.0;
      // last trajectory point inside the budget (the first stands in when
      // even the first evaluation overran it)
      TrajectoryPoint at = sr.trajectory.front();
      for (const TrajectoryPoint& p : sr.trajectory) {
        if (p.elapsed_ms > limit) break;
        at = p;
      }
      const auto b = static_cast<std::int64_t>(bi);
      out.rows.push_back(row(exp, config, options.train_size, b, label + "_budget_seconds",
                             options.budgets_seconds[bi]));
      out.rows.push_back(row(exp, config, options.train_size, b, label + "_best_cost",
                             at.best_value, at.elapsed_ms));
      out.rows.push_back(row(exp, config, options.train_size, b, label + "_candidates",
                             static_cast<double>(at.evaluations), at.elapsed_ms));
    }
  }
  if (!options.scaling_sizes.empty()) {
    ScalingOptions sc;
    sc.sizes = options.scaling_sizes;
    sc.modes = options.modes;
    const ExperimentReport sub = run_scaling_benchmark(instance, demand, sc, config);
    out.rows.insert(out.rows.end(), sub.rows.begin(), sub.rows.end());
  }
  return out;
}

}  // namespace scendp
