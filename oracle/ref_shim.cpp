// ref_shim.cpp -- extern "C" entry points into the REAL reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together
// with the reference's own sources, in place under /root/reference/proj/src,
// into oracle/_ref/libscendp_ref.so (hidden visibility, so the reference's
// C++ symbols never interpose on the product's drop-in facade).  Used by
// tests/ to pin the oracle restatement and as bench.py's CPU baseline
// (`cpu_baseline.kind = "reference"`, `--impl reference`).
#include <cstdio>
#include <cstring>
#include <fstream>
#include <exception>
#include <numeric>
#include <string>
#include <vector>

#include "scendp/engine.hpp"
#include "scendp/io.hpp"
#include "scendp/minplus.hpp"
#include "scendp/oracle.hpp"
#include "scendp/oudp.hpp"
#include "scendp/saa.hpp"
#include "scendp/scenario.hpp"
#include "scendp/split.hpp"

#include "io_dump.hpp"
#include "run_batched_probe.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

using namespace scendp;

namespace {

thread_local std::string g_err;

RoutingInstance make_inst(int n, long long Q, int hard, double beta,
                          const double* costs) {
  RoutingInstance inst;
  inst.n = n;
  inst.capacity = Q;
  inst.hard = hard != 0;
  inst.penalty_beta = beta;
  inst.costs.assign(costs, costs + static_cast<size_t>(n + 2) * (n + 2));
  return inst;
}

GiantTour make_tour(int n, const int* tour) {
  GiantTour t;
  t.order.assign(tour, tour + n);
  return t;
}

BackendConfig make_cfg(unsigned threads) {
  return threads <= 1 ? BackendConfig::single_thread()
                      : BackendConfig::multi_thread(threads);
}

template <typename R>
void fill_agg(const BatchResultSet<R>& res, double* mean, int* has_mean,
              unsigned long long* finite, unsigned long long* infeasible) {
  if (mean) *mean = res.mean_cost ? *res.mean_cost : 0.0;
  if (has_mean) *has_mean = res.mean_cost.has_value();
  if (finite) *finite = res.finite_count;
  if (infeasible) *infeasible = res.infeasible_count;
}

struct CustomerArgs {
  int U, I0, H;
  double h, rho;
  int R;
  const double* fixed;
  const double* unit;
  int delivery_tabular;
  const double* delivery_table;
  int holding_tabular;
  const double* holding_table;
};

void make_customer(const CustomerArgs* a, CustomerSpec& spec,
                   DeliveryCostModel& del, HoldingPenaltyModel& hold) {
  spec.capacity = a->U;
  spec.initial_inventory = a->I0;
  spec.horizon = a->H;
  spec.holding = a->h;
  spec.stockout_multiplier = a->rho;
  del.horizon = a->H;
  del.options = a->R;
  if (a->delivery_tabular) {
    del.tabular = true;
    del.table_quantities = a->U + 1;
    del.table.assign(a->delivery_table,
                     a->delivery_table + static_cast<size_t>(a->H) * (a->U + 1));
    del.fixed.assign(static_cast<size_t>(a->H) * a->R, 0.0);
    del.unit.assign(static_cast<size_t>(a->H) * a->R, 0.0);
  } else {
    del.fixed.assign(a->fixed, a->fixed + static_cast<size_t>(a->H) * a->R);
    del.unit.assign(a->unit, a->unit + static_cast<size_t>(a->H) * a->R);
  }
  if (a->holding_tabular) {
    hold.tabular = true;
    hold.table.assign(a->holding_table, a->holding_table + a->U + 1);
  }
}

DistributionSpec make_dist(int kind, long long lo, long long hi, double mean,
                           double stddev, unsigned long long seed) {
  DistributionSpec d;
  d.kind = kind == 1 ? DistributionSpec::Kind::kTruncatedNormal
                     : DistributionSpec::Kind::kUniformInt;
  d.lo = lo;
  d.hi = hi;
  d.mean = mean;
  d.stddev = stddev;
  d.seed = seed;
  return d;
}

}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// The reference's run_batched template on the probe workload.
REF_API int ref_run_batched_probe(size_t count, size_t batch, unsigned threads,
                                  unsigned long long budget, unsigned long long per_bytes,
                                  char* out, size_t cap) {
  const std::string s = run_batched_probe(count, batch, threads, budget, per_bytes);
  std::snprintf(out, cap, "%s", s.c_str());
  return 0;
}

REF_API void ref_make_random_instance(int n, unsigned long long seed,
                                      double* costs) {
  RoutingInstance inst = make_random_instance(n, seed, 1, true, 0.0);
  std::memcpy(costs, inst.costs.data(), inst.costs.size() * sizeof(double));
}

REF_API void ref_generate_scenarios(int kind, long long lo, long long hi,
                                    double mean, double stddev,
                                    unsigned long long seed, size_t entities,
                                    size_t steps, size_t count,
                                    unsigned* out) {
  ScenarioBatch b = generate_scenarios(make_dist(kind, lo, hi, mean, stddev, seed),
                                       entities, steps, count);
  std::memcpy(out, b.data.data(), b.data.size() * sizeof(unsigned));
}

REF_API unsigned long long ref_derive_stream(unsigned long long seed,
                                             unsigned long long tag,
                                             unsigned long long index) {
  return derive_stream(seed, tag, index);
}

// batched_split_costs (split.cpp:363-371) over a reference-layout batch.
REF_API int ref_split_costs(int n, long long Q, int hard, double beta,
                            const double* costs, const int* tour,
                            const unsigned* demand, size_t m, unsigned threads,
                            double* totals, double* mean, int* has_mean,
                            unsigned long long* finite,
                            unsigned long long* infeasible) {
  try {
    RoutingInstance inst = make_inst(n, Q, hard, beta, costs);
    GiantTour t = make_tour(n, tour);
    ScenarioBatch b;
    b.rows = n;
    b.count = m;
    b.data.assign(demand, demand + static_cast<size_t>(n) * m);
    auto res = batched_split_costs(inst, t, b, make_cfg(threads));
    if (totals)
      for (size_t w = 0; w < m; ++w) totals[w] = res.per_scenario[w].value;
    fill_agg(res, mean, has_mean, finite, infeasible);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// batched_split_costs_generated (split.cpp:373-388): the reference's own
// throughput-benchmark call (saa.cpp:366-375).  Scenario index w of the
// call uses stream derive_stream(seed, kStreamScenario, w).
REF_API int ref_split_costs_generated(int n, long long Q, int hard,
                                      double beta, const double* costs,
                                      const int* tour, int kind, long long lo,
                                      long long hi, double dmean, double dstd,
                                      unsigned long long seed, size_t m,
                                      unsigned threads, double* totals,
                                      double* mean, int* has_mean,
                                      unsigned long long* finite,
                                      unsigned long long* infeasible) {
  try {
    RoutingInstance inst = make_inst(n, Q, hard, beta, costs);
    GiantTour t = make_tour(n, tour);
    auto res = batched_split_costs_generated(
        inst, t, make_dist(kind, lo, hi, dmean, dstd, seed), m,
        make_cfg(threads));
    if (totals)
      for (size_t w = 0; w < m; ++w) totals[w] = res.per_scenario[w].value;
    fill_agg(res, mean, has_mean, finite, infeasible);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// batched_expected_split (split.cpp:303-329); V/cuts are m x (n+1).
REF_API int ref_expected_split(int n, long long Q, int hard, double beta,
                               const double* costs, const int* tour,
                               const unsigned* demand, size_t m,
                               unsigned threads, double* totals, double* V,
                               int* cuts, int* route_count,
                               unsigned char* feasible, double* mean,
                               int* has_mean, unsigned long long* finite,
                               unsigned long long* infeasible) {
  try {
    RoutingInstance inst = make_inst(n, Q, hard, beta, costs);
    GiantTour t = make_tour(n, tour);
    ScenarioBatch b;
    b.rows = n;
    b.count = m;
    b.data.assign(demand, demand + static_cast<size_t>(n) * m);
    auto res = batched_expected_split(inst, t, b, make_cfg(threads));
    for (size_t w = 0; w < m; ++w) {
      const SplitSolution& s = res.per_scenario[w];
      if (totals) totals[w] = s.total.value;
      for (int i = 0; i <= n; ++i) {
        if (V) V[w * (n + 1) + i] = s.values.values[i].value;
        if (cuts) cuts[w * (n + 1) + i] = s.cuts[i];
      }
      if (route_count) route_count[w] = s.route_count;
      if (feasible) feasible[w] = s.feasible;
    }
    fill_agg(res, mean, has_mean, finite, infeasible);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// split_scenario_linear / split_scenario_quadratic (split.cpp:335-372).
REF_API int ref_split_scenario(int linear, int n, long long Q, int hard,
                               double beta, const double* costs,
                               const int* tour, const unsigned* demand,
                               double* V, int* cuts, int* route_count) {
  try {
    RoutingInstance inst = make_inst(n, Q, hard, beta, costs);
    GiantTour t = make_tour(n, tour);
    std::span<const std::uint32_t> d(demand, n);
    SplitSolution s = linear ? split_scenario_linear(inst, t, d)
                             : split_scenario_quadratic(inst, t, d);
    for (int i = 0; i <= n; ++i) {
      V[i] = s.values.values[i].value;
      cuts[i] = s.cuts[i];
    }
    *route_count = s.route_count;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

REF_API double ref_brute_force_split(int n, long long Q, int hard, double beta,
                                     const double* costs, const int* tour,
                                     const unsigned* demand) {
  return brute_force_split(make_inst(n, Q, hard, beta, costs), make_tour(n, tour),
                           std::span<const std::uint32_t>(demand, n))
      .value;
}

// batched_expected_cost (oudp.cpp:398-438) for one customer, rows == H.
// evaluated[w] = 0 marks an error slot (engine.hpp:159-165).
REF_API int ref_expected_cost(const CustomerArgs* c, const unsigned* demand,
                              size_t m, unsigned threads, double* totals,
                              unsigned char* deliver, int* quantity,
                              int* end_inventory, int* route_option,
                              unsigned char* evaluated, double* mean,
                              int* has_mean, unsigned long long* finite,
                              unsigned long long* infeasible) {
  try {
    CustomerSpec spec;
    DeliveryCostModel del;
    HoldingPenaltyModel hold;
    make_customer(c, spec, del, hold);
    ScenarioBatch b;
    b.rows = c->H;
    b.count = m;
    b.data.assign(demand, demand + static_cast<size_t>(c->H) * m);
    auto res = batched_expected_cost(spec, del, hold, b, make_cfg(threads));
    const size_t H = c->H;
    for (size_t w = 0; w < m; ++w) {
      const ScheduleResult& s = res.per_scenario[w];
      if (totals) totals[w] = s.total.value;
      if (evaluated) evaluated[w] = res.evaluated[w];
      if (!res.evaluated[w]) continue;
      for (size_t t = 0; t < H; ++t) {
        if (deliver) deliver[w * H + t] = s.deliver[t];
        if (quantity) quantity[w * H + t] = s.quantity[t];
        if (end_inventory) end_inventory[w * H + t] = s.end_inventory[t];
        if (route_option) route_option[w * H + t] = s.route_option[t];
      }
    }
    fill_agg(res, mean, has_mean, finite, infeasible);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// sweep_customer_scenario (oudp.cpp:249-266): H+1 frontiers of U+1 values.
REF_API int ref_sweep_customer(const CustomerArgs* c, const unsigned* demand,
                               double* frontiers) {
  try {
    CustomerSpec spec;
    DeliveryCostModel del;
    HoldingPenaltyModel hold;
    make_customer(c, spec, del, hold);
    auto fr = sweep_customer_scenario(spec, del, hold,
                                      std::span<const std::uint32_t>(demand, c->H));
    for (size_t k = 0; k < fr.size(); ++k)
      for (int s = 0; s <= c->U; ++s)
        frontiers[k * (c->U + 1) + s] = fr[k].values[s].value;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// solve_customer_scenario (oudp.cpp:268-323): the dense oracle path.
REF_API int ref_solve_customer(const CustomerArgs* c, const unsigned* demand,
                               double* total, unsigned char* deliver,
                               int* quantity, int* end_inventory,
                               int* route_option) {
  try {
    CustomerSpec spec;
    DeliveryCostModel del;
    HoldingPenaltyModel hold;
    make_customer(c, spec, del, hold);
    ScheduleResult s = solve_customer_scenario(
        spec, del, hold, std::span<const std::uint32_t>(demand, c->H));
    *total = s.total.value;
    for (int t = 0; t < c->H; ++t) {
      deliver[t] = s.deliver[t];
      quantity[t] = s.quantity[t];
      end_inventory[t] = s.end_inventory[t];
      route_option[t] = s.route_option[t];
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// minplus_apply (minplus.cpp:56-73) for golden A.2; +inf encoded as inf.
REF_API int ref_minplus_apply(size_t rows, size_t cols, const double* a,
                              const double* j, double* out) {
  try {
    MaskedTransition t(rows, cols, 1);
    for (size_t r = 0; r < rows; ++r)
      for (size_t c = 0; c < cols; ++c) t.at(r, c) = ExtendedCost{a[r * cols + c]};
    ValueFrontier f;
    f.values.resize(rows);
    for (size_t r = 0; r < rows; ++r) f.values[r] = ExtendedCost{j[r]};
    ValueFrontier o = minplus_apply(t, f);
    for (size_t c = 0; c < cols; ++c) out[c] = o.values[c].value;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The reference's own randomized oracles (oracle.cpp:61-172).
REF_API unsigned long long ref_oracle_trials(int which, size_t trials,
                                             unsigned long long seed,
                                             int max_n) {
  OracleOutcome o;
  if (which == 0) o = run_split_oracle_trials(trials, seed);
  else if (which == 1) o = run_split_agreement_trials(trials, seed, max_n);
  else o = run_dsirp_oracle_trials(trials, seed);
  g_err = o.first_failure;
  return o.mismatches;
}

// improve_first_stage (saa.cpp:106-189): trajectory of best values.
REF_API int ref_improve_first_stage(int n, long long Q, double beta,
                                    const double* costs, const unsigned* train,
                                    size_t m, unsigned threads,
                                    unsigned long long max_evals,
                                    int* tour_out, double* value,
                                    unsigned long long* evaluations,
                                    unsigned long long* best_found_at,
                                    double* traj_best, size_t traj_cap) {
  try {
    RoutingInstance inst = make_inst(n, Q, 0, beta, costs);
    ScenarioBatch b;
    b.rows = n;
    b.count = m;
    b.data.assign(train, train + static_cast<size_t>(n) * m);
    SearchBudget budget;
    budget.max_evaluations = max_evals;
    SearchResult r = improve_first_stage(inst, b, make_cfg(threads), budget);
    for (int i = 0; i < n; ++i) tour_out[i] = r.tour.order[i];
    *value = r.value;
    *evaluations = r.evaluations;
    *best_found_at = r.best_found_at;
    for (size_t k = 0; k < r.trajectory.size() && k < traj_cap; ++k)
      traj_best[k] = r.trajectory[k].best_value;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// ---- io.hpp (io.cpp): scenario files, instance grammar, reports ----------
REF_API int ref_write_scenario_file(const char* path, const unsigned* data, size_t rows,
                                    size_t count) {
  try {
    ScenarioBatch b;
    b.rows = rows;
    b.count = count;
    b.data.assign(data, data + rows * count);
    write_scenario_file(b, path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

REF_API int ref_read_scenario_file(const char* path, size_t* rows, size_t* count,
                                   unsigned* out, size_t cap) {
  try {
    ScenarioBatch b = read_scenario_file(path);
    *rows = b.rows;
    *count = b.count;
    if (out && b.data.size() <= cap) std::memcpy(out, b.data.data(), b.data.size() * 4);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// parse_instance_file -> canonical dump (io_dump.hpp) or "error <what>"
REF_API int ref_parse_instance_file(const char* path, const char* out_path) {
  std::string text;
  try {
    text = io_dump::instance<ParsedInstance, RoutingInstance, DsirpInstance>(
        parse_instance_file(path));
  } catch (const std::exception& e) {
    text = std::string("error ") + e.what() + "\n";
  }
  std::ofstream(out_path) << text;
  return 0;
}

REF_API int ref_write_routing_instance(int n, long long Q, int hard, double beta,
                                       const double* costs, const char* out_path) {
  std::ofstream f(out_path);
  write_routing_instance(make_inst(n, Q, hard, beta, costs), f);
  return 0;
}

// SAA experiments (saa.cpp:191-443) -> write_report_csv.  which: 0 bias,
// 1 convergence, 2 quality, 3 scaling, 4 time budget.
REF_API int ref_experiment(int which, int n, long long Q, double beta, const double* costs,
                           int kind, long long lo, long long hi, double mean, double sd,
                           const size_t* m_list, size_t nm, int reps, size_t eval_size,
                           size_t ref_size, unsigned long long seed,
                           unsigned long long evals, unsigned threads,
                           const char* out_path) {
  try {
    RoutingInstance inst = make_inst(n, Q, 0, beta, costs);
    DistributionSpec d = make_dist(kind, lo, hi, mean, sd, 0);
    ExperimentConfig cfg;
    cfg.instance_label = "inst";
    cfg.seed = seed;
    cfg.backend = make_cfg(threads);
    cfg.search_evaluations = evals;
    std::vector<size_t> ms(m_list, m_list + nm);
    ExperimentReport rep;
    if (which == 0) rep = run_bias_experiment(inst, d, ms, reps, eval_size, ref_size, cfg);
    else if (which == 1) rep = run_convergence_experiment(inst, d, ms, reps, cfg);
    else if (which == 2) rep = run_quality_experiment(inst, d, ms, reps, eval_size, cfg);
    else if (which == 3) {
      ScalingOptions so;
      so.sizes = ms;
      so.modes = {cfg.backend};
      so.target_evaluations = eval_size;
      rep = run_scaling_benchmark(inst, d, so, cfg);
    } else {
      TimeBudgetOptions to;
      to.budgets_seconds = {0.05, 0.1, 0.2};
      to.modes = {cfg.backend};
      to.train_size = eval_size;
      rep = run_time_budget_experiment(inst, d, to, cfg);
    }
    RunMetadata meta;
    meta.command = "experiment";
    meta.seed = seed;
    std::ofstream f(out_path);
    write_report_csv(f, meta, rep.rows);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// forward_sweep (minplus.cpp:94-102) over option-sliced stages; writes every
// frontier (initial included) back to back.
REF_API int ref_forward_sweep(size_t n_stages, const size_t* rows, const size_t* cols,
                              const size_t* depth, const double* entries,
                              const double* init, size_t width, double* out) {
  try {
    std::vector<MaskedTransition> st;
    size_t off = 0;
    for (size_t s = 0; s < n_stages; ++s) {
      MaskedTransition a(rows[s], cols[s], depth[s]);
      for (size_t r = 0; r < depth[s]; ++r)
        for (size_t i = 0; i < rows[s]; ++i)
          for (size_t j = 0; j < cols[s]; ++j) a.at(i, j, r) = ExtendedCost{entries[off++]};
      st.push_back(std::move(a));
    }
    ValueFrontier f;
    f.values.resize(width);
    for (size_t k = 0; k < width; ++k) f.values[k] = ExtendedCost{init[k]};
    size_t o = 0;
    for (const ValueFrontier& fr : forward_sweep(st, f))
      for (const ExtendedCost& v : fr.values) out[o++] = v.value;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
