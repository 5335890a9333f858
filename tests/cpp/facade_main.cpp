// facade_main.cpp -- drives the C++ drop-in facade (include/scendp/*.hpp)
// exactly as a user of the reference would, and prints the results as plain
// text for tests/test_gpu_facade.py, which compares them with the real
// reference library (oracle/_ref) on identical inputs.
//
//   facade_main split <n> <Q> <hard> <beta> <inst_seed> <scen_seed> <m> <tour_seed>
//   facade_main dsirp <U> <I0> <H> <R> <seed> <m>
//   facade_main saa <n> <Q> <beta> <inst_seed> <scen_seed> <m> <max_evals> <kbatch>
//   facade_main gen <kind> <lo> <hi> <mean> <std> <seed> <entities> <steps> <count>
//   facade_main io-write <path> <rows> <count> <seed>        (no GPU)
//   facade_main io-read <path>                               (no GPU)
//   facade_main io-parse <path> <out>                        (no GPU)
//   facade_main io-write-inst <n> <Q> <hard> <beta> <inst_seed> <out>   (no GPU)
//   facade_main trials <which> <trials> <seed> <max_n>
//   facade_main dense <U> <I0> <H> <R> <seed> <m>
//   facade_main exp <which> <n> <Q> <beta> <inst_seed> <kind> <lo> <hi> <mean> <sd>
//                   <seed> <evals> <reps> <eval_size> <ref_size> <out> <m...>
#include <cstdio>
#include <fstream>
#include <cstdlib>
#include <exception>
#include <numeric>
#include <string>
#include <vector>

#include "scendp/io.hpp"
#include "scendp/minplus.hpp"
#include "scendp/oracle.hpp"
#include "scendp/oudp.hpp"
#include "scendp/saa.hpp"
#include "scendp/scenario.hpp"
#include "scendp/split.hpp"

#include "../../oracle/io_dump.hpp"
#include "../../oracle/run_batched_probe.hpp"

using namespace scendp;

namespace {

void print_vec(const char* tag, const std::vector<double>& v) {
  std::printf("%s %zu", tag, v.size());
  for (double x : v) std::printf(" %.17g", x);
  std::printf("\n");
}

template <typename I>
void print_ivec(const char* tag, const std::vector<I>& v) {
  std::printf("%s %zu", tag, v.size());
  for (I x : v) std::printf(" %lld", static_cast<long long>(x));
  std::printf("\n");
}

GiantTour tour_of(int n, unsigned long long seed) {
  GiantTour t;
  t.order.resize(n);
  std::iota(t.order.begin(), t.order.end(), 1);
  if (seed == 0) return t;
  SplitMix64 rng(seed);
  for (int i = n - 1; i > 0; --i) {  // Fisher-Yates as oracle.cpp:23-32
    const int j = static_cast<int>(rng.next_below(i + 1));
    std::swap(t.order[i], t.order[j]);
  }
  return t;
}

int run_split(char** a) {
  const int n = std::atoi(a[0]);
  const long long Q = std::atoll(a[1]);
  const bool hard = std::atoi(a[2]) != 0;
  const double beta = std::atof(a[3]);
  const unsigned long long iseed = std::strtoull(a[4], nullptr, 10);
  const unsigned long long sseed = std::strtoull(a[5], nullptr, 10);
  const std::size_t m = std::strtoull(a[6], nullptr, 10);
  const unsigned long long tseed = std::strtoull(a[7], nullptr, 10);
  RoutingInstance inst = make_random_instance(n, iseed, Q, hard, beta);
  GiantTour tour = tour_of(n, tseed);
  DistributionSpec dist = DistributionSpec::parse("uniform:1:10", sseed);
  ScenarioBatch batch = generate_scenarios(dist, n, 1, m);
  std::printf("demand_sum %llu\n",
              static_cast<unsigned long long>(std::accumulate(batch.data.begin(), batch.data.end(), 0ull)));
  auto costs = batched_split_costs(inst, tour, batch, BackendConfig::multi_thread(8));
  std::vector<double> tot(m);
  for (std::size_t w = 0; w < m; ++w) tot[w] = costs.per_scenario[w].value;
  print_vec("totals", tot);
  std::printf("mean %.17g finite %zu infeasible %zu\n", costs.mean_cost ? *costs.mean_cost : -1.0,
              costs.finite_count, costs.infeasible_count);
  auto full = batched_expected_split(inst, tour, batch, BackendConfig::single_thread());
  {
    // the same call sharded over a device list ({0, 0}: two shards on one
    // GPU) in waves of 300 scenarios: bitwise the same results
    BackendConfig sh = BackendConfig::gpu();
    sh.devices = {0, 0};
    sh.batch_size = 300;
    auto c2 = batched_split_costs(inst, tour, batch, sh);
    bool same = c2.finite_count == costs.finite_count &&
                c2.infeasible_count == costs.infeasible_count &&
                c2.mean_cost.has_value() == costs.mean_cost.has_value() &&
                (!c2.mean_cost || *c2.mean_cost == *costs.mean_cost);
    for (std::size_t w = 0; w < m && same; ++w)
      same = c2.per_scenario[w].value == costs.per_scenario[w].value;
    auto f2 = batched_expected_split(inst, tour, batch, sh);
    same = same && f2.mean_cost == full.mean_cost;
    for (std::size_t w = 0; w < m && same; ++w) {
      const SplitSolution &x = f2.per_scenario[w], &y = full.per_scenario[w];
      same = x.cuts == y.cuts && x.route_count == y.route_count && x.feasible == y.feasible &&
             x.total.value == y.total.value && x.values.values.size() == y.values.values.size();
      for (std::size_t i = 0; same && i < x.values.values.size(); ++i)
        same = x.values.values[i].value == y.values.values[i].value;
    }
    std::printf("sharded_equal %d\n", same ? 1 : 0);
    // one BatchTiming per batch (engine.hpp:150-192): waves of 300 within
    // each device shard, and on one device exactly the reference's batches
    auto timing_sizes = [](const char* name, const std::vector<BatchTiming>& t, std::size_t per) {
      std::vector<int> sz;
      bool ok = true;
      for (std::size_t i = 0; i < t.size(); ++i) {
        sz.push_back(static_cast<int>(t[i].size));
        ok = ok && t[i].batch_index == i && t[i].bytes_estimate == t[i].size * per &&
             t[i].wall_ms >= 0.0;
      }
      print_ivec(name, sz);
      std::printf("%s_ok %d\n", name, ok ? 1 : 0);
    };
    timing_sizes("timings_sharded", c2.timings, sizeof(ExtendedCost));
    BackendConfig one = BackendConfig::gpu();
    one.batch_size = 300;
    timing_sizes("timings_one", batched_split_costs(inst, tour, batch, one).timings,
                 sizeof(ExtendedCost));
    timing_sizes("timings_full", batched_expected_split(inst, tour, batch, one).timings,
                 split_per_scenario_bytes(n));
  }
  std::vector<double> v0;
  std::vector<int> c0, rcs;
  for (std::size_t w = 0; w < m && w < 4; ++w) {
    for (auto& x : full.per_scenario[w].values.values) v0.push_back(x.value);
    for (int c : full.per_scenario[w].cuts) c0.push_back(c);
  }
  for (std::size_t w = 0; w < m; ++w) rcs.push_back(full.per_scenario[w].route_count);
  print_vec("V4", v0);
  print_ivec("cuts4", c0);
  print_ivec("route_count", rcs);
  std::printf("full_mean %.17g\n", full.mean_cost ? *full.mean_cost : -1.0);
  auto gen = batched_split_costs_generated(inst, tour, dist, m, BackendConfig::gpu());
  std::vector<double> gt(m);
  for (std::size_t w = 0; w < m; ++w) gt[w] = gen.per_scenario[w].value;
  print_vec("gen_totals", gt);
  // routes of scenario 0
  for (auto [p, i] : recover_routes(full.per_scenario[0])) std::printf("route %d %d\n", p, i);
  return 0;
}

int run_dsirp(char** a) {
  CustomerSpec spec;
  spec.capacity = std::atoi(a[0]);
  spec.initial_inventory = std::atoi(a[1]);
  spec.horizon = std::atoi(a[2]);
  const int R = std::atoi(a[3]);
  const unsigned long long seed = std::strtoull(a[4], nullptr, 10);
  const std::size_t m = std::strtoull(a[5], nullptr, 10);
  spec.holding = 1.25;
  spec.stockout_multiplier = 2.5;
  DeliveryCostModel del = DeliveryCostModel::linear(spec.horizon, R, 40.0, 0.5);
  for (int t = 0; t < spec.horizon; ++t)
    for (int r = 0; r < R; ++r) {
      del.fixed[t * R + r] = 40.0 + 5.0 * r + 0.125 * t;
      del.unit[t * R + r] = 0.5 + 0.25 * r;
    }
  HoldingPenaltyModel hold;
  DistributionSpec dist = DistributionSpec::parse("uniform:0:33", seed);
  ScenarioBatch batch = generate_scenarios(dist, 1, spec.horizon, m);
  auto res = batched_expected_cost(spec, del, hold, batch, BackendConfig::gpu());
  std::vector<double> tot;
  std::vector<int> dl, q, ei, ro;
  for (std::size_t w = 0; w < m; ++w) {
    const ScheduleResult& s = res.per_scenario[w];
    tot.push_back(s.total.value);
    for (int t = 0; t < spec.horizon; ++t) {
      dl.push_back(s.deliver[t]);
      q.push_back(s.quantity[t]);
      ei.push_back(s.end_inventory[t]);
      ro.push_back(s.route_option[t]);
    }
  }
  print_vec("totals", tot);
  print_ivec("deliver", dl);
  print_ivec("quantity", q);
  print_ivec("end_inventory", ei);
  print_ivec("route_option", ro);
  std::printf("mean %.17g errors %zu\n", res.mean_cost ? *res.mean_cost : -1.0, res.error_count());
  // single-scenario API and the replay helper
  ScheduleResult one = solve_customer_scenario(spec, del, hold, batch.column(0));
  ExtendedCost replay = simulate_schedule(spec, del, hold, batch.column(0), one.deliver, one.route_option);
  std::printf("one %.17g replay %.17g\n", one.total.value, replay.value);
  return 0;
}

int run_saa(char** a) {
  const int n = std::atoi(a[0]);
  const long long Q = std::atoll(a[1]);
  const double beta = std::atof(a[2]);
  const unsigned long long iseed = std::strtoull(a[3], nullptr, 10);
  const unsigned long long sseed = std::strtoull(a[4], nullptr, 10);
  const std::size_t m = std::strtoull(a[5], nullptr, 10);
  const unsigned long long max_evals = std::strtoull(a[6], nullptr, 10);
  set_candidate_batch(std::strtoull(a[7], nullptr, 10));
  RoutingInstance inst = make_random_instance(n, iseed, Q, false, beta);
  ScenarioBatch train = generate_scenarios(DistributionSpec::parse("uniform:1:10", sseed), n, 1, m);
  SearchBudget budget;
  budget.max_evaluations = max_evals;
  SearchResult r = improve_first_stage(inst, train, BackendConfig::gpu(), budget);
  print_ivec("tour", r.tour.order);
  std::printf("value %.17g evaluations %llu best_found_at %llu\n", r.value,
              static_cast<unsigned long long>(r.evaluations),
              static_cast<unsigned long long>(r.best_found_at));
  std::vector<double> traj;
  for (auto& p : r.trajectory) traj.push_back(p.best_value);
  print_vec("trajectory", traj);
  std::printf("oos %.17g\n", out_of_sample_eval(inst, r.tour, train, BackendConfig::gpu()));
  return 0;
}

int run_gen(char** a) {
  DistributionSpec d;
  const int kind = std::atoi(a[0]);
  d.kind = kind == 0 ? DistributionSpec::Kind::kUniformInt
                     : (kind == 1 ? DistributionSpec::Kind::kTruncatedNormal
                                  : DistributionSpec::Kind::kPoisson);
  d.lo = std::atoll(a[1]);
  d.hi = std::atoll(a[2]);
  d.mean = std::atof(a[3]);
  d.stddev = std::atof(a[4]);
  d.seed = std::strtoull(a[5], nullptr, 10);
  ScenarioBatch b = generate_scenarios(d, std::strtoull(a[6], nullptr, 10),
                                       std::strtoull(a[7], nullptr, 10),
                                       std::strtoull(a[8], nullptr, 10));
  print_ivec("data", b.data);
  std::vector<std::uint32_t> col(b.rows);
  generate_scenario_column(d, 3, col);
  print_ivec("col3", col);
  return 0;
}

int run_io_write(char** a) {
  ScenarioBatch b;
  b.rows = std::strtoull(a[1], nullptr, 10);
  b.count = std::strtoull(a[2], nullptr, 10);
  SplitMix64 rng(std::strtoull(a[3], nullptr, 10));
  b.data.resize(b.rows * b.count);
  for (auto& v : b.data) v = static_cast<std::uint32_t>(rng.next() >> 40);
  write_scenario_file(b, a[0]);
  print_ivec("data", b.data);
  return 0;
}

int run_io_read(char** a) {
  ScenarioBatch b = read_scenario_file(a[0]);
  std::printf("rows %zu count %zu\n", b.rows, b.count);
  print_ivec("data", b.data);
  return 0;
}

int run_io_parse(char** a) {
  std::string text;
  try {
    text = io_dump::instance<ParsedInstance, RoutingInstance, DsirpInstance>(
        parse_instance_file(a[0]));
  } catch (const std::exception& e) {
    text = std::string("error ") + e.what() + "\n";
  }
  std::ofstream(a[1]) << text;
  return 0;
}

int run_io_write_inst(char** a) {
  RoutingInstance inst = make_random_instance(std::atoi(a[0]), std::strtoull(a[4], nullptr, 10),
                                              std::atoll(a[1]), std::atoi(a[2]) != 0,
                                              std::atof(a[3]));
  std::ofstream f(a[5]);
  write_routing_instance(inst, f);
  return 0;
}

// SAA experiment -> write_report_csv (same arguments as ref_experiment)
int run_exp(char** a, int nm) {
  const int which = std::atoi(a[0]);
  const int n = std::atoi(a[1]);
  RoutingInstance inst = make_random_instance(n, std::strtoull(a[4], nullptr, 10),
                                              std::atoll(a[2]), false, std::atof(a[3]));
  DistributionSpec d;
  const int kind = std::atoi(a[5]);
  d.kind = kind == 0 ? DistributionSpec::Kind::kUniformInt
                     : (kind == 1 ? DistributionSpec::Kind::kTruncatedNormal
                                  : DistributionSpec::Kind::kPoisson);
  d.lo = std::atoll(a[6]);
  d.hi = std::atoll(a[7]);
  d.mean = std::atof(a[8]);
  d.stddev = std::atof(a[9]);
  ExperimentConfig cfg;
  cfg.instance_label = "inst";
  cfg.seed = std::strtoull(a[10], nullptr, 10);
  cfg.backend = BackendConfig::gpu();
  cfg.search_evaluations = std::strtoull(a[11], nullptr, 10);
  const int reps = std::atoi(a[12]);
  const std::size_t eval_size = std::strtoull(a[13], nullptr, 10);
  const std::size_t ref_size = std::strtoull(a[14], nullptr, 10);
  std::vector<std::size_t> ms;
  for (int k = 0; k < nm; ++k) ms.push_back(std::strtoull(a[16 + k], nullptr, 10));
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
  meta.seed = cfg.seed;
  std::ofstream f(a[15]);
  write_report_csv(f, meta, rep.rows);
  return 0;
}

// the reference's randomized self-checks against this library
int run_trials(char** a) {
  const int which = std::atoi(a[0]);
  const std::size_t trials = std::strtoull(a[1], nullptr, 10);
  const std::uint64_t seed = std::strtoull(a[2], nullptr, 10);
  const OracleOutcome o = which == 0   ? run_split_oracle_trials(trials, seed)
                          : which == 1 ? run_split_agreement_trials(trials, seed, std::atoi(a[3]))
                                       : run_dsirp_oracle_trials(trials, seed);
  std::printf("trials %zu mismatches %zu\n", o.trials, o.mismatches);
  if (!o.ok()) std::printf("failure %s\n", o.first_failure.c_str());
  return 0;
}

// dense DSIRP path: every frontier of sweep_customer_scenario for m scenarios
// (the customer of run_dsirp), plus forward_sweep_batch of the scenario-0
// stage chain from m different start states
int run_dense(char** a) {
  CustomerSpec spec;
  spec.capacity = std::atoi(a[0]);
  spec.initial_inventory = std::atoi(a[1]);
  spec.horizon = std::atoi(a[2]);
  const int R = std::atoi(a[3]);
  const unsigned long long seed = std::strtoull(a[4], nullptr, 10);
  const std::size_t m = std::strtoull(a[5], nullptr, 10);
  spec.holding = 1.25;
  spec.stockout_multiplier = 2.5;
  DeliveryCostModel del = DeliveryCostModel::linear(spec.horizon, R, 40.0, 0.5);
  for (int t = 0; t < spec.horizon; ++t)
    for (int r = 0; r < R; ++r) {
      del.fixed[t * R + r] = 40.0 + 5.0 * r + 0.125 * t;
      del.unit[t * R + r] = 0.5 + 0.25 * r;
    }
  HoldingPenaltyModel hold;
  ScenarioBatch batch = generate_scenarios(DistributionSpec::parse("uniform:0:33", seed), 1,
                                           spec.horizon, m);
  std::vector<double> fr;
  for (std::size_t w = 0; w < m; ++w)
    for (const ValueFrontier& f : sweep_customer_scenario(spec, del, hold, batch.column(w)))
      for (const ExtendedCost& v : f.values) fr.push_back(v.value);
  print_vec("frontiers", fr);
  std::vector<MaskedTransition> stages;
  for (int t = 1; t <= spec.horizon; ++t)
    stages.push_back(build_transition_matrix(spec, del, hold, t, static_cast<int>(batch.column(0)[t - 1])));
  std::vector<ValueFrontier> starts;
  for (int s = 0; s <= spec.capacity; ++s) starts.push_back(ValueFrontier::initial(1, spec.capacity + 1, s));
  std::vector<double> last;
  for (const ValueFrontier& f : forward_sweep_batch(stages, starts))
    for (const ExtendedCost& v : f.values) last.push_back(v.value);
  print_vec("batch_last", last);
  return 0;
}

}  // namespace

int run_batched_cmd(char** a) {
  std::printf("%s\n", run_batched_probe(std::strtoull(a[0], nullptr, 10), std::strtoull(a[1], nullptr, 10),
                                         static_cast<unsigned>(std::atoi(a[2])),
                                         std::strtoull(a[3], nullptr, 10),
                                         std::strtoull(a[4], nullptr, 10)).c_str());
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string mode = argv[1];
  try {
    if (mode == "split" && argc == 10) return run_split(argv + 2);
    if (mode == "dsirp" && argc == 8) return run_dsirp(argv + 2);
    if (mode == "saa" && argc == 10) return run_saa(argv + 2);
    if (mode == "gen" && argc == 11) return run_gen(argv + 2);
    if (mode == "io-write" && argc == 6) return run_io_write(argv + 2);
    if (mode == "io-read" && argc == 3) return run_io_read(argv + 2);
    if (mode == "io-parse" && argc == 4) return run_io_parse(argv + 2);
    if (mode == "io-write-inst" && argc == 8) return run_io_write_inst(argv + 2);
    if (mode == "trials" && argc == 6) return run_trials(argv + 2);
    if (mode == "dense" && argc == 8) return run_dense(argv + 2);
    if (mode == "exp" && argc >= 19) return run_exp(argv + 2, argc - 18);
    if (mode == "batched" && argc == 7) return run_batched_cmd(argv + 2);
  } catch (const std::exception& e) {
    std::printf("exception %s\n", e.what());
    return 1;
  }
  return 2;
}
