// facade_bench.cpp -- wall-clock timing of the C++ drop-in facade calls at
// the BASELINE C2 shape (n = 200, 10^6 scenarios, uniform:1:10) and of
// batched_expected_cost at U = 100, H = 6, R = 3, 10^5 scenarios: what a user
// of the reference's headers sees after relinking against this library.
// Build (from the repo root, after make):
//   g++ -std=c++20 -O2 -Iinclude profiles/facade_bench.cpp -o profiles/facade_bench \
//     -Lpaper_2602_05179_b200 -lscendp_b200 -nostdlib++ -l:libstdc++.so.6 \
//     -Wl,-rpath,'$ORIGIN/../paper_2602_05179_b200'
// Results: profiles/r01_facade.txt, profiles/r02_facade.txt.
#include <chrono>
#include <cstdio>
#include <numeric>
#include "scendp/split.hpp"
#include "scendp/oudp.hpp"
#include "scendp/saa.hpp"
using namespace scendp;
int main() {
  const int n = 200; const std::size_t m = 1000000;
  RoutingInstance inst = make_random_instance(n, 1, 100, true, 0.0);
  GiantTour tour; tour.order.resize(n); std::iota(tour.order.begin(), tour.order.end(), 1);
  auto dist = DistributionSpec::parse("uniform:1:10", 7);
  { auto w = generate_scenarios(dist, n, 1, 64); (void)batched_split_costs(inst, tour, w, BackendConfig::gpu()); }
  auto t0 = std::chrono::steady_clock::now();
  ScenarioBatch b = generate_scenarios(dist, n, 1, m);
  auto t1 = std::chrono::steady_clock::now();
  auto r1 = batched_split_costs(inst, tour, b, BackendConfig::gpu());
  r1 = batched_split_costs(inst, tour, b, BackendConfig::gpu());
  auto t2 = std::chrono::steady_clock::now();
  auto r2 = batched_expected_split(inst, tour, b, BackendConfig::gpu());
  auto t25 = std::chrono::steady_clock::now();
  r2 = batched_expected_split(inst, tour, b, BackendConfig::gpu());
  auto t3 = std::chrono::steady_clock::now();
  auto r3 = batched_split_costs_generated(inst, tour, dist, m, BackendConfig::gpu());
  auto t35 = std::chrono::steady_clock::now();  // second call timed (first: scratch growth)
  r3 = batched_split_costs_generated(inst, tour, dist, m, BackendConfig::gpu());
  auto t4 = std::chrono::steady_clock::now();
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  std::printf("generate_scenarios %.1f ms\nbatched_split_costs %.1f ms\nbatched_expected_split %.1f ms\nbatched_split_costs_generated %.1f ms\n",
              ms(t0, t1), ms(t1, t2) / 2, ms(t25, t3), ms(t35, t4));
  std::printf("first expected_split %.1f ms\n", ms(t2, t25));
  std::printf("means %.6f %.6f %.6f\n", *r1.mean_cost, *r2.mean_cost, *r3.mean_cost);
  {
    CustomerSpec spec; spec.capacity = 100; spec.initial_inventory = 50; spec.horizon = 6; spec.holding = 1.0;
    auto del = DeliveryCostModel::linear(6, 3, 10.0, 0.5);
    HoldingPenaltyModel hold;
    auto dd = DistributionSpec::parse("uniform:0:40", 3);
    ScenarioBatch sb = generate_scenarios(dd, 1, 6, 100000);
    auto a0 = std::chrono::steady_clock::now();
    auto q1 = batched_expected_cost(spec, del, hold, sb, BackendConfig::gpu());
    auto a1 = std::chrono::steady_clock::now();
    q1 = batched_expected_cost(spec, del, hold, sb, BackendConfig::gpu());
    auto a2 = std::chrono::steady_clock::now();
    std::printf("batched_expected_cost C3-unit 1e5: first %.1f ms, second %.1f ms mean %.6f\n", ms(a0, a1), ms(a1, a2), *q1.mean_cost);
  }
  {
    // SAA first-improvement search (saa.cpp:106-189), n = 50, beta = 10,
    // 10^5 training scenarios, 2000 candidate evaluations
    RoutingInstance pin = make_random_instance(50, 5, 100, false, 10.0);
    ScenarioBatch train = generate_scenarios(DistributionSpec::parse("uniform:1:10", 11), 50, 1, 100000);
    SearchBudget budget;
    budget.max_evaluations = 2000;
    (void)improve_first_stage(pin, train, BackendConfig::gpu(), SearchBudget{20, budget.max_wall_seconds});
    auto s0 = std::chrono::steady_clock::now();
    SearchResult r = improve_first_stage(pin, train, BackendConfig::gpu(), budget);
    auto s1 = std::chrono::steady_clock::now();
    std::printf("improve_first_stage n=50 m=1e5: %llu evaluations in %.1f ms (%.3f ms/evaluation), value %.6f\n",
                static_cast<unsigned long long>(r.evaluations), ms(s0, s1),
                ms(s0, s1) / static_cast<double>(r.evaluations), r.value);
  }
  return 0;
}
