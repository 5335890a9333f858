// oudp.cpp -- DSIRP evaluators of the drop-in facade (reference:
// proj/src/oudp.cpp).  Validators and the small replay helpers run on the
// host; the DP runs on the GPU through scendp_dsirp_eval.
#include "scendp/oudp.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>

#include "runtime.hpp"

namespace scendp {

void CustomerSpec::validate() const {
  if (capacity < 0 || capacity > 65535)
    throw std::invalid_argument("capacity U must be in [0, 65535]");
  if (initial_inventory < 0 || initial_inventory > capacity)
    throw std::invalid_argument("initial inventory must be in [0, U]");
  if (horizon < 1) throw std::invalid_argument("horizon H must be >= 1");
  if (!(holding >= 0.0)) throw std::invalid_argument("holding cost must be >= 0");
  if (!(stockout_multiplier > 1.0)) throw std::invalid_argument("stockout multiplier rho must be > 1");
}

DeliveryCostModel DeliveryCostModel::linear(int horizon, int options, double fixed_cost,
                                            double unit_cost) {
  DeliveryCostModel m;
  m.horizon = horizon;
  m.options = options;
  m.fixed.assign(static_cast<std::size_t>(horizon) * options, fixed_cost);
  m.unit.assign(static_cast<std::size_t>(horizon) * options, unit_cost);
  return m;
}

void DeliveryCostModel::validate(const CustomerSpec& spec) const {
  if (horizon != spec.horizon) throw std::invalid_argument("delivery model horizon does not match spec");
  if (options < 1 || options > 256) throw std::invalid_argument("route options R must be in [1, 256]");
  if (tabular) {
    if (table_quantities != spec.capacity + 1 ||
        table.size() != static_cast<std::size_t>(horizon) * table_quantities)
      throw std::invalid_argument("delivery table must be H x (U+1)");
    for (int t = 1; t <= horizon; ++t)
      if (table[(t - 1) * table_quantities] != 0.0)
        throw std::invalid_argument("delivery table requires F_t(0) = 0");
    for (double v : table)
      if (!std::isfinite(v) || v < 0.0)
        throw std::invalid_argument("delivery table entries must be finite and >= 0");
  } else {
    const std::size_t want = static_cast<std::size_t>(horizon) * options;
    if (fixed.size() != want || unit.size() != want)
      throw std::invalid_argument("delivery model needs H x R fixed and unit costs");
    for (std::size_t k = 0; k < want; ++k)
      if (!std::isfinite(fixed[k]) || fixed[k] < 0.0 || !std::isfinite(unit[k]) || unit[k] < 0.0)
        throw std::invalid_argument("delivery costs must be finite and >= 0");
  }
}

void HoldingPenaltyModel::validate(const CustomerSpec& spec) const {
  if (!tabular) return;
  if (table.size() != static_cast<std::size_t>(spec.capacity) + 1)
    throw std::invalid_argument("holding table must have U+1 entries");
  for (double v : table)
    if (!std::isfinite(v) || v < 0.0)
      throw std::invalid_argument("holding table entries must be finite and >= 0");
}

DayOutcome simulate_day(const CustomerSpec& spec, int inventory, int quantity, int demand) {
  if (inventory < 0 || inventory > spec.capacity) throw std::invalid_argument("inventory outside [0, U]");
  if (quantity != 0 && quantity != spec.capacity - inventory)
    throw std::invalid_argument("order-up-to quantity must be 0 or U - I, got " +
                                std::to_string(quantity));
  if (demand < 0) throw std::invalid_argument("demand must be >= 0");
  DayOutcome out;
  out.end_inventory = std::max(0, inventory + quantity - demand);
  out.shortage = std::max(0, demand - inventory - quantity);
  return out;
}

ExtendedCost simulate_schedule(const CustomerSpec& spec, const DeliveryCostModel& delivery,
                               const HoldingPenaltyModel& holding,
                               std::span<const std::uint32_t> demands,
                               std::span<const std::uint8_t> deliver,
                               std::span<const std::int32_t> route_option) {
  if (demands.size() != static_cast<std::size_t>(spec.horizon))
    throw std::invalid_argument("scenario has " + std::to_string(demands.size()) +
                                " days, spec horizon is " + std::to_string(spec.horizon));
  double total = 0.0;
  int inv = spec.initial_inventory;
  for (int t = 1; t <= spec.horizon; ++t) {
    const int d = static_cast<int>(demands[t - 1]);
    const int q = deliver[t - 1] ? spec.capacity - inv : 0;
    const int r = deliver[t - 1] ? route_option[t - 1] : 0;
    const int j = std::max(0, inv + q - d);
    const int s = std::max(0, d - inv - q);
    total += delivery.cost(t, r, q) + holding.cost(spec, j, s);
    inv = j;
  }
  return ExtendedCost{total};
}

MaskedTransition build_transition_matrix(const CustomerSpec& spec,
                                         const DeliveryCostModel& delivery,
                                         const HoldingPenaltyModel& holding, int day,
                                         int demand) {
  const int states = spec.capacity + 1;
  MaskedTransition a(states, states, 1);
  for (int i = 0; i < states; ++i) {
    // the two order-up-to actions in tie order: no delivery (one cost), then
    // a delivery of U - I over every route option (absent when I == U)
    const int full = spec.capacity - i;
    for (int act = 0; act < (full > 0 ? 2 : 1); ++act) {
      const int q = act == 0 ? 0 : full;
      const int j = std::max(0, i + q - demand);
      const int shortage = std::max(0, demand - i - q);
      const int opts = q == 0 ? 1 : delivery.options;
      for (int r = 0; r < opts; ++r)
        a.at(i, j) = extended_min(
            a.at(i, j), ExtendedCost{delivery.cost(day, r, q) + holding.cost(spec, j, shortage)});
    }
  }
  return a;
}

std::vector<ValueFrontier> sweep_customer_scenario(const CustomerSpec& spec,
                                                   const DeliveryCostModel& delivery,
                                                   const HoldingPenaltyModel& holding,
                                                   std::span<const std::uint32_t> demands) {
  spec.validate();
  delivery.validate(spec);
  holding.validate(spec);
  if (demands.size() != static_cast<std::size_t>(spec.horizon))
    throw std::invalid_argument("scenario has " + std::to_string(demands.size()) +
                                " days, spec horizon is " + std::to_string(spec.horizon));
  std::vector<MaskedTransition> stages;
  stages.reserve(spec.horizon);
  for (int t = 1; t <= spec.horizon; ++t)
    stages.push_back(
        build_transition_matrix(spec, delivery, holding, t, static_cast<int>(demands[t - 1])));
  return forward_sweep(stages, ValueFrontier::initial(1, spec.capacity + 1,
                                                      static_cast<std::size_t>(spec.initial_inventory)));
}

ExtendedCost brute_force_schedule(const CustomerSpec& spec, const DeliveryCostModel& delivery,
                                  const HoldingPenaltyModel& holding,
                                  std::span<const std::uint32_t> demands) {
  spec.validate();
  delivery.validate(spec);
  holding.validate(spec);
  if (demands.size() != static_cast<std::size_t>(spec.horizon))
    throw std::invalid_argument("scenario has " + std::to_string(demands.size()) +
                                " days, spec horizon is " + std::to_string(spec.horizon));
  if (spec.horizon > 14) throw std::invalid_argument("brute-force schedule is limited to H <= 14");
  double best = std::numeric_limits<double>::infinity();
  for (std::uint32_t pattern = 0; pattern < (1u << spec.horizon); ++pattern) {
    double total = 0.0;
    int inv = spec.initial_inventory;
    for (int t = 1; t <= spec.horizon; ++t) {
      const int d = static_cast<int>(demands[t - 1]);
      const int q = (pattern >> (t - 1)) & 1u ? spec.capacity - inv : 0;
      // options add independently per day: the cheapest one is optimal
      double f = delivery.cost(t, 0, q);
      for (int r = 1; q > 0 && r < delivery.options; ++r) f = std::min(f, delivery.cost(t, r, q));
      const int j = std::max(0, inv + q - d);
      total += f + holding.cost(spec, j, std::max(0, d - inv - q));
      inv = j;
    }
    best = std::min(best, total);
  }
  return ExtendedCost{best};
}

std::uint64_t oudp_per_scenario_bytes(const CustomerSpec& spec) {
  const std::uint64_t states = static_cast<std::uint64_t>(spec.capacity) + 1;
  const std::uint64_t h = static_cast<std::uint64_t>(spec.horizon);
  return h * states * sizeof(std::uint32_t) + 2 * states * sizeof(double) +
         h * sizeof(std::uint32_t) + h * 13 + 160;
}

FootprintModel oudp_footprint_model(const CustomerSpec& spec) {
  FootprintModel m;
  m.fixed_bytes = std::uint64_t{1} << 20;
  m.per_scenario_bytes = oudp_per_scenario_bytes(spec);
  return m;
}

namespace {

scendp_customer to_c(const CustomerSpec& spec, const DeliveryCostModel& del,
                     const HoldingPenaltyModel& hold) {
  scendp_customer c{};
  c.capacity = spec.capacity;
  c.initial_inventory = spec.initial_inventory;
  c.horizon = spec.horizon;
  c.holding = spec.holding;
  c.stockout_multiplier = spec.stockout_multiplier;
  c.options = del.options;
  c.fixed = del.fixed.data();
  c.unit = del.unit.data();
  c.delivery_tabular = del.tabular ? 1 : 0;
  c.delivery_table = del.table.data();
  c.holding_tabular = hold.tabular ? 1 : 0;
  c.holding_table = hold.table.data();
  return c;
}

// Full schedules for `count` host columns on one context.
void schedules(scendp_ctx* ctx, const scendp_customer& c, const std::uint32_t* data,
               std::size_t count, ScheduleResult* dst, std::uint8_t* evaluated) {
  const std::size_t H = static_cast<std::size_t>(c.horizon);
  // scratch filled entirely by the evaluator: default-initialized
  std::unique_ptr<double[]> totals(new double[count]);
  std::unique_ptr<std::uint8_t[]> dl(new std::uint8_t[count * H]);
  std::unique_ptr<std::int32_t[]> q(new std::int32_t[count * H]), ei(new std::int32_t[count * H]),
      ro(new std::int32_t[count * H]);
  scendp_scenarios sc{};
  sc.mem_kind = SCENDP_MEM_HOST;
  sc.data = data;
  sc.rows = H;
  sc.count = count;
  scendp_dsirp_out o{};
  o.mem_kind = SCENDP_MEM_HOST;
  o.totals = totals.get();
  o.evaluated = evaluated;
  o.deliver = dl.get();
  o.quantity = q.get();
  o.end_inventory = ei.get();
  o.route_option = ro.get();
  detail::check(scendp_dsirp_eval(ctx, &c, 1, &sc, SCENDP_DSIRP_FULL, &o));
  detail::MallocPadScope pad(std::size_t{64} << 20);
  detail::parallel_for(count, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t w = lo; w < hi; ++w) {
      if (!evaluated[w]) continue;
      ScheduleResult& r = dst[w];
      r.total = ExtendedCost{totals[w]};
      r.deliver.assign(dl.get() + w * H, dl.get() + (w + 1) * H);
      r.quantity.assign(q.get() + w * H, q.get() + (w + 1) * H);
      r.end_inventory.assign(ei.get() + w * H, ei.get() + (w + 1) * H);
      r.route_option.assign(ro.get() + w * H, ro.get() + (w + 1) * H);
    }
  });
}

constexpr const char* kAllInfinite = "inventory DP produced an all-infinite frontier";

}  // namespace

ScheduleResult solve_customer_scenario(const CustomerSpec& spec, const DeliveryCostModel& delivery,
                                       const HoldingPenaltyModel& holding,
                                       std::span<const std::uint32_t> demands) {
  spec.validate();
  delivery.validate(spec);
  holding.validate(spec);
  if (demands.size() != static_cast<std::size_t>(spec.horizon))
    throw std::invalid_argument("scenario has " + std::to_string(demands.size()) +
                                " days, spec horizon is " + std::to_string(spec.horizon));
  const scendp_customer c = to_c(spec, delivery, holding);
  ScheduleResult r;
  std::uint8_t ev = 0;
  detail::DeviceSlot& slot = detail::device_slot(-1);
  {
    std::lock_guard<std::mutex> g(slot.mu);
    detail::check(scendp_ctx_set_max_batch(slot.ctx, 0));
    schedules(slot.ctx, c, demands.data(), 1, &r, &ev);
  }
  if (!ev) throw std::logic_error(kAllInfinite);
  return r;
}

BatchResultSet<ScheduleResult> batched_expected_cost(const CustomerSpec& spec,
                                                     const DeliveryCostModel& delivery,
                                                     const HoldingPenaltyModel& holding,
                                                     const ScenarioBatch& scenarios,
                                                     const BackendConfig& cfg) {
  spec.validate();
  delivery.validate(spec);
  holding.validate(spec);
  if (scenarios.rows != static_cast<std::size_t>(spec.horizon))
    throw std::invalid_argument("scenario batch rows must equal the horizon");
  BatchResultSet<ScheduleResult> out;
  const std::size_t m = scenarios.count;
  const std::size_t wave = detail::wave_size(cfg, m, oudp_per_scenario_bytes(spec), &out.warnings);
  out.per_scenario.resize(m);
  out.evaluated.assign(m, 0);
  if (m == 0) return out;
  const scendp_customer c = to_c(spec, delivery, holding);
  const auto waves = detail::make_waves(detail::make_shards(m, detail::devices_of(cfg)), wave);
  detail::run_waves(waves, oudp_per_scenario_bytes(spec), &out.timings,
                    [&](std::size_t, const detail::Shard& s, scendp_ctx* ctx) {
    detail::check(scendp_ctx_set_max_batch(ctx, wave));
    schedules(ctx, c, scenarios.data.data() + s.lo * scenarios.rows, s.hi - s.lo,
              out.per_scenario.data() + s.lo, out.evaluated.data() + s.lo);
  });
  for (std::size_t w = 0; w < m; ++w)
    if (!out.evaluated[w]) out.errors.emplace(w, kAllInfinite);
  detail::sequential_aggregate(out, [](const ScheduleResult& r) { return r.total.value; });
  return out;
}

std::vector<ExactAggregate> batched_expected_cost_multi(const std::vector<DsirpCustomer>& customers,
                                                        const ScenarioBatch& scenarios,
                                                        const BackendConfig& cfg) {
  if (customers.empty()) return {};
  const int H = customers.front().spec.horizon;
  std::vector<scendp_customer> cs;
  for (const DsirpCustomer& c : customers) {
    c.spec.validate();
    c.delivery.validate(c.spec);
    c.holding.validate(c.spec);
    if (c.spec.horizon != H)
      throw std::invalid_argument("all customers of a call must share the horizon");
    cs.push_back(to_c(c.spec, c.delivery, c.holding));
  }
  if (scenarios.rows != customers.size() * static_cast<std::size_t>(H))
    throw std::invalid_argument("scenario batch rows must equal customers x horizon");
  const std::uint32_t nc = static_cast<std::uint32_t>(customers.size());
  const auto shards = detail::make_shards(scenarios.count, detail::devices_of(cfg));
  std::vector<scendp_agg_raw> raw(shards.size() * nc);
  detail::run_shards(shards, [&](const detail::Shard& s, scendp_ctx* ctx) {
    detail::check(scendp_ctx_set_max_batch(ctx, 0));
    scendp_scenarios sc{};
    sc.mem_kind = SCENDP_MEM_HOST;
    sc.data = scenarios.data.data() + s.lo * scenarios.rows;
    sc.rows = scenarios.rows;
    sc.count = s.hi - s.lo;
    scendp_dsirp_out o{};
    o.mem_kind = SCENDP_MEM_HOST;
    o.agg_raw = raw.data() + (&s - shards.data()) * nc;
    detail::check(scendp_dsirp_eval(ctx, cs.data(), nc, &sc, SCENDP_DSIRP_COST_ONLY, &o));
  });
  std::vector<scendp_agg> agg(nc);
  detail::check(scendp_agg_finalize(raw.data(), static_cast<std::uint32_t>(shards.size()), nc,
                                    agg.data()));
  std::vector<ExactAggregate> out(nc);
  for (std::uint32_t c = 0; c < nc; ++c) out[c] = detail::to_exact(agg[c]);
  return out;
}

}  // namespace scendp
