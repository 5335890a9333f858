// dsirp.cu -- K3: the DSIRP order-up-to inventory DP over (customer, scenario).
//
// Reference (paths under /root/reference/proj):
//   forward_pass          src/oudp.cpp:40-87    dense frontier, two scans/day
//   pick_terminal         src/oudp.cpp:94-106   smallest state, first minimum
//   assemble_schedule     src/oudp.cpp:108-132
//   batched_expected_cost src/oudp.cpp:398-438  one customer, rows == H
//   validators            src/oudp.cpp:136-207
//
// B200 formulation.  Starting from the single state I0, day t maps every
// reachable state i to max(0, i-d) (no delivery) and adds exactly one new
// state max(0, U-d) (order-up-to delivery), so at most t+1 states are
// reachable after day t.  Each thread keeps that sparse frontier in
// registers as slots; slot e is created on day e and all slots shift by the
// same demand, so slot order == state order (equal states only at 0, where
// the first strict minimum survives, exactly like the reference's ascending
// strict-< scan into b[0]).  The delivery candidate is the first minimum over
// (r outer, state inner) of a[i] + (F(t,r,U-i) + hold(j1,s1)), merged into the
// no-delivery value at j1 with strict <.  Schedules are tracked forward: a
// per-slot delivery bitmask plus one route option per day (only one delivery
// target exists per day), then replayed from I0.
//
// One thread per (customer, scenario); a CTA = one customer x 128 scenarios,
// so customer parameters are CTA-uniform (shared memory) and demand rows
// c*H+t are coalesced 128-byte lines of the tiled layout.
#include <algorithm>
#include <string_view>
#include <unordered_map>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

using namespace scendp_dev;
using namespace scendp_host;

namespace scendp_host {
template <typename T>
void launch_from_tiled(scendp_ctx* ctx, const T* src, uint64_t rows, uint64_t count, T* dst);
}

#include "dsirp_kernels.cuh"

using namespace scendp_dsirp;

namespace scendp_dsirp {

}  // namespace scendp_dsirp

namespace {

constexpr double kInfH = std::numeric_limits<double>::infinity();
constexpr size_t kFastSmemMax = 48 * 1024;  // fast-form customer tables in shared memory

// ---- host ----------------------------------------------------------------
void validate_customer(const scendp_customer& s, int H) {
  if (s.capacity < 0 || s.capacity > 65535)
    fail(SCENDP_ERR_INVALID_ARGUMENT, "capacity U must be in [0, 65535]");
  if (s.initial_inventory < 0 || s.initial_inventory > s.capacity)
    fail(SCENDP_ERR_INVALID_ARGUMENT, "initial inventory must be in [0, U]");
  if (s.horizon < 1) fail(SCENDP_ERR_INVALID_ARGUMENT, "horizon H must be >= 1");
  if (!(s.holding >= 0.0)) fail(SCENDP_ERR_INVALID_ARGUMENT, "holding cost must be >= 0");
  if (!(s.stockout_multiplier > 1.0))
    fail(SCENDP_ERR_INVALID_ARGUMENT, "stockout multiplier rho must be > 1");
  if (s.horizon != H)
    fail(SCENDP_ERR_INVALID_ARGUMENT, "all customers of a call must share the horizon");
  if (s.options < 1 || s.options > 256)
    fail(SCENDP_ERR_INVALID_ARGUMENT, "route options R must be in [1, 256]");
  const size_t HR = static_cast<size_t>(H) * s.options;
  if (s.delivery_tabular) {
    if (!s.delivery_table) fail(SCENDP_ERR_INVALID_ARGUMENT, "delivery table must be H x (U+1)");
    for (int t = 0; t < H; ++t)
      if (s.delivery_table[static_cast<size_t>(t) * (s.capacity + 1)] != 0.0)
        fail(SCENDP_ERR_INVALID_ARGUMENT, "delivery table requires F_t(0) = 0");
    for (size_t x = 0; x < static_cast<size_t>(H) * (s.capacity + 1); ++x) {
      const double v = s.delivery_table[x];
      if (!std::isfinite(v) || v < 0.0)
        fail(SCENDP_ERR_INVALID_ARGUMENT, "delivery table entries must be finite and >= 0");
    }
  } else {
    if (!s.fixed || !s.unit)
      fail(SCENDP_ERR_INVALID_ARGUMENT, "delivery model needs H x R fixed and unit costs");
    for (size_t x = 0; x < HR; ++x)
      if (!std::isfinite(s.fixed[x]) || s.fixed[x] < 0.0 || !std::isfinite(s.unit[x]) ||
          s.unit[x] < 0.0)
        fail(SCENDP_ERR_INVALID_ARGUMENT, "delivery costs must be finite and >= 0");
  }
  if (s.holding_tabular) {
    if (!s.holding_table) fail(SCENDP_ERR_INVALID_ARGUMENT, "holding table must have U+1 entries");
    for (int j = 0; j <= s.capacity; ++j)
      if (!std::isfinite(s.holding_table[j]) || s.holding_table[j] < 0.0)
        fail(SCENDP_ERR_INVALID_ARGUMENT, "holding table entries must be finite and >= 0");
  }
}

// Exact scaled-integer eligibility of one customer (dsirp_int_kernel): every
// parameter the reference multiplies or adds is a multiple of 2^-shift and
// every path cost stays below 2^22 after scaling, for demands <= dlim.
bool prepare_int(const scendp_customer& s, int H, CustDev& d, std::vector<int32_t>& ipool) {
  constexpr double kBound = 4194304.0;  // 2^22
  const int U = s.capacity, R = s.options;
  const double rh = s.stockout_multiplier * s.holding;  // the reference's rounding
  std::vector<double> vals = {s.holding, rh};
  if (s.delivery_tabular) vals.insert(vals.end(), s.delivery_table, s.delivery_table + static_cast<size_t>(H) * (U + 1));
  else {
    vals.insert(vals.end(), s.fixed, s.fixed + static_cast<size_t>(H) * R);
    vals.insert(vals.end(), s.unit, s.unit + static_cast<size_t>(H) * R);
  }
  if (s.holding_tabular) vals.insert(vals.end(), s.holding_table, s.holding_table + U + 1);
  int shift = -1;
  for (int k = 0; k <= 12 && shift < 0; ++k) {
    const double sc = std::ldexp(1.0, k);
    bool ok = true;
    for (double v : vals) {
      const double x = v * sc;
      if (!(x < kBound) || x != std::floor(x)) { ok = false; break; }
    }
    if (ok) shift = k;
  }
  if (shift < 0) return false;
  const double sc = std::ldexp(1.0, shift);
  // per (day, quantity): minimal scaled F and the first option attaining it
  const size_t base = ipool.size();
  // q = 0 (state U: no delivery possible) holds INT32_MIN, read as the
  // unsigned key 0x80000000 by the fast kernel, above every real key
  ipool.resize(base + static_cast<size_t>(H) * (U + 1), INT32_MIN);
  double maxF = 0.0;
  for (int t = 0; t < H; ++t)
    for (int q = 1; q <= U; ++q) {
      double best = 0.0;
      int br = -1;
      for (int r = 0; r < (s.delivery_tabular ? 1 : R); ++r) {
        const double F = s.delivery_tabular ? s.delivery_table[static_cast<size_t>(t) * (U + 1) + q] * sc
                                            : s.fixed[t * R + r] * sc + s.unit[t * R + r] * sc * q;
        if (br < 0 || F < best) { best = F; br = r; }
      }
      if (!(best < kBound)) return false;
      maxF = std::max(maxF, best);
      ipool[base + static_cast<size_t>(t) * (U + 1) + q] =
          (static_cast<int32_t>(best) << 8) | br;
    }
  double maxHoldJ = 0.0;
  size_t htab_off = 0;
  if (s.holding_tabular) {
    htab_off = ipool.size();
    for (int j = 0; j <= U; ++j) {
      ipool.push_back(static_cast<int32_t>(s.holding_table[j] * sc));
      maxHoldJ = std::max(maxHoldJ, s.holding_table[j] * sc);
    }
  } else {
    maxHoldJ = s.holding * sc * U;
  }
  const double perday = kBound / H - maxF - maxHoldJ;
  if (!(perday > 0.0)) return false;
  double dlim = 1073741824.0;
  if (!s.holding_tabular && rh * sc > 0.0) dlim = std::min(dlim, std::floor(perday / (rh * sc)));
  d.int_ok = 1;
  d.shift = shift;
  d.h_i = static_cast<int32_t>(s.holding * sc);
  d.rh_i = static_cast<int32_t>(rh * sc);
  d.dlim = static_cast<int32_t>(dlim);
  d.off_gkey = base;
  d.off_htab_i = htab_off;
  return true;
}

// Bytes of everything the device tables of one customer depend on (the
// scenarios, outputs and flags aside): equal bytes => equal tables.
void append_customer_key(const scendp_customer& s, int H, std::vector<char>& key) {
  auto put = [&key](const void* p, size_t n) {
    const char* c = static_cast<const char*>(p);
    key.insert(key.end(), c, c + n);
  };
  const int32_t ints[6] = {s.capacity, s.initial_inventory, H, s.options, s.delivery_tabular,
                           s.holding_tabular};
  const double dbl[2] = {s.holding, s.stockout_multiplier};
  put(ints, sizeof(ints));
  put(dbl, sizeof(dbl));
  const size_t HR = static_cast<size_t>(H) * s.options;
  if (s.delivery_tabular) {
    put(s.delivery_table, static_cast<size_t>(H) * (s.capacity + 1) * 8);
  } else {
    put(s.fixed, HR * 8);
    put(s.unit, HR * 8);
  }
  if (s.holding_tabular) put(s.holding_table, static_cast<size_t>(s.capacity + 1) * 8);
}

// Device footprint model of one scendp_dsirp_eval call (device analogue of
// the reference's oudp footprint, oudp.cpp:383-396): fixed bytes (customer
// tables, aggregates, dense long-horizon scratch), bytes per scenario of a
// wave (staged input, host-bound outputs), and the wave under the budget.
struct DsirpFootprint {
  uint64_t fixed = 0, per_scenario = 0, wave = 0, budget = 0;
};

DsirpFootprint dsirp_footprint(scendp_ctx* ctx, uint32_t nc, int H, const scendp_scenarios* sc,
                               uint32_t flags, const scendp_dsirp_out* out, uint64_t table_bytes) {
  const bool full = (flags & SCENDP_DSIRP_FULL) != 0;
  const bool host_out = out->mem_kind == SCENDP_MEM_HOST;
  const uint64_t NC = nc, Hh = static_cast<uint64_t>(H);
  DsirpFootprint f;
  f.fixed = table_bytes + NC * sizeof(scendp_agg_raw) + (H > 32 ? (512ull << 20) : 0);
  uint64_t in_fixed = 0;
  f.per_scenario = stage_footprint(sc, &in_fixed);
  f.fixed += in_fixed;
  if (host_out && out->totals && !mapped_host_alias(out->totals)) f.per_scenario += NC * 8;
  if (host_out && out->evaluated) f.per_scenario += NC;
  if (full && out->mem_kind != SCENDP_MEM_DEVICE_TILED) f.per_scenario += 13 * NC * Hh;  // tiled
  if (full && host_out) f.per_scenario += 13 * NC * Hh;  // reference layout
  f.wave = ctx->wave_for_model(sc->count, f.fixed, f.per_scenario, &f.budget);
  return f;
}

struct DsirpWaveBufs {
  double* totals = nullptr;
  uint8_t* evaluated = nullptr;
  uint8_t *dl = nullptr, *r_dl = nullptr;
  int32_t *q = nullptr, *ei = nullptr, *ro = nullptr, *r_q = nullptr, *r_ei = nullptr,
          *r_ro = nullptr;
};

DsirpWaveBufs reserve_dsirp_wave(scendp_ctx* ctx, uint32_t nc, int H, const scendp_scenarios* sc,
                                 bool full, const scendp_dsirp_out* out, bool call_totals,
                                 uint64_t mw) {
  const bool host_out = out->mem_kind == SCENDP_MEM_HOST;
  const uint64_t NC = nc, Hh = static_cast<uint64_t>(H), fcount = NC * ((mw + 31) / 32) * 32 * Hh;
  DsirpWaveBufs b;
  reserve_stage(ctx, sc, mw);
  if (host_out && out->totals && !call_totals)
    b.totals = static_cast<double*>(ctx->scratch_get(kScrTotals, NC * mw * 8));
  if (host_out && out->evaluated) b.evaluated = static_cast<uint8_t*>(ctx->scratch_get(kScrOut5, NC * mw));
  if (full && out->mem_kind != SCENDP_MEM_DEVICE_TILED) {
    b.dl = static_cast<uint8_t*>(ctx->scratch_get(kScrOut1, fcount));
    b.q = static_cast<int32_t*>(ctx->scratch_get(kScrOut2, fcount * 4));
    b.ei = static_cast<int32_t*>(ctx->scratch_get(kScrOut3, fcount * 4));
    b.ro = static_cast<int32_t*>(ctx->scratch_get(kScrOut4, fcount * 4));
  }
  if (full && host_out) {
    b.r_dl = static_cast<uint8_t*>(ctx->scratch_get(kScrOut7, NC * mw * Hh));
    b.r_q = static_cast<int32_t*>(ctx->scratch_get(kScrOut6, NC * mw * Hh * 4));
    b.r_ei = static_cast<int32_t*>(ctx->scratch_get(kScrOut8, NC * mw * Hh * 4));
    b.r_ro = static_cast<int32_t*>(ctx->scratch_get(kScrOut9, NC * mw * Hh * 4));
  }
  return b;
}

// rows x wave_pitch bytes of per-wave scratch -> host rows of host_pitch
// bytes at byte offset `off` (one contiguous copy for a single-wave call).
template <typename T>
void copy_rows_back(scendp_ctx* ctx, T* host, const T* dev, uint64_t rows, uint64_t host_pitch,
                    uint64_t wave_pitch, uint64_t off) {
  char* h = reinterpret_cast<char*>(host) + off;
  if (host_pitch == wave_pitch || rows == 1) {
    download(ctx, h, dev, rows * wave_pitch);
  } else {
    CUDA_CHECK(cudaMemcpy2DAsync(h, host_pitch, dev, wave_pitch, wave_pitch, rows,
                                 cudaMemcpyDeviceToHost, ctx->stream));
    ctx->stats.d2h_bytes += rows * wave_pitch;
  }
}

}  // namespace

extern "C" scendp_status scendp_dsirp_eval(scendp_ctx* ctx, const scendp_customer* customers,
                                           uint32_t n_customers, const scendp_scenarios* sc,
                                           uint32_t flags, const scendp_dsirp_out* out) {
  NvtxRange nvtx("scendp_dsirp_eval");
  return guard([&] {
    if (!ctx) fail(SCENDP_ERR_INVALID_ARGUMENT, "ctx is null");
    if (!customers || n_customers == 0) fail(SCENDP_ERR_INVALID_ARGUMENT, "need at least one customer");
    if (!sc || !out) fail(SCENDP_ERR_INVALID_ARGUMENT, "scenarios/out is null");
    if (n_customers > 65535) fail(SCENDP_ERR_UNSUPPORTED, "at most 65535 customers per call");
    const int H = customers[0].horizon;
    for (uint32_t c = 0; c < n_customers; ++c) validate_customer(customers[c], H);
    if (sc->rows != static_cast<uint64_t>(n_customers) * H)
      fail(SCENDP_ERR_INVALID_ARGUMENT, "scenario batch rows must equal customers x horizon");
    const bool full = (flags & SCENDP_DSIRP_FULL) != 0;
    if (full && (!out->deliver || !out->quantity || !out->end_inventory || !out->route_option))
      fail(SCENDP_ERR_INVALID_ARGUMENT, "full mode needs deliver, quantity, end_inventory, route_option");
    const uint64_t m = sc->count;
    const uint32_t nc = n_customers;
    CUDA_CHECK(cudaSetDevice(ctx->device));

    // customer records + parameter pools.  Customers with identical
    // parameters share one table set; a call whose whole customer set equals
    // the previous call's reuses the device tables as they are.
    const bool want_int = !(flags & SCENDP_DSIRP_FP64);
    std::vector<char> key;
    std::vector<size_t> kofs(nc + 1, 0);
    for (uint32_t c = 0; c < nc; ++c) {
      append_customer_key(customers[c], H, key);
      kofs[c + 1] = key.size();
    }
    key.push_back(want_int ? 1 : 0);
    bool int_path;
    bool fast_fp64 = true;  // every customer admits the fast fp64 form
    int maxR = 1;
    if (!ctx->dsirp_key.empty() && ctx->dsirp_key == key) {
      int_path = ctx->dsirp_int_path;
      maxR = ctx->dsirp_maxR;
      fast_fp64 = ctx->dsirp_fast_fp64;
    } else {
      std::vector<CustDev> cds(nc, CustDev{});
      std::vector<double> pool;
      std::vector<int32_t> ipool;
      int_path = want_int;
      std::unordered_map<std::string_view, uint32_t> seen;  // key bytes -> first customer
      for (uint32_t c = 0; c < nc; ++c) {
        const scendp_customer& s = customers[c];
        maxR = std::max(maxR, s.options);
        const std::string_view kc(key.data() + kofs[c], kofs[c + 1] - kofs[c]);
        const auto hit = seen.find(kc);
        if (hit != seen.end()) {
          cds[c] = cds[hit->second];
          continue;
        }
        seen.emplace(kc, c);
        CustDev& d = cds[c];
        d.U = s.capacity;
        d.I0 = s.initial_inventory;
        d.H = H;
        d.R = s.options;
        d.h = s.holding;
        d.rh = s.stockout_multiplier * s.holding;
        d.del_tab = s.delivery_tabular;
        d.hold_tab = s.holding_tabular;
        const size_t HR = static_cast<size_t>(H) * s.options;
        d.off_fixed = pool.size();
        if (!s.delivery_tabular) pool.insert(pool.end(), s.fixed, s.fixed + HR);
        d.off_unit = pool.size();
        if (!s.delivery_tabular) pool.insert(pool.end(), s.unit, s.unit + HR);
        d.off_dtable = pool.size();
        if (s.delivery_tabular)
          pool.insert(pool.end(), s.delivery_table, s.delivery_table + static_cast<size_t>(H) * (s.capacity + 1));
        d.off_htable = pool.size();
        if (s.holding_tabular) pool.insert(pool.end(), s.holding_table, s.holding_table + s.capacity + 1);
        // fast fp64 form: min over r of the reference's rounded F(t, r, q)
        // (DeliveryCostModel::cost, oudp.hpp:40-45), +inf at q = 0
        d.off_fmin = pool.size();
        for (int t = 0; t < H; ++t) {
          pool.push_back(kInfH);
          for (int q = 1; q <= s.capacity; ++q) {
            double best = kInfH;
            if (s.delivery_tabular) {
              best = s.delivery_table[static_cast<size_t>(t) * (s.capacity + 1) + q];
            } else {
              for (int r = 0; r < s.options; ++r) {
                const double F = s.fixed[t * s.options + r] + s.unit[t * s.options + r] * static_cast<double>(q);
                if (F < best) best = F;
              }
            }
            pool.push_back(best);
          }
        }
        fast_fp64 &= std::isfinite(d.rh);
        // exact scaled-integer path when every customer admits it
        if (int_path) int_path = prepare_int(s, H, d, ipool);
      }
      if (pool.empty()) pool.push_back(0.0);
      if (ipool.empty()) ipool.push_back(0);
      const size_t o_pool = (nc * sizeof(CustDev) + 15) & ~size_t(15);
      const size_t o_ipool = (o_pool + pool.size() * 8 + 15) & ~size_t(15);
      ctx->dsirp_key.clear();
      char* dc = static_cast<char*>(ctx->scratch_get(kScrCustomers, o_ipool + ipool.size() * 4));
      ctx->copy(dc, cds.data(), nc * sizeof(CustDev), cudaMemcpyHostToDevice);
      ctx->copy(dc + o_pool, pool.data(), pool.size() * 8, cudaMemcpyHostToDevice);
      ctx->copy(dc + o_ipool, ipool.data(), ipool.size() * 4, cudaMemcpyHostToDevice);
      ctx->dsirp_key = std::move(key);
      ctx->dsirp_int_path = int_path;
      ctx->dsirp_maxR = maxR;
      ctx->dsirp_fast_fp64 = fast_fp64;
      ctx->dsirp_o_pool = o_pool;
      ctx->dsirp_o_ipool = o_ipool;
    }
    // layout of kScrCustomers (rebuilt above or reused): records | pool | ipool
    char* dcust = static_cast<char*>(ctx->scratch[kScrCustomers]);
    const CustDev* d_cust = reinterpret_cast<const CustDev*>(dcust);
    const double* d_pool = reinterpret_cast<const double*>(dcust + ctx->dsirp_o_pool);
    const int32_t* d_ipool = reinterpret_cast<const int32_t*>(dcust + ctx->dsirp_o_ipool);
    const size_t smem = static_cast<size_t>(H) * maxR * 2 * sizeof(double);

    auto* d_agg = static_cast<unsigned long long*>(ctx->agg_buffer(nc * sizeof(scendp_agg_raw)));
    CUDA_CHECK(cudaMemsetAsync(d_agg, 0, nc * sizeof(scendp_agg_raw), ctx->stream));

    // outputs: the caller's device buffers and page-locked host totals are
    // written in place at each wave's offset; whatever is bound for pageable
    // host memory goes through per-wave scratch, copied back after its wave
    const bool out_dev_tiled = out->mem_kind == SCENDP_MEM_DEVICE_TILED;
    const bool out_dev_ref = out->mem_kind == SCENDP_MEM_DEVICE;
    const bool host_out = out->mem_kind == SCENDP_MEM_HOST;
    double* zc_totals = host_out ? static_cast<double*>(mapped_host_alias(out->totals)) : nullptr;
    double* call_totals = !out->totals ? nullptr : host_out ? zc_totals : out->totals;

    int max_u = 0;
    for (uint32_t c = 0; c < nc; ++c) max_u = std::max(max_u, customers[c].capacity);
    // device footprint model -> wave size
    const DsirpFootprint fpm = dsirp_footprint(ctx, nc, H, sc, flags, out,
                                               ctx->scratch_bytes[kScrCustomers]);
    uint64_t wave = fpm.wave;
    const uint64_t Hh = static_cast<uint64_t>(H);
    for (uint64_t w0 = 0; w0 < m;) {
      const uint64_t mw = std::min(wave, m - w0);
      const uint64_t wtiles = (mw + 31) / 32;
      DsirpWaveBufs wb;
      try {
        wb = reserve_dsirp_wave(ctx, nc, H, sc, full, out, call_totals != nullptr, mw);
      } catch (const Error& e) {
        if (e.status != SCENDP_ERR_OUT_OF_MEMORY || wave <= 32) throw;
        wave = std::max<uint64_t>(32, (wave / 2) & ~uint64_t{31});
        release_wave_scratch(ctx);
        ++ctx->oom_retries;
        continue;
      }
      ctx->last_wave = wave;
      scendp_scenarios sw = *sc;
      sw.count = mw;
      sw.first_index = sc->first_index + w0;
      if (sc->mem_kind == SCENDP_MEM_DEVICE_TILED) sw.data = sc->data + (w0 / 32) * sc->rows * 32;
      else if (sc->mem_kind == SCENDP_MEM_HOST || sc->mem_kind == SCENDP_MEM_DEVICE)
        sw.data = sc->data + w0 * sc->rows;
      GenParams gp{};
      bool fused = false;
      const uint32_t* tiled = stage_scenarios(ctx, &sw, true, &gp, &fused);
      DsirpArgs a{};
      a.cust = d_cust;
      a.pool = d_pool;
      a.ipool = d_ipool;
      a.nc = nc;
      a.H = H;
      a.all_std_hold = 1;
      for (uint32_t c = 0; c < nc; ++c) a.all_std_hold &= customers[c].holding_tabular ? 0 : 1;
      a.rows = sc->rows;
      a.m_wave = mw;
      // wave-local addressing: call-level destinations at the wave's offset
      a.w_base = 0;
      a.tiled = fused ? nullptr : tiled;
      a.gen = gp;
      a.totals = !out->totals ? nullptr : call_totals ? call_totals + w0 : wb.totals;
      a.tot_stride = call_totals ? m : mw;
      a.evaluated = !out->evaluated ? nullptr : host_out ? wb.evaluated : out->evaluated + w0;
      a.ev_stride = host_out ? mw : m;
      if (full) {
        const uint64_t toff = (w0 / 32) * Hh * 32;
        a.deliver = out_dev_tiled ? out->deliver + toff : wb.dl;
        a.quantity = out_dev_tiled ? out->quantity + toff : wb.q;
        a.end_inventory = out_dev_tiled ? out->end_inventory + toff : wb.ei;
        a.route_option = out_dev_tiled ? out->route_option + toff : wb.ro;
        a.sched_tiles = out_dev_tiled ? (m + 31) / 32 : wtiles;
      }
      a.agg = d_agg;
      // fast form (H <= 8) when the customer tables fit in shared memory:
      // the exact-integer path (cost-only and schedules) and fp64 cost-only
      const size_t vt = int_path ? 4 : 8;
      const size_t fast_smem = (static_cast<size_t>(H) + (a.all_std_hold ? 0 : 1)) * (max_u + 1) * vt;
      const bool fast = H <= 8 && fast_smem <= kFastSmemMax && (int_path || (!full && fast_fp64));
      if (fast) launch_fast(ctx, a, fast_smem, int_path, full);
      else if (H <= 8) launch_exact(ctx, a, smem, int_path, full);
      else if (H <= 16) launch_h16(ctx, a, smem, int_path, full);
      else if (H <= 32) launch_h32(ctx, a, smem, int_path, full);
      else launch_long(ctx, a, full, max_u, H);  // the reference's dense pass

      // per-wave copies back
      if (host_out) {
        if (out->totals && !call_totals)
          copy_rows_back(ctx, out->totals, wb.totals, nc, m * 8, mw * 8, w0 * 8);
        if (out->evaluated) copy_rows_back(ctx, out->evaluated, wb.evaluated, nc, m, mw, w0);
      }
      if (full && !out_dev_tiled) {
        // tiled [c][mw/32][H][32] -> [c][mw][H], into the caller's device
        // buffers at the wave's rows or through scratch to host memory
        for (uint32_t c = 0; c < nc; ++c) {
          const uint64_t src = static_cast<uint64_t>(c) * wtiles * 32 * Hh;
          const uint64_t dst = out_dev_ref ? (static_cast<uint64_t>(c) * m + w0) * Hh
                                           : static_cast<uint64_t>(c) * mw * Hh;
          launch_from_tiled<uint8_t>(ctx, wb.dl + src, Hh, mw, (out_dev_ref ? out->deliver : wb.r_dl) + dst);
          launch_from_tiled<int32_t>(ctx, wb.q + src, Hh, mw, (out_dev_ref ? out->quantity : wb.r_q) + dst);
          launch_from_tiled<int32_t>(ctx, wb.ei + src, Hh, mw, (out_dev_ref ? out->end_inventory : wb.r_ei) + dst);
          launch_from_tiled<int32_t>(ctx, wb.ro + src, Hh, mw, (out_dev_ref ? out->route_option : wb.r_ro) + dst);
        }
        if (host_out) {
          copy_rows_back(ctx, out->deliver, wb.r_dl, nc, m * Hh, mw * Hh, w0 * Hh);
          copy_rows_back(ctx, out->quantity, wb.r_q, nc, m * Hh * 4, mw * Hh * 4, w0 * Hh * 4);
          copy_rows_back(ctx, out->end_inventory, wb.r_ei, nc, m * Hh * 4, mw * Hh * 4, w0 * Hh * 4);
          copy_rows_back(ctx, out->route_option, wb.r_ro, nc, m * Hh * 4, mw * Hh * 4, w0 * Hh * 4);
        }
      }
      w0 += mw;
    }

    ctx->allreduce_agg(d_agg, static_cast<uint64_t>(nc) * kAggWords);
    if (host_out && out->totals && zc_totals) ctx->stats.d2h_bytes += nc * m * 8;  // stored by the kernels
    const bool want_agg = out->agg || out->agg_raw;
    scendp_agg_raw* h_raw = nullptr;
    if (want_agg) {
      h_raw = static_cast<scendp_agg_raw*>(ctx->pinned_agg(nc * sizeof(scendp_agg_raw)));
      ctx->agg_readback(h_raw, d_agg, nc * sizeof(scendp_agg_raw));
    }
    if (!(flags & SCENDP_ASYNC) || host_out || want_agg) ctx->sync();
    if (want_agg) {
      if (out->agg_raw) std::memcpy(out->agg_raw, h_raw, nc * sizeof(scendp_agg_raw));
      if (out->agg) finalize_agg(h_raw, 1, nc, out->agg);
    }
  });
}

extern "C" scendp_status scendp_dsirp_footprint(scendp_ctx* ctx, const scendp_customer* customers,
                                                uint32_t n_customers, const scendp_scenarios* sc,
                                                uint32_t flags, const scendp_dsirp_out* out,
                                                scendp_footprint* fp) {
  return guard([&] {
    if (!ctx || !customers || !n_customers || !sc || !out || !fp)
      fail(SCENDP_ERR_INVALID_ARGUMENT, "null argument");
    CUDA_CHECK(cudaSetDevice(ctx->device));
    const int H = customers[0].horizon;
    // customer tables without deduplication (an upper bound of the cached
    // record | pool | ipool block)
    uint64_t tb = 0;
    for (uint32_t c = 0; c < n_customers; ++c) {
      const scendp_customer& s = customers[c];
      const uint64_t U1 = static_cast<uint64_t>(s.capacity) + 1, Hh = static_cast<uint64_t>(H);
      tb += sizeof(CustDev) + 8 * (2 * Hh * s.options + Hh * U1 + (s.delivery_tabular ? Hh * U1 : 0) +
                                   (s.holding_tabular ? U1 : 0)) +
            4 * (Hh * U1 + (s.holding_tabular ? U1 : 0)) + 48;
    }
    const DsirpFootprint f = dsirp_footprint(ctx, n_customers, H, sc, flags, out, tb);
    fp->fixed_bytes = f.fixed;
    fp->per_scenario_bytes = f.per_scenario;
    fp->wave = f.wave;
    fp->budget = f.budget;
  });
}
