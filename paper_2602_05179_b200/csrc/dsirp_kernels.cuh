// dsirp_kernels.cuh -- K3 device code (included by dsirp.cu inside its
// anonymous namespace).  See dsirp.cu for the formulation.
//
//  * dsirp_unit_fp64: one (customer, scenario) unit with the reference's fp64
//    arithmetic (forward_pass, oudp.cpp:40-87) on the register-resident sparse
//    frontier; shared by the fp64 kernel and, as the exact fallback, by the
//    integer kernel.
//  * dsirp_kernel: fp64 path, CTA = one customer x 128 scenarios.
//  * dsirp_int_kernel: exact scaled-integer path for dyadic cost models.
#pragma once

namespace scendp_dsirp {

using namespace scendp_dev;

constexpr double kInfD = __builtin_huge_val();
constexpr int kDsirpThreads = 128;
constexpr int kDsirpIntUnits = 4;  // 128-scenario blocks per CTA (exact-integer kernel)
constexpr int kDsirpFastMaxUnits = 32;  // 128-scenario blocks per CTA (fast form), upper bound

struct CustDev {
  int32_t U, I0, H, R;
  double h, rh;            // rh = rho * h, same rounding as the reference
  int32_t del_tab, hold_tab;
  uint64_t off_fixed, off_unit, off_dtable, off_htable;  // into the pool
  // exact integer path (int_ok): every cost scaled by 2^shift is an integer
  int32_t int_ok, shift;
  int32_t h_i, rh_i;       // scaled h and rho*h
  int32_t dlim;            // demands above this leave the exact int32 range
  uint64_t off_gkey;       // int pool: [H][U+1] packed keys (minF << 8 | r), q = 0: INT32_MIN
  uint64_t off_htab_i;     // int pool: [U+1] scaled holding table
  uint64_t off_fmin;       // pool: [H][U+1] min over r of F(t, r, q), q = 0: +inf
};

struct DsirpArgs {
  const CustDev* cust;   // [nc]
  const double* pool;
  const int32_t* ipool;  // integer tables (gkeys, scaled holding tables)
  uint32_t nc;
  int32_t H;
  int32_t all_std_hold;  // every customer uses the standard holding model
  int32_t units;         // fast form: 128-scenario blocks per CTA
  uint64_t rows;         // nc * H
  uint64_t m_wave, w_base;
  // outputs are addressed by w = w_base + wl (the host passes them at the
  // wave's offset with w_base = 0); row strides per customer:
  uint64_t tot_stride;   // totals [nc][tot_stride]
  uint64_t ev_stride;    // evaluated [nc][ev_stride]
  uint64_t sched_tiles;  // schedules [nc][sched_tiles][H][32]
  const uint32_t* tiled; // wave-local tiled demands
  GenParams gen;
  double* totals;        // or null
  uint8_t* evaluated;    // or null
  uint8_t* deliver;      // FULL tiled
  int32_t* quantity;
  int32_t* end_inventory;
  int32_t* route_option;
  unsigned long long* agg;  // [nc][16]
};

template <int K>
__device__ __forceinline__ double sel_d(const double (&a)[K], int idx) {
  double r = a[0];
#pragma unroll
  for (int e = 1; e < K; ++e) r = (e == idx) ? a[e] : r;
  return r;
}
template <int K>
__device__ __forceinline__ uint32_t sel_u(const uint32_t (&a)[K], int idx) {
  uint32_t r = a[0];
#pragma unroll
  for (int e = 1; e < K; ++e) r = (e == idx) ? a[e] : r;
  return r;
}

template <int HMAX>
__device__ __forceinline__ void dsirp_load_demands(const DsirpArgs& a, uint32_t c, uint64_t wl,
                                                   int H, int (&dem)[HMAX]) {
  const uint64_t row0 = static_cast<uint64_t>(c) * H;
  if (a.tiled) {
    const uint32_t* base = a.tiled + ((wl >> 5) * a.rows + row0) * kTile + (wl & 31);
#pragma unroll
    for (int t = 0; t < HMAX; ++t) dem[t] = t < H ? static_cast<int>(__ldg(base + t * kTile)) : 0;
  } else {
    const uint64_t stream = derive_stream(a.gen.seed, kStreamScenario, a.gen.first_index + wl);
#pragma unroll
    for (int t = 0; t < HMAX; ++t)
      dem[t] = t < H ? static_cast<int>(draw_counter(a.gen, stream, row0 + t)) : 0;
  }
}

// Schedule replay from the delivery mask (assemble_schedule, oudp.cpp:108-132).
template <int HMAX>
__device__ __forceinline__ void dsirp_write_schedule(const DsirpArgs& a, uint32_t c, uint64_t w,
                                                     int U, int I0, int H, bool ok,
                                                     uint32_t mask, const int (&opt)[HMAX],
                                                     const int (&dem)[HMAX]) {
  const uint64_t tiles = a.sched_tiles;
  const uint64_t ob = ((static_cast<uint64_t>(c) * tiles + (w >> 5)) * H) * kTile + (w & 31);
  int inv = I0;
#pragma unroll
  for (int t = 0; t < HMAX; ++t) {
    if (t < H) {
      const bool z = ok && ((mask >> t) & 1u);
      const int q = z ? U - inv : 0;
      const int j = max(0, inv + q - dem[t]);
      a.deliver[ob + t * kTile] = z ? 1 : 0;
      a.quantity[ob + t * kTile] = ok ? q : 0;
      a.end_inventory[ob + t * kTile] = ok ? j : 0;
      a.route_option[ob + t * kTile] = z ? opt[t] : 0;
      inv = j;
    }
  }
}

// One unit, fp64, reference arithmetic.  fixed/unit point to [H][R] arrays
// (shared or global memory).  Writes totals/evaluated/schedule; returns the
// total (+inf and ok = false for the all-infinite logic_error slot).
template <int HMAX, bool FULL>
__device__ __forceinline__ double dsirp_unit_fp64(const DsirpArgs& a, const CustDev& cd,
                                                  const double* fixed, const double* unit,
                                                  uint32_t c, uint64_t w, const int (&dem)[HMAX],
                                                  bool& ok) {
  constexpr int K = HMAX + 1;
  // slot loops with a constant trip count (guarded by e <= t) unroll fully,
  // keeping the slot arrays in registers; long horizons keep t+1 trips
  constexpr bool kSlotsExact = HMAX <= 8;
  constexpr int kUnr = HMAX <= 16 ? HMAX + 1 : 1;  // long horizons: rolled loops
  const int U = cd.U, H = cd.H, R = cd.R;
  const double h = cd.h, rh = cd.rh;
  const double* dtable = a.pool + cd.off_dtable;  // [H][U+1]
  const double* htable = a.pool + cd.off_htable;  // [U+1]
  const bool dtab = cd.del_tab != 0, htab = cd.hold_tab != 0;
  // HoldingPenaltyModel::cost (oudp.hpp:58-62): h*J + (rho*h)*s, or table[J]
  auto hold = [&](int j, int s) -> double {
    if (htab) return __ldg(htable + j);
    return __dadd_rn(__dmul_rn(h, static_cast<double>(j)), __dmul_rn(rh, static_cast<double>(s)));
  };
  int st[K];
  double vl[K];
  uint32_t dm[K];  // FULL: delivery-day bitmask per slot
  int opt[HMAX];   // FULL: route option of the day's delivery target
#pragma unroll
  for (int e = 0; e < K; ++e) {
    st[e] = 0;
    vl[e] = kInfD;
    dm[e] = 0u;
  }
#pragma unroll
  for (int t = 0; t < HMAX; ++t) opt[t] = 0;
  st[0] = cd.I0;
  vl[0] = 0.0;
  uint64_t live = 1ull;

#pragma unroll kUnr
  for (int t = 0; t < HMAX; ++t) {
    if (t < H) {
      const int d = dem[t];
      const int j1 = max(0, U - d), s1 = max(0, d - U);
      const double hold1 = hold(j1, s1);
      // (1) delivery: first minimum over (r, state) of a[i] + (F + hold1)
      double bv = kInfD;
      int br = 0, be = -1;
      for (int r = 0; r < R; ++r) {
        const double fx = dtab ? 0.0 : fixed[t * R + r];
        const double un = dtab ? 0.0 : unit[t * R + r];
#pragma unroll kUnr
        for (int e = 0; e < (kSlotsExact ? K : t + 1); ++e) if (e <= t) {
          if (((live >> e) & 1ull) && st[e] < U) {
            const int q = U - st[e];
            const double F = dtab ? __ldg(dtable + t * (U + 1) + q)
                                  : __dadd_rn(fx, __dmul_rn(un, static_cast<double>(q)));
            const double cand = __dadd_rn(vl[e], __dadd_rn(F, hold1));
            if (cand < bv) {
              bv = cand;
              br = r;
              be = e;
            }
          }
        }
      }
      // (2) no delivery, in place; states <= d collapse onto 0 keeping the
      // first strict minimum
      double b0 = kInfD;
      int k0 = -1, tgt = -1;
#pragma unroll kUnr
      for (int e = 0; e < (kSlotsExact ? K : t + 1); ++e) if (e <= t) {
        if ((live >> e) & 1ull) {
          const int i = st[e];
          const int j = max(0, i - d), s = max(0, d - i);
          const double nv = __dadd_rn(vl[e], hold(j, s));
          if (i == U && j1 > 0) tgt = e;
          st[e] = j;
          vl[e] = nv;
          if (i <= d) {
            if (nv < b0) {
              if (k0 >= 0) live &= ~(1ull << k0);
              b0 = nv;
              k0 = e;
            } else {
              live &= ~(1ull << e);
            }
          } else if (!(nv < kInfD)) {
            live &= ~(1ull << e);
          }
        }
      }
      if (j1 == 0) tgt = k0;
      // (3) merge the delivery candidate into state j1 (strict <)
      if (be >= 0) {
        const uint32_t nm = FULL ? (sel_u<K>(dm, be) | (1u << t)) : 0u;
        if (tgt >= 0) {
          const double tv = ((live >> tgt) & 1ull) ? sel_d<K>(vl, tgt) : kInfD;
          if (bv < tv) {
#pragma unroll kUnr
            for (int e = 0; e < (kSlotsExact ? K : t + 1); ++e) if (e <= t) {
              // per-slot selects (not `vl[tgt] = bv`): a dynamic index
              // would move the slot arrays to local memory
              const bool hit = e == tgt;
              vl[e] = hit ? bv : vl[e];
              if (FULL) dm[e] = hit ? nm : dm[e];
            }
            live |= 1ull << tgt;
            if (FULL) opt[t] = br;
          }
        } else {
          st[t + 1] = j1;
          vl[t + 1] = bv;
          live |= 1ull << (t + 1);
          if (FULL) {
            dm[t + 1] = nm;
            opt[t] = br;
          }
        }
      }
    }
  }
  // pick_terminal: smallest state with the minimal value
  double total = kInfD;
  int ts = -1;
#pragma unroll
  for (int e = 0; e < K; ++e) {
    if (((live >> e) & 1ull) && vl[e] < total) {
      total = vl[e];
      ts = e;
    }
  }
  ok = ts >= 0;
  if (!ok) total = kInfD;  // logic_error slot: evaluated = 0
  if (a.totals) a.totals[static_cast<uint64_t>(c) * a.tot_stride + w] = total;
  if (a.evaluated) a.evaluated[static_cast<uint64_t>(c) * a.ev_stride + w] = ok ? 1 : 0;
  if (FULL) dsirp_write_schedule<HMAX>(a, c, w, U, cd.I0, H, ok, ok ? sel_u<K>(dm, ts) : 0u, opt, dem);
  return total;
}

template <int HMAX, bool FULL>
__global__ void __launch_bounds__(kDsirpThreads)
dsirp_kernel(DsirpArgs a) {
  extern __shared__ __align__(16) double s_fu[];  // fixed [H][R], unit [H][R]
  __shared__ unsigned long long s_agg[kAggSlots];
  const uint32_t c = blockIdx.y;
  const CustDev cd = a.cust[c];
  const int HR = cd.H * cd.R;
  double* s_fixed = s_fu;
  double* s_unit = s_fu + HR;
  if (!cd.del_tab) {
    for (int x = threadIdx.x; x < HR; x += blockDim.x) {
      s_fixed[x] = a.pool[cd.off_fixed + x];
      s_unit[x] = a.pool[cd.off_unit + x];
    }
  }
  agg_cta_init(s_agg);
  __syncthreads();
  const uint64_t wl = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const bool active = wl < a.m_wave;
  double total = kInfD;
  bool ok = false;
  if (active) {
    int dem[HMAX];
    dsirp_load_demands<HMAX>(a, c, wl, cd.H, dem);
    total = dsirp_unit_fp64<HMAX, FULL>(a, cd, s_fixed, s_unit, c, a.w_base + wl, dem, ok);
  }
  __syncwarp();
  agg_warp_add(s_agg, agg_pieces(total, ok), active);
  __syncthreads();
  agg_cta_flush(s_agg, a.agg + static_cast<uint64_t>(c) * kAggWords);
}

// ---------------------------------------------------------------------------
// Exact scaled-integer path.  When every cost parameter of a customer is a
// multiple of 2^-shift (dyadic, e.g. the 1/4 steps of the BASELINE pins) and
// every path cost stays below 2^22 after scaling, each fp64 operation of the
// reference (fixed + unit*q, h*J + (rho h)*s, the sums) is exact, so scaled
// int32 arithmetic reproduces its doubles bit for bit.  Exactness also makes
// the route-option scan separable: for a fixed state the reference's first
// minimum over r is the smallest r with minimal F(t, r, q), independent of
// the frontier value, so the host precomputes per (day, quantity) the key
// (min_r F << 8) | argmin_r, and the per-slot delivery candidate becomes one
// table lookup + add: key = gkey[t][U-i] + ((a[i] + hold1) << 8).  Comparing
// packed keys with strict < over states in ascending order yields the
// reference's (value, option, state) order.  A demand above `dlim` (bounds)
// sends the unit through dsirp_unit_fp64 instead (global parameters).
// STDHOLD: every customer of the launch uses the standard holding model
// h*J + rho*h*s (no per-evaluation table test).
template <int HMAX, bool FULL, bool STDHOLD = false>
__global__ void __launch_bounds__(kDsirpThreads, HMAX <= 8 ? 8 : 1)  // 8 CTAs/SM: -7 % at C3/C4
dsirp_int_kernel(DsirpArgs a) {
  constexpr int K = HMAX + 1;
  // slot loops with a constant trip count (guarded by e <= t) unroll fully,
  // keeping the slot arrays in registers; long horizons keep t+1 trips
  constexpr bool kSlotsExact = HMAX <= 8;
  constexpr int kUnr = HMAX <= 16 ? HMAX + 1 : 1;  // long horizons: rolled loops
  // horizons <= 8 are launched with HMAX == H exactly (launch_exact): every
  // day/slot loop is then fully unrolled with compile-time bounds, so the
  // frontier arrays stay in registers
  constexpr bool kExact = HMAX <= 8;
  using Mask = typename std::conditional<(K <= 32), uint32_t, uint64_t>::type;
  __shared__ unsigned long long s_agg[kAggSlots];
  const uint32_t c = blockIdx.y;
  const CustDev cd = a.cust[c];
  agg_cta_init(s_agg);
  __syncthreads();
  const int U = cd.U, H = kExact ? HMAX : cd.H;
  const int32_t* gkey = a.ipool + cd.off_gkey;     // [H][U+1]
  const int32_t* htab = a.ipool + cd.off_htab_i;   // [U+1]
  const bool htabular = cd.hold_tab != 0;
  const int32_t hI = cd.h_i, rhI = cd.rh_i;
  const double inv_scale = __longlong_as_double(static_cast<long long>(1023 - cd.shift) << 52);
  // kDsirpIntUnits consecutive 128-scenario blocks per CTA: one customer
  // record, aggregate init and flush per CTA instead of per block (the unit
  // itself is short; the prologue/epilogue barriers were a visible stall)
  for (int rep = 0; rep < kDsirpIntUnits; ++rep) {
    const uint64_t wl = (blockIdx.x * static_cast<uint64_t>(kDsirpIntUnits) + rep) * blockDim.x +
                        threadIdx.x;
    const bool active = wl < a.m_wave;
    const uint64_t w = a.w_base + wl;

    double total = kInfD;
    bool ok = false;
    if (active) {
      int dem[HMAX];
      dsirp_load_demands<HMAX>(a, c, wl, H, dem);
      bool in_range = true;
  #pragma unroll
      for (int t = 0; t < HMAX; ++t)
        if (t < H) in_range &= static_cast<unsigned>(dem[t]) <= static_cast<unsigned>(cd.dlim);
      if (!in_range) {
        total = dsirp_unit_fp64<HMAX, FULL>(a, cd, a.pool + cd.off_fixed, a.pool + cd.off_unit, c,
                                            w, dem, ok);
      } else {
        auto hold = [&](int j, int s) -> int32_t {
          if (!STDHOLD && htabular) return __ldg(htab + j);
          return hI * j + rhI * s;
        };
        int st[K];
        int32_t vl[K];
        uint32_t dm[K];
        int opt[HMAX];
  #pragma unroll
        for (int e = 0; e < K; ++e) {
          st[e] = 0;
          vl[e] = 0;
          dm[e] = 0u;
        }
  #pragma unroll
        for (int t = 0; t < HMAX; ++t) opt[t] = 0;
        st[0] = cd.I0;
        Mask live = 1u;  // K = HMAX+1 slots can exceed 32
  #pragma unroll kUnr
        for (int t = 0; t < HMAX; ++t) {
          if (t < H) {
            const int d = dem[t];
            const int j1 = max(0, U - d), s1 = max(0, d - U);
            const int32_t hold1 = hold(j1, s1);
            const int32_t* grow = gkey + t * (U + 1) + U;  // grow[-i] = key for q = U - i
            // (1) delivery candidate: packed (cand << 8 | r), first minimum
            int32_t bk = INT32_MAX;
            int be = -1;
  #pragma unroll kUnr
            for (int e = 0; e < (kSlotsExact ? K : t + 1); ++e) if (e <= t) {
              if (((live >> e) & 1u) && st[e] < U) {
                const int32_t key = __ldg(grow - st[e]) + ((vl[e] + hold1) << 8);
                if (key < bk) {
                  bk = key;
                  be = e;
                }
              }
            }
            // (2) no delivery
            int32_t b0 = INT32_MAX;
            int k0 = -1, tgt = -1;
  #pragma unroll kUnr
            for (int e = 0; e < (kSlotsExact ? K : t + 1); ++e) if (e <= t) {
              if ((live >> e) & 1u) {
                const int i = st[e];
                const int j = max(0, i - d), s = max(0, d - i);
                const int32_t nv = vl[e] + hold(j, s);
                if (i == U && j1 > 0) tgt = e;
                st[e] = j;
                vl[e] = nv;
                if (i <= d) {
                  if (nv < b0) {
                    if (k0 >= 0) live &= ~(Mask{1} << k0);
                    b0 = nv;
                    k0 = e;
                  } else {
                    live &= ~(Mask{1} << e);
                  }
                }
              }
            }
            if (j1 == 0) tgt = k0;
            // (3) merge (strict <)
            if (be >= 0) {
              const int32_t bv = bk >> 8;
              const int br = bk & 0xff;
              const uint32_t nm = FULL ? (sel_u<K>(dm, be) | (1u << t)) : 0u;
              if (tgt >= 0) {
                int32_t tv = INT32_MAX;
  #pragma unroll kUnr
                for (int e = 0; e < (kSlotsExact ? K : t + 1); ++e)
                  if (e == tgt && ((live >> e) & 1u)) tv = vl[e];
                if (bv < tv) {
  #pragma unroll kUnr
                  for (int e = 0; e < (kSlotsExact ? K : t + 1); ++e) if (e <= t) {
                    const bool hit = e == tgt;  // per-slot selects (see above)
                    vl[e] = hit ? bv : vl[e];
                    if (FULL) dm[e] = hit ? nm : dm[e];
                  }
                  live |= Mask{1} << tgt;
                  if (FULL) opt[t] = br;
                }
              } else {
                st[t + 1] = j1;
                vl[t + 1] = bv;
                live |= Mask{1} << (t + 1);
                if (FULL) {
                  dm[t + 1] = nm;
                  opt[t] = br;
                }
              }
            }
          }
        }
        int32_t tv = INT32_MAX;
        int ts = -1;
  #pragma unroll
        for (int e = 0; e < K; ++e) {
          if (((live >> e) & 1u) && vl[e] < tv) {
            tv = vl[e];
            ts = e;
          }
        }
        ok = ts >= 0;  // always: the no-delivery chain keeps a state alive
        total = ok ? static_cast<double>(tv) * inv_scale : kInfD;
        if (a.totals) a.totals[static_cast<uint64_t>(c) * a.tot_stride + w] = total;
        if (a.evaluated) a.evaluated[static_cast<uint64_t>(c) * a.ev_stride + w] = ok ? 1 : 0;
        if (FULL) dsirp_write_schedule<HMAX>(a, c, w, U, cd.I0, H, ok, ok ? sel_u<K>(dm, ts) : 0u, opt, dem);
      }
    }
    __syncwarp();
    agg_warp_add(s_agg, agg_pieces(total, ok), active);
  }
  __syncthreads();
  agg_cta_flush(s_agg, a.agg + static_cast<uint64_t>(c) * kAggWords);
}

// ---------------------------------------------------------------------------
// K3 fast form (horizons 1..8, launched with HMAX == H): the frontier without
// liveness bookkeeping.  Slot e (created at the end of day e-1; slot 0 holds
// I0) keeps one (state, value) pair; every slot is updated every day, so the
// per-slot work is a fixed, branch-free sequence and all 32 lanes stay busy.
//
// Why no slot ever needs to be removed: states are non-decreasing in slot
// order (a day maps i -> max(0, i-d) monotonically and appends the largest
// state max(0, U-d)), and two slots reach the same state only by a merge at 0
// or when the appended state equals a shifted one.  The reference keeps, per
// state, the first strict minimum over its candidates in ascending predecessor
// order, no-delivery before delivery (oudp.cpp:56-84).  Here the same
// candidates sit in adjacent slots in exactly that order and identical states
// receive identical increments afterwards, so "first minimum in slot order"
// selects the reference's value (and, FULL, its backpointer path) wherever the
// frontier is read: the delivery argmin, the terminal pick (oudp.cpp:94-106).
// A slot the reference would have merged away only ever holds a larger or
// equal value at an equal state, later in slot order.
//
// Per slot and day: delivery candidate = table[t][U - state] + value (one
// shared-memory lookup; the route-option minimum is folded into the table on
// the host), then the no-delivery shift.
//  * INT (exact scaled-integer customers, see dsirp_int_kernel): the table
//    holds (min_r F << 8 | argmin_r), so the packed key orders (value, option)
//    and the cost-only minimum is one unsigned min; state U (no delivery
//    possible) holds 0x80000000, a key no real candidate reaches.  A day
//    without any delivery candidate, or a demand above dlim, sends the unit
//    to dsirp_unit_fp64 (the reference's arithmetic), which also serves FULL.
//  * fp64 (cost-only): table = min over r of the reference's rounded
//    F(t, r, q) (+inf at q = 0).  Rounding is monotone, so
//    min_r (v + (F_r + hold1)) = v + (min_r F_r + hold1) bit for bit; the
//    hold term of the no-delivery step, h*J + (rho h)*s, is h*x for x = i-d
//    >= 0 and (rho h)*(-x) otherwise (the other product is +0).
template <int H, bool INT, bool FULL, bool STDHOLD, bool STAB>
// register caps: exact-integer 40 (12 CTAs/SM), fp64 48 (10 CTAs/SM), no
// spills (measured: C4 2.74 -> 2.46 ms against the uncapped 64 registers)
__global__ void __launch_bounds__(kDsirpThreads, INT ? 12 : 10)
dsirp_fast_kernel(DsirpArgs a) {
  static_assert(INT || !FULL, "fp64 schedules run dsirp_kernel");
  using VT = typename std::conditional<INT, int32_t, double>::type;
  constexpr int K = H + 1;
  extern __shared__ __align__(16) char s_dyn[];
  __shared__ unsigned long long s_agg[kAggSlots];
  const uint32_t c = blockIdx.y;
  const CustDev cd = a.cust[c];
  const int U = cd.U, U1 = cd.U + 1;
  const VT* g_del = INT ? reinterpret_cast<const VT*>(a.ipool + cd.off_gkey)
                        : reinterpret_cast<const VT*>(a.pool + cd.off_fmin);
  const VT* g_hold = INT ? reinterpret_cast<const VT*>(a.ipool + cd.off_htab_i)
                         : reinterpret_cast<const VT*>(a.pool + cd.off_htable);
  const VT* t_del = g_del;
  const VT* t_hold = g_hold;
  if constexpr (STAB) {
    VT* s_del = reinterpret_cast<VT*>(s_dyn);
    VT* s_hold = s_del + H * U1;
    for (int x = threadIdx.x; x < H * U1; x += kDsirpThreads) s_del[x] = g_del[x];
    if (!STDHOLD && cd.hold_tab)
      for (int x = threadIdx.x; x < U1; x += kDsirpThreads) s_hold[x] = g_hold[x];
    t_del = s_del;
    t_hold = s_hold;
  }
  agg_cta_init(s_agg);
  __syncthreads();
  const int32_t nrhI = -cd.rh_i, hrI = cd.h_i + cd.rh_i;
  const double h = cd.h, rh = cd.rh;
  const double inv_scale = __longlong_as_double(static_cast<long long>(1023 - cd.shift) << 52);
  // hold(J = j, s = j - x); !STDHOLD: the launch has tabular customers
  const bool htabular = !STDHOLD && cd.hold_tab != 0;
  auto hold_of = [&](int x, int j) -> VT {
    if (htabular) return t_hold[j];
    if constexpr (INT) return hrI * j + nrhI * x;
    // h*j + (rho h)*s with s = j - x: one of j, s is 0, so the FMA adds an
    // exact +0 to (or scales +0 into) the single rounded product -- the same
    // bits as __dmul_rn(x >= 0 ? h : rh, |x|), without the ALU selects
    else return __fma_rn(h, static_cast<double>(j), __dmul_rn(rh, static_cast<double>(j - x)));
  };
  // aggregates: INT sums the scaled integer totals per thread (one exact
  // add per CTA and warp at the end); fp64 keeps a per-warp register
  // accumulator.  Units run by dsirp_unit_fp64 go through agg_warp_add.
  uint32_t isum = 0u, icnt = 0u;  // < 32 units x 2^22 per thread
  unsigned long long wacc = 0ull;
  const int units = a.units;
  for (int rep = 0; rep < units; ++rep) {
    const uint64_t wl = (blockIdx.x * static_cast<uint64_t>(units) + rep) * kDsirpThreads +
                        threadIdx.x;
    const bool active = wl < a.m_wave;
    const uint64_t w = a.w_base + wl;
    double total = kInfD;
    bool ok = false;
    bool fb = false;  // run the reference-arithmetic unit instead
    if (active) {
      int dem[H];
      dsirp_load_demands<H>(a, c, wl, H, dem);
      if constexpr (INT) {
        uint32_t dmax = 0;
#pragma unroll
        for (int t = 0; t < H; ++t) dmax = max(dmax, static_cast<uint32_t>(dem[t]));
        fb = dmax > static_cast<uint32_t>(cd.dlim);
      }
      if (!fb) {
        int st[K];
        VT vl[K];
        uint32_t dm[K];
        int opt[H];
#pragma unroll
        for (int e = 0; e < K; ++e) {
          st[e] = 0;
          vl[e] = VT(0);
          dm[e] = 0u;
        }
#pragma unroll
        for (int t = 0; t < H; ++t) opt[t] = 0;
        st[0] = cd.I0;
        uint32_t flag = 0u;
#pragma unroll
        for (int t = 0; t < H; ++t) {
          const int d = dem[t];
          const int j1 = max(0, U - d);
          const VT hold1 = hold_of(U - d, j1);
          const VT* row = t_del + t * U1 + U;  // row[-i]: quantity U - i
          // (1) delivery: first minimum over (value, option, slot)
          uint32_t bk = 0xffffffffu;
          int be = 0;
          double bv = kInfD;
#pragma unroll
          for (int e = 0; e < K; ++e) {
            if (e <= t) {
              const VT g = row[-st[e]];
              if constexpr (INT) {
                const uint32_t key = static_cast<uint32_t>(g) + (static_cast<uint32_t>(vl[e]) << 8);
                if constexpr (FULL) {
                  if (key < bk) {
                    bk = key;
                    be = e;
                  }
                } else {
                  bk = min(bk, key);
                }
              } else {
                const double cand = __dadd_rn(vl[e], __dadd_rn(g, hold1));
                bv = cand < bv ? cand : bv;
              }
            }
          }
          // (2) no delivery: every slot shifts by d
#pragma unroll
          for (int e = 0; e < K; ++e) {
            if (e <= t) {
              const int x = st[e] - d;
              const int j = max(x, 0);
              if constexpr (INT) vl[e] += hold_of(x, j);
              else vl[e] = __dadd_rn(vl[e], hold_of(x, j));
              st[e] = j;
            }
          }
          // (3) the delivery target: a new slot with the largest state
          st[t + 1] = j1;
          if constexpr (INT) {
            flag |= bk;
            vl[t + 1] = static_cast<int32_t>(bk >> 8) + hold1;
            if constexpr (FULL) {
              dm[t + 1] = sel_u<K>(dm, be) | (1u << t);
              opt[t] = static_cast<int>(bk & 0xffu);
            }
          } else {
            vl[t + 1] = bv;
          }
        }
        if (INT && (flag & 0x80000000u)) {
          fb = true;  // some day offered no delivery candidate at all
        } else {
          // pick_terminal: first minimum in slot (= state) order
          VT tv = vl[0];
          int ts = 0;
#pragma unroll
          for (int e = 1; e < K; ++e) {
            if constexpr (FULL) {
              if (vl[e] < tv) {
                tv = vl[e];
                ts = e;
              }
            } else {
              tv = vl[e] < tv ? vl[e] : tv;
            }
          }
          if constexpr (INT) {
            ok = true;
            total = static_cast<double>(tv) * inv_scale;
            isum += static_cast<uint32_t>(tv);
            icnt += 1u;
          } else {
            ok = tv < kInfD;  // all-infinite: the reference's logic_error slot
            total = ok ? tv : kInfD;
          }
          if (a.totals) a.totals[static_cast<uint64_t>(c) * a.tot_stride + w] = total;
          if (a.evaluated) a.evaluated[static_cast<uint64_t>(c) * a.ev_stride + w] = ok ? 1 : 0;
          if constexpr (FULL)
            dsirp_write_schedule<H>(a, c, w, U, cd.I0, H, ok, sel_u<K>(dm, ts), opt, dem);
        }
      }
      if (fb)
        total = dsirp_unit_fp64<H, FULL>(a, cd, a.pool + cd.off_fixed, a.pool + cd.off_unit, c, w,
                                         dem, ok);
    }
    __syncwarp();
    if constexpr (INT) {
      if (__any_sync(0xffffffffu, fb)) agg_warp_add(s_agg, agg_pieces(total, ok), fb);
    } else {
      agg_warp_acc(wacc, s_agg, agg_pieces(total, ok), active);
    }
  }
  if constexpr (INT) {
    const uint32_t S = __reduce_add_sync(0xffffffffu, isum);  // < 32 x 32 x 2^22 = 2^32
    const uint32_t n = __reduce_add_sync(0xffffffffu, icnt);
    if ((threadIdx.x & 31) == 0) agg_cta_add_scaled(s_agg, S, cd.shift, n);
  } else {
    agg_warp_acc_flush(wacc, s_agg);
  }
  __syncthreads();
  agg_cta_flush(s_agg, a.agg + static_cast<uint64_t>(c) * kAggWords);
}

// Launch one HMAX instantiation (fp64 or exact-integer kernel).
template <typename Kern>
void launch_kernel(scendp_ctx* ctx, Kern kernel, const DsirpArgs& a, size_t smem, int units = 1) {
  scendp_host::cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem < 16 ? 16 : smem)),
                          "cudaFuncSetAttribute");
  const uint64_t per_cta = static_cast<uint64_t>(kDsirpThreads) * units;
  dim3 grid(static_cast<unsigned>((a.m_wave + per_cta - 1) / per_cta), a.nc);
  const int tok = ctx->timing_begin(0);
  kernel<<<grid, kDsirpThreads, smem, ctx->stream>>>(a);
  scendp_host::cuda_check(cudaGetLastError(), "dsirp kernel launch");
  ctx->timing_end(tok);
  ctx->count_launch();
}

template <int HMAX>
void launch_h(scendp_ctx* ctx, const DsirpArgs& a, size_t smem, bool int_path, bool full);

// Horizons 1..8: instantiations with HMAX == H (dsirp_exact.cu).
void launch_exact(scendp_ctx* ctx, const DsirpArgs& a, size_t smem, bool int_path, bool full);

// Fast form for horizons 1..8 (dsirp_fast_a.cu / dsirp_fast_b.cu): INT with
// or without schedules, fp64 cost-only.  smem = the customer tables.
template <int H>
void launch_fast_h(scendp_ctx* ctx, const DsirpArgs& a_in, size_t smem, bool int_path, bool full) {
  // blocks per CTA: as many as keep >= 2.5 waves of CTAs (the customer
  // table load and the aggregate flush are per CTA; measured C4 2.46 ->
  // 2.16 ms with 32, C3 best with 8)
  DsirpArgs a = a_in;
  const uint64_t slots = static_cast<uint64_t>(ctx->sm_count) * (int_path ? 12 : 10);
  int units = kDsirpFastMaxUnits;
  while (units > 1 && 2 * a.nc * ((a.m_wave + 128ull * units - 1) / (128ull * units)) < 5 * slots)
    units /= 2;
  a.units = units;
  auto go = [&](auto kernel) { launch_kernel(ctx, kernel, a, smem, units); };
  if (int_path) {
    if (a.all_std_hold) {
      if (full) go(dsirp_fast_kernel<H, true, true, true, true>);
      else go(dsirp_fast_kernel<H, true, false, true, true>);
    } else {
      if (full) go(dsirp_fast_kernel<H, true, true, false, true>);
      else go(dsirp_fast_kernel<H, true, false, false, true>);
    }
  } else {
    if (a.all_std_hold) go(dsirp_fast_kernel<H, false, false, true, true>);
    else go(dsirp_fast_kernel<H, false, false, false, true>);
  }
}
bool launch_fast(scendp_ctx* ctx, const DsirpArgs& a, size_t smem, bool int_path, bool full);

template <int HMAX>
void launch_h(scendp_ctx* ctx, const DsirpArgs& a, size_t smem, bool int_path, bool full) {
  if (int_path) {
    if (a.all_std_hold) {
      if (full) launch_kernel(ctx, dsirp_int_kernel<HMAX, true, true>, a, 0, kDsirpIntUnits);
      else launch_kernel(ctx, dsirp_int_kernel<HMAX, false, true>, a, 0, kDsirpIntUnits);
    } else {
      if (full) launch_kernel(ctx, dsirp_int_kernel<HMAX, true>, a, 0, kDsirpIntUnits);
      else launch_kernel(ctx, dsirp_int_kernel<HMAX, false>, a, 0, kDsirpIntUnits);
    }
  } else {
    if (full) launch_kernel(ctx, dsirp_kernel<HMAX, true>, a, smem);
    else launch_kernel(ctx, dsirp_kernel<HMAX, false>, a, smem);
  }
}

// Horizons above 32: the reference's dense forward pass (dsirp_long.cu).
void launch_long(scendp_ctx* ctx, const DsirpArgs& a, bool full, int max_u, int H);

// One translation unit per horizon bound (parallel builds).
void launch_h16(scendp_ctx*, const DsirpArgs&, size_t, bool, bool);  // dsirp_h16.cu
void launch_h32(scendp_ctx*, const DsirpArgs&, size_t, bool, bool);  // dsirp_h32.cu

}  // namespace scendp_dsirp
