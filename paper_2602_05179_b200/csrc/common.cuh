// common.cuh -- shared device-side building blocks of the B200 engine.
//
//  * tiled scenario layout   [w/32][row][w%32]: a warp of 32 consecutive
//    scenarios reads one 128-byte line per row, for any tour order;
//  * counter-based SplitMix64 (scenario.hpp:12-57): row r of column w is
//    mix64(s_w + r*gamma), s_w = derive_stream(seed, kStreamScenario, w);
//  * exact fixed-point aggregate (scendp_cuda.h "aggregates"): order- and
//    shard-invariant sums of finite costs.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "scendp_cuda.h"

namespace scendp_dev {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kStreamScenario = 0x5343454eULL;  // scenario.hpp:49
constexpr int kTile = 32;                            // scenarios per tile
constexpr int kAggWords = 16;                        // scendp_agg_raw / u64
constexpr int kAggSlots = 17;  // 13 digits (12 + always-zero guard) + 4 counts
constexpr int kDigitFinite = 13, kDigitInfeasible = 14, kDigitError = 15,
              kDigitRange = 16;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += kGamma;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t derive_stream(uint64_t seed,
                                                           uint64_t tag,
                                                           uint64_t index) {
  return mix64(mix64(mix64(seed) ^ tag) ^ index);
}

// Element index of (scenario w, row r) in the tiled layout.
__host__ __device__ __forceinline__ uint64_t tiled_index(uint64_t w, uint64_t r,
                                                         uint64_t rows) {
  return ((w >> 5) * rows + r) * kTile + (w & 31);
}

// Generator parameters shared by the fused (in-DP) and materializing paths.
struct GenParams {
  int32_t kind;        // SCENDP_DIST_*
  int64_t lo;
  uint64_t span;       // uniform: hi - lo + 1
  uint32_t span32;     // span when it is < 2^32 (the common case), else 0
  const double* cdf;   // poisson: P[0..cdf_len-1], device
  int32_t cdf_len;
  const int32_t* guide;  // poisson: guide[j] = min{k : cdf[k] >= j/64}, j = 0..64
  uint64_t seed;
  uint64_t first_index;
};

// next_below(span) = (x * span) >> 64 (scenario.hpp:33-37).  For span < 2^32
// the 128-bit product's high word is (x_hi*span + (x_lo*span >> 32)) >> 32:
// two 32x32->64 multiplies instead of a full 64x64 high multiply (exact: the
// dropped low 32 bits of x_lo*span cannot carry into bit 64).
__device__ __forceinline__ uint32_t uniform_draw(const GenParams& g, uint64_t x) {
  if (g.span32) {
    const uint64_t lo = static_cast<uint64_t>(static_cast<uint32_t>(x)) * g.span32;
    const uint64_t hi = static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * g.span32 + (lo >> 32);
    return static_cast<uint32_t>(g.lo) + static_cast<uint32_t>(hi >> 32);
  }
  return static_cast<uint32_t>(g.lo + static_cast<int64_t>(__umul64hi(x, g.span)));
}

// The value of one next() output x (uniform or poisson).
__device__ __forceinline__ uint32_t draw_value(const GenParams& g, uint64_t x);

// uniform_draw for a launch known to have span < 2^32 (no tests).
__device__ __forceinline__ uint32_t uniform_draw32(const GenParams& g, uint64_t x) {
  const uint64_t lo = static_cast<uint64_t>(static_cast<uint32_t>(x)) * g.span32;
  const uint64_t hi = static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * g.span32 + (lo >> 32);
  return static_cast<uint32_t>(g.lo) + static_cast<uint32_t>(hi >> 32);
}

// uniform_draw32(g, mix64(z)) with the low word of mix64's result computed
// only when it can matter.  The draw is (x_hi*span + c) >> 32 with the carry
// term c = (x_lo*span) >> 32 < span, so it differs from (x_hi*span) >> 32
// only when the low word of x_hi*span is >= 2^32 - span + 1 (probability
// ~span / 2^32 per draw: a branch that is almost never taken).  x_hi needs
// only the high word of z (x = z ^ (z >> 31)); the low word costs the
// shift/xor pair and a wide multiply it no longer always pays.  Same result
// as uniform_draw32(g, mix64(z)) for every z.
__device__ __forceinline__ uint32_t mix_uniform32(const GenParams& g, uint64_t z) {
  z += kGamma;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  const uint32_t zh = static_cast<uint32_t>(z >> 32), zl = static_cast<uint32_t>(z);
  const uint32_t xh = zh ^ (zh >> 31);
  const uint64_t q = static_cast<uint64_t>(xh) * g.span32;
  uint32_t r = static_cast<uint32_t>(q >> 32);
  const uint32_t ql = static_cast<uint32_t>(q);
  if (ql > 0xffffffffu - g.span32 + 1u) {
    const uint32_t xl = zl ^ ((zl >> 31) | (zh << 1));
    const uint32_t c = static_cast<uint32_t>((static_cast<uint64_t>(xl) * g.span32) >> 32);
    r += (static_cast<uint64_t>(ql) + c) >> 32 ? 1u : 0u;
  }
  return static_cast<uint32_t>(g.lo) + r;
}

// One counter-based draw: DistributionSpec::sample for the kinds that use
// exactly one next() per value (scenario.cpp:23-26; poisson: SURVEY App. A).
__device__ __forceinline__ uint32_t draw_counter(const GenParams& g,
                                                 uint64_t stream, uint64_t row) {
  return draw_value(g, mix64(stream + row * kGamma));
}

__device__ __forceinline__ uint32_t draw_value(const GenParams& g, uint64_t x) {
  if (g.kind == SCENDP_DIST_UNIFORM) return uniform_draw(g, x);
  // next_unit: ((x >> 11) + 1) * 2^-53, exact in fp64
  const double u = static_cast<double>((x >> 11) + 1) * 0x1.0p-53;
  // the answer min{k : u <= cdf[k]} is >= guide[floor(64 u)] (cdf[k] >= u
  // >= floor(64 u) / 64; both sides exact), so the scan starts there
  int32_t k = __ldg(g.guide + static_cast<int>(u * 64.0));
  while (u > __ldg(g.cdf + k)) ++k;  // cdf[len-1] == 1.0 terminates
  return static_cast<uint32_t>(k);
}

// ---------------------------------------------------------------------------
// Exact aggregate.  A finite cost v >= 0 is v = M * 2^E (M < 2^53); it adds
// M << (E + 192) into a 384-bit integer held as 32-bit digits d[0..11] (one
// u64 word each, weight 2^(32j-192)).  Bits below 2^-192 are truncated
// (deterministically); v >= 2^192 counts as a range error.
struct AggPieces {
  uint32_t p0, p1, p2;
  int32_t li;       // digit index of p0
  int32_t kind;     // 0 finite, 1 infeasible(+inf), 2 error, 3 range, 4 none
};

__device__ __forceinline__ AggPieces agg_pieces(double v, bool evaluated) {
  AggPieces a{0u, 0u, 0u, 0, 4};
  if (!evaluated) { a.kind = 2; return a; }
  if (!(v < __longlong_as_double(0x7ff0000000000000LL))) { a.kind = 1; return a; }
  const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v));
  const int be = static_cast<int>((bits >> 52) & 0x7ff);
  uint64_t M = bits & ((1ULL << 52) - 1);
  int E;
  if (be == 0) { E = -1074; } else { M |= (1ULL << 52); E = be - 1075; }
  int pos = E + 192;
  if (pos + 53 > 384) { a.kind = 3; return a; }
  if (pos < 0) {
    M = (-pos >= 64) ? 0ULL : (M >> (-pos));
    pos = 0;
  }
  const int sub = pos & 31;
  const uint32_t lo = static_cast<uint32_t>(M);
  const uint32_t hi = static_cast<uint32_t>(M >> 32);
  a.li = pos >> 5;
  a.p0 = lo << sub;
  a.p1 = __funnelshift_l(lo, hi, sub);
  a.p2 = sub ? (hi >> (32 - sub)) : 0u;
  a.kind = 0;
  return a;
}

// Warp-cooperative accumulation into a CTA accumulator in shared memory
// (kAggSlots u64).  Must be called by all 32 lanes of the warp, converged;
// lanes without a value pass valid = false.
__device__ __forceinline__ void agg_warp_add(unsigned long long* cta_acc,
                                             AggPieces a, bool valid) {
  const unsigned full = 0xffffffffu;
  if (!valid) a.kind = 4;
  const int lane = threadIdx.x & 31;
  const unsigned fin = __ballot_sync(full, a.kind == 0);
  const unsigned inf = __ballot_sync(full, a.kind == 1);
  const unsigned err = __ballot_sync(full, a.kind == 2);
  const unsigned rng = __ballot_sync(full, a.kind == 3);
  const int leader = __ffs(full) - 1;
  if (lane == leader) {
    if (fin) atomicAdd(cta_acc + kDigitFinite, static_cast<unsigned long long>(__popc(fin)));
    if (inf) atomicAdd(cta_acc + kDigitInfeasible, static_cast<unsigned long long>(__popc(inf)));
    if (err) atomicAdd(cta_acc + kDigitError, static_cast<unsigned long long>(__popc(err)));
    if (rng) atomicAdd(cta_acc + kDigitRange, static_cast<unsigned long long>(__popc(rng)));
  }
  if (!fin) return;
  if (a.kind == 0) {
    // lanes with the same digit index reduce together (one group in the
    // common case of costs of similar magnitude)
    const unsigned grp = __match_any_sync(fin, a.li);
    const unsigned s0l = __reduce_add_sync(grp, a.p0 & 0xffffu);
    const unsigned s0h = __reduce_add_sync(grp, a.p0 >> 16);
    const unsigned s1l = __reduce_add_sync(grp, a.p1 & 0xffffu);
    const unsigned s1h = __reduce_add_sync(grp, a.p1 >> 16);
    const unsigned s2l = __reduce_add_sync(grp, a.p2 & 0xffffu);
    const unsigned s2h = __reduce_add_sync(grp, a.p2 >> 16);
    if (lane == __ffs(grp) - 1) {
      atomicAdd(cta_acc + a.li, static_cast<unsigned long long>(s0l) +
                                    (static_cast<unsigned long long>(s0h) << 16));
      atomicAdd(cta_acc + a.li + 1, static_cast<unsigned long long>(s1l) +
                                        (static_cast<unsigned long long>(s1h) << 16));
      if (s2l | s2h)
        atomicAdd(cta_acc + a.li + 2, static_cast<unsigned long long>(s2l) +
                                          (static_cast<unsigned long long>(s2h) << 16));
    }
  }
}

// Per-warp register accumulator for kernels that add many warps of values
// per CTA: lane L (< kAggSlots) holds word L of the CTA accumulator layout.
// The common warp -- every lane finite, all digit indices equal -- costs the
// six reductions and three selects, with no atomics; anything else takes
// agg_warp_add into the shared accumulator.  Converged warp, all 32 lanes.
__device__ __forceinline__ void agg_warp_acc(unsigned long long& acc, unsigned long long* cta_acc,
                                             AggPieces a, bool valid) {
  const unsigned full = 0xffffffffu;
  if (!valid) a.kind = 4;
  int same = 0;
  __match_all_sync(full, a.kind == 0 ? a.li : -1 - a.kind, &same);
  if (!same || a.kind != 0) {
    agg_warp_add(cta_acc, a, valid);
    return;
  }
  const int lane = threadIdx.x & 31;
  const unsigned long long s0 = __reduce_add_sync(full, a.p0 & 0xffffu) +
                                (static_cast<unsigned long long>(__reduce_add_sync(full, a.p0 >> 16)) << 16);
  const unsigned long long s1 = __reduce_add_sync(full, a.p1 & 0xffffu) +
                                (static_cast<unsigned long long>(__reduce_add_sync(full, a.p1 >> 16)) << 16);
  const unsigned long long s2 = __reduce_add_sync(full, a.p2 & 0xffffu) +
                                (static_cast<unsigned long long>(__reduce_add_sync(full, a.p2 >> 16)) << 16);
  const int o = lane - a.li;
  acc += o == 0 ? s0 : o == 1 ? s1 : o == 2 ? s2 : 0ull;
  acc += lane == kDigitFinite ? 32ull : 0ull;
}

// Flush a per-warp register accumulator into the CTA accumulator.
__device__ __forceinline__ void agg_warp_acc_flush(unsigned long long acc,
                                                   unsigned long long* cta_acc) {
  const int lane = threadIdx.x & 31;
  if (lane < kAggSlots && acc) atomicAdd(cta_acc + lane, acc);
}

// Add an exact integer sum S * 2^-shift (S < 2^53, 0 <= shift <= 64) and a
// finite count into the CTA accumulator (one lane).
__device__ __forceinline__ void agg_cta_add_scaled(unsigned long long* cta_acc, uint64_t S,
                                                   int shift, uint32_t count) {
  if (count) atomicAdd(cta_acc + kDigitFinite, static_cast<unsigned long long>(count));
  if (!S) return;
  const int pos = 192 - shift;
  const int li = pos >> 5, sub = pos & 31;
  const uint32_t lo = static_cast<uint32_t>(S), hi = static_cast<uint32_t>(S >> 32);
  atomicAdd(cta_acc + li, static_cast<unsigned long long>(lo << sub));
  atomicAdd(cta_acc + li + 1, static_cast<unsigned long long>(__funnelshift_l(lo, hi, sub)));
  const uint32_t p2 = sub ? (hi >> (32 - sub)) : 0u;
  if (p2) atomicAdd(cta_acc + li + 2, static_cast<unsigned long long>(p2));
}

// CTA epilogue: add the CTA accumulator into the global raw aggregate of one
// candidate (scendp_agg_raw layout: 12 digits, finite, infeasible, error,
// range).  Integer atomics: associative, hence deterministic.
__device__ __forceinline__ void agg_cta_flush(const unsigned long long* cta_acc,
                                              unsigned long long* global_raw) {
  const int t = threadIdx.x;
  if (t < 12) {
    const unsigned long long v = cta_acc[t];
    if (v) atomicAdd(global_raw + t, v);
  } else if (t >= 13 && t < kAggSlots) {
    const unsigned long long v = cta_acc[t];
    if (v) atomicAdd(global_raw + (t - 1), v);
  }
}

// One item's aggregate straight into a global raw aggregate (kernels whose
// items of one warp may belong to different candidates).
__device__ __forceinline__ void agg_item_global(unsigned long long* g, double v, bool evaluated) {
  const AggPieces pc = agg_pieces(v, evaluated);
  if (pc.kind == 0) {
    atomicAdd(g + pc.li, static_cast<unsigned long long>(pc.p0));
    atomicAdd(g + pc.li + 1, static_cast<unsigned long long>(pc.p1));
    if (pc.p2) atomicAdd(g + pc.li + 2, static_cast<unsigned long long>(pc.p2));
    atomicAdd(g + 12, 1ULL);
  } else if (pc.kind < 4) {
    atomicAdd(g + 12 + pc.kind, 1ULL);  // infeasible, error, range
  }
}

__device__ __forceinline__ void agg_cta_init(unsigned long long* cta_acc) {
  for (int t = threadIdx.x; t < kAggSlots; t += blockDim.x) cta_acc[t] = 0ULL;
}

}  // namespace scendp_dev
