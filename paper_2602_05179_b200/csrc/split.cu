// split.cu -- K1/K2/K6: the CVRPSD split DP over scenario batches.
//
// Reference (paths under /root/reference/proj):
//   fill_prefixes         src/split.cpp:24-39   (load by customer id, dist
//                                               summed sequentially)
//   split_core_quadratic  src/split.cpp:45-75   (penalized / forced)
//   split_core_linear     src/split.cpp:77-118  (hard capacities)
//   finalize_solution     src/split.cpp:120-126
//   batched_*             src/split.cpp:303-388
//
// Execution model (B200): one thread per (tour, scenario); a CTA holds T
// scenarios of one tour.  Tour-only constants (dist prefix, depot legs,
// customer rows) are computed once on the host in the reference's order and
// staged in shared memory; demands are read from the tiled HBM layout (one
// 128-byte line per warp and tour position, any tour order) or generated in
// registers (fused).  The hard-mode deque lives in a 16-entry shared-memory
// ring per thread (occupancy <= 9 observed on every BASELINE shape); a
// scenario whose deque would overflow is re-run by the generic fallback
// kernel, which also serves very large n.
//
// Exactness: every double op is a single IEEE op in the reference's
// association (built with -fmad=false; no FMA contraction): f(p) =
// (V(p) + c(0,s_{p+1})) - dist[p+1], V(i) = (f(front) + dist[i]) + c(s_i,n+1),
// penalized cand = ((f + dist[i]) + ret) + beta*(double)excess.  Ties keep
// the earliest predecessor (strict <), as the reference.
#include <algorithm>
#include <thread>
#include <map>
#include <mutex>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <type_traits>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

using namespace scendp_dev;
using namespace scendp_host;

namespace scendp_host {
GenParams make_gen_params(scendp_ctx* ctx, const scendp_dist* d, uint64_t first_index);
template <typename T>
void launch_from_tiled(scendp_ctx* ctx, const T* src, uint64_t rows, uint64_t count, T* dst);
}  // namespace scendp_host

namespace {

constexpr int kRing = 16;  // deque ring entries per thread (power of two)
constexpr double kInfD = __builtin_huge_val();

// kSrcGenU32: generated uniform draws with span < 2^32 (the common case),
// specialized in K1 so no per-draw distribution test remains
enum Src { kSrcTiled = 0, kSrcGen = 1, kSrcGenU32 = 2 };

struct SplitArgs {
  int32_t n;
  int64_t Q;
  int32_t hard;
  int32_t linear;      // 1: deque form (hard mode), 0: quadratic form
  double beta;
  uint32_t k;          // tours
  uint64_t m_wave;     // scenarios in this launch
  uint64_t w_base;     // offset of this wave inside the call
  uint64_t m_total;    // scenarios in the call (output stride)
  // per-tour tables, [k][n+1]
  const double* dist;  // dist[i], i = 0..n (dist[0] = dist[1] = 0)
  const double* ret;   // c(s_i, n+1), i = 1..n
  const double* c0;    // c(0, s_{i+1}), i = 0..n-1
  const uint32_t* col; // s_i - 1, i = 1..n
  // K1 chunked tables, [k][npad] per row; slot s = position s+1
  int32_t npad;
  int32_t ident;         // every tour is the identity 1..n
  uint32_t pen_lmax;     // K2-int: loads above this leave the exact int32 range
  int32_t pen_bits;      // K2-bits (window bitmap): Q <= 127, demands known in [1, 31]
  int32_t pen_units;     // K2-bits: blocks of scenarios per CTA
  const uint32_t* ccol;  // customer row of position s+1
  const int32_t* itab;   // [k][2][npad]: A = dist+ret, B = c0 - dist_next (int path)
  const double* dtab;    // [k][npad][4]: dist, ret, c0, dist_next (interleaved)
  const double* f0d;     // [k] f(0) = (0.0 + c(0,s_1)) - dist[1]
  const int32_t* f0i;    // [k] same, integer path
  // scenarios
  const uint32_t* tiled;  // wave-local tiled demands (kSrcTiled)
  GenParams gen;          // kSrcGen (first_index already includes w_base)
  // outputs
  double* totals;       // [k][m_total] or null
  double* V;            // FULL, tiled [m/32][n+1][32]
  int32_t* cuts;        // FULL, tiled
  int32_t* route_count; // FULL, [m]
  uint8_t* feasible;    // FULL, [m]
  unsigned long long* agg;  // [k][16]
  // overflow list: items (k << 40 | w_wave)
  unsigned int* ovf_count;
  unsigned long long* ovf_items;
  uint32_t ovf_cap;
  uint32_t* ovf_bits;   // [k * m_wave / 32]: items beyond the list (all-zero at rest)
};

__device__ __forceinline__ uint32_t demand_at(const SplitArgs& a, int src, uint64_t stream,
                                              const uint32_t* tile_base, uint32_t row) {
  if (src == kSrcTiled) return __ldg(tile_base + static_cast<uint64_t>(row) * kTile);
  if (src == kSrcGenU32) return mix_uniform32(a.gen, stream + row * kGamma);
  return draw_counter(a.gen, stream, row);
}

// Shared memory: tour tables + per-thread rings.
struct TourSmem {
  double* dist;
  double* ret;
  double* c0;
  uint32_t* col;
};

__device__ __forceinline__ TourSmem load_tour(const SplitArgs& a, uint32_t k, char* smem) {
  const int n1 = a.n + 1;
  TourSmem t;
  t.dist = reinterpret_cast<double*>(smem);
  t.ret = t.dist + n1;
  t.c0 = t.ret + n1;
  t.col = reinterpret_cast<uint32_t*>(t.c0 + n1);
  const uint64_t off = static_cast<uint64_t>(k) * n1;
  for (int i = threadIdx.x; i < n1; i += blockDim.x) {
    t.dist[i] = a.dist[off + i];
    t.ret[i] = a.ret[off + i];
    t.c0[i] = a.c0[off + i];
    t.col[i] = a.col[off + i];
  }
  return t;
}

__host__ __device__ constexpr size_t tour_smem_bytes(int n) {
  return static_cast<size_t>(n + 1) * (3 * sizeof(double) + sizeof(uint32_t));
}

// A (tour, scenario) item for the generic kernel: into the list while it has
// room, else flagged in the bitmap (correct for any overflow count).
__device__ __forceinline__ void push_overflow(const SplitArgs& a, uint32_t k, uint64_t wl) {
  const unsigned int slot = atomicAdd(a.ovf_count, 1u);
  if (slot < a.ovf_cap) {
    a.ovf_items[slot] = (static_cast<unsigned long long>(k) << 40) | wl;
  } else {
    const uint64_t item = static_cast<uint64_t>(k) * a.m_wave + wl;
    atomicOr(a.ovf_bits + (item >> 5), 1u << (item & 31));
  }
}

#include "split_linear.cuh"
#include "split_penal.cuh"
#include "split_penal_bits.cuh"

// K2-bits eligibility of a materialized wave: does any valid scenario hold a
// demand outside [dlo, dhi]?  One pass over the tiled wave (lanes beyond m
// of the last tile are padding and skipped); a warp vote, one atomic per
// warp that saw one.
__global__ void demand_range_kernel(const uint32_t* __restrict__ tiled, uint32_t rows, uint64_t m,
                                    uint32_t dlo, uint32_t dhi, unsigned int* outside) {
  const uint64_t total = ((m + 31) / 32) * static_cast<uint64_t>(rows) * kTile;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * 4;
  bool bad = false;
  for (uint64_t e = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) * 4; e < total;
       e += stride) {
    // 4 consecutive lanes of one row (kTile is a multiple of 4); the padding
    // lanes of the last tile are never read (they may be uninitialized)
    const uint64_t w = (e / (static_cast<uint64_t>(rows) * kTile)) * kTile + (e & 31);
    if (w + 3 < m) {
      const uint4 v = *reinterpret_cast<const uint4*>(tiled + e);
      bad |= v.x < dlo || v.x > dhi || v.y < dlo || v.y > dhi || v.z < dlo || v.z > dhi ||
             v.w < dlo || v.w > dhi;
    } else {
      for (int j = 0; w + j < m; ++j) bad |= tiled[e + j] < dlo || tiled[e + j] > dhi;
    }
  }
  if (__any_sync(__activemask(), bad) && (threadIdx.x & 31) == 0) atomicOr(outside, 1u);
}

// ---------------------------------------------------------------------------
// K2: O(n^2) Bellman min (split.cpp:45-75), penalized (or forced) mode.
// Per-thread f(p) and load(p) in shared memory, [p][T] (conflict-free).
template <bool FULL, int SRC>
__global__ void __launch_bounds__(256)
split_quadratic_kernel(SplitArgs a) {
  extern __shared__ __align__(16) char smem[];
  __shared__ unsigned long long s_agg[kAggSlots];
  const uint32_t k = blockIdx.y;
  const int T = blockDim.x;
  const int n = a.n;
  TourSmem tour = load_tour(a, k, smem);
  char* arr_base = smem + ((tour_smem_bytes(n) + 15) & ~size_t(15));
  double* sf = reinterpret_cast<double*>(arr_base);        // [n][T] f(p)
  uint32_t* sl = reinterpret_cast<uint32_t*>(sf + static_cast<size_t>(n) * T);  // [n][T]
  int32_t* sr = reinterpret_cast<int32_t*>(sl + static_cast<size_t>(n) * T);    // FULL rc
  agg_cta_init(s_agg);
  __syncthreads();

  const int tid = threadIdx.x;
  const uint64_t wl = blockIdx.x * static_cast<uint64_t>(T) + tid;
  const bool active = wl < a.m_wave;
  const uint64_t w = a.w_base + wl;
  const bool hard = a.hard != 0;
  const double beta = a.beta;
  const int64_t Q = a.Q;

  double v = 0.0;
  bool overflow = false;
  if (active) {
    const uint32_t* tile_base = nullptr;
    uint64_t stream = 0;
    if (SRC == kSrcTiled) tile_base = a.tiled + (wl >> 5) * static_cast<uint64_t>(n) * kTile + (wl & 31);
    else stream = derive_stream(a.gen.seed, kStreamScenario, a.gen.first_index + wl);
    double* Vout = nullptr;
    int32_t* Cout = nullptr;
    if (FULL) {
      const uint64_t base = ((w >> 5) * static_cast<uint64_t>(n + 1)) * kTile + (w & 31);
      Vout = a.V + base;
      Cout = a.cuts + base;
      Vout[0] = 0.0;
      Cout[0] = 0;
    }
    // p = 0 entry
    sf[tid] = __dsub_rn(__dadd_rn(0.0, tour.c0[0]), tour.dist[1]);
    sl[tid] = 0u;
    if (FULL) sr[tid] = 0;
    uint32_t load = 0;
    int32_t rc = 0;
    uint32_t dnext = demand_at(a, SRC, stream, tile_base, tour.col[1]);
    for (int i = 1; i <= n; ++i) {
      const uint32_t d = dnext;
      if (i < n) dnext = demand_at(a, SRC, stream, tile_base, tour.col[i + 1]);
      const uint32_t nl = load + d;
      if (nl < load) { overflow = true; break; }  // u32 load wrapped: 64-bit fallback
      load = nl;
      const double di = tour.dist[i];
      const double ret = tour.ret[i];
      double best = kInfD;
      int32_t bestp = -1;
      for (int p = 0; p < i; ++p) {
        const double fp = sf[p * T + tid];
        if (!(fp < kInfD)) continue;  // V(p) = +inf  <=>  f(p) = +inf
        const int64_t excess = static_cast<int64_t>(load - sl[p * T + tid]) - Q;
        double cand = __dadd_rn(__dadd_rn(fp, di), ret);
        if (excess > 0) {
          if (hard) continue;
          cand = __dadd_rn(cand, __dmul_rn(beta, static_cast<double>(excess)));
        }
        if (cand < best) {
          best = cand;
          bestp = p;
        }
      }
      v = best;
      if (FULL) {
        Vout[static_cast<uint64_t>(i) * kTile] = best;
        Cout[static_cast<uint64_t>(i) * kTile] = bestp;
        rc = bestp >= 0 ? sr[bestp * T + tid] + 1 : 0;
      }
      if (i < n) {
        sf[i * T + tid] = __dsub_rn(__dadd_rn(best, tour.c0[i]), tour.dist[i + 1]);
        sl[i * T + tid] = load;
        if (FULL) sr[i * T + tid] = rc;
      }
    }
    if (overflow) {
      push_overflow(a, k, wl);
    } else {
      if (a.totals) a.totals[static_cast<uint64_t>(k) * a.m_total + w] = v;
      if (FULL) {
        const bool fin = v < kInfD;
        a.route_count[w] = fin ? rc : 0;
        a.feasible[w] = fin ? 1 : 0;
      }
    }
  }
  __syncwarp();
  agg_warp_add(s_agg, agg_pieces(v, true), active && !overflow);
  __syncthreads();
  agg_cta_flush(s_agg, a.agg + static_cast<uint64_t>(k) * kAggWords);
}

// Element i of a per-thread array interleaved across the grid.
template <typename T>
struct Strided {
  T* p;
  uint64_t s;
  __device__ __forceinline__ T& operator[](int64_t i) const { return p[i * static_cast<int64_t>(s)]; }
};

// ---------------------------------------------------------------------------
// Generic path: one thread per item with O(n) global-memory scratch and
// 64-bit loads -- the reference algorithm verbatim for any n, Q or demand
// magnitude.  Items come from the overflow list (list mode) or are all
// (tour, scenario) pairs of the wave (range mode, used for very large n).
template <bool FULL, int SRC>
__global__ void __launch_bounds__(64)
split_generic_kernel(SplitArgs a, int list_mode, uint64_t n_range_items,
                     char* scratch, uint64_t scratch_stride) {
  // launched with programmatic stream serialization after the primary
  // kernel: wait for it to complete (and its writes -- the hand-off list,
  // aggregates -- to be visible) before reading anything it wrote
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n = a.n;
  const uint64_t gtid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // per-thread arrays [n+1], interleaved across the grid ([i][thread]): the
  // lanes of a warp step through positions together, so the writes at i
  // (and most reads) coalesce instead of touching 32 lines
  (void)scratch_stride;
  const uint64_t plane = static_cast<uint64_t>(n + 1) * nthreads;
  const Strided<double> f{reinterpret_cast<double*>(scratch) + gtid, nthreads};
  const Strided<int64_t> ld{reinterpret_cast<int64_t*>(scratch) + plane + gtid, nthreads};
  const Strided<int32_t> dq{reinterpret_cast<int32_t*>(scratch + plane * 16) + gtid, nthreads};
  const Strided<int32_t> rcs{reinterpret_cast<int32_t*>(scratch + plane * 20) + gtid, nthreads};
  // one (tour, scenario) item: the reference's algorithm, totals / full
  // outputs, and its aggregate straight to global (items of one warp may
  // belong to different tours; integer atomics keep the sum exact)
  auto run_item = [&](uint32_t k, uint64_t wl) {
    double v = 0.0;
    const uint64_t w = a.w_base + wl;
    const uint64_t toff = static_cast<uint64_t>(k) * (n + 1);
    const double* dist = a.dist + toff;
    const double* ret = a.ret + toff;
    const double* c0 = a.c0 + toff;
    const uint32_t* col = a.col + toff;
    const uint32_t* tile_base = nullptr;
    uint64_t stream = 0;
    if (SRC == kSrcTiled) tile_base = a.tiled + (wl >> 5) * static_cast<uint64_t>(n) * kTile + (wl & 31);
    else stream = derive_stream(a.gen.seed, kStreamScenario, a.gen.first_index + wl);
    double* Vout = nullptr;
    int32_t* Cout = nullptr;
    if (FULL) {
      const uint64_t base = ((w >> 5) * static_cast<uint64_t>(n + 1)) * kTile + (w & 31);
      Vout = a.V + base;
      Cout = a.cuts + base;
      Vout[0] = 0.0;
      Cout[0] = 0;
    }
    const double f0 = __dsub_rn(__dadd_rn(0.0, c0[0]), dist[1]);
    if (a.linear) {
      // the reference's deque (split.cpp:77-118) with its entries' f, load,
      // index and route count stored in the deque slots (scratch planes
      // reused: f | ld | dq | rcs) and both ends cached in registers, so a
      // position touches global scratch only when an end moves -- not
      // through dependent dq -> f / ld lookups (5x fewer round trips)
      int head = 0, tail = 1;
      f[0] = f0;
      ld[0] = 0;
      dq[0] = 0;
      rcs[0] = 0;
      double front_f = f0, back_f = f0;
      int64_t front_l = 0, load = 0;
      int32_t front_i = 0, front_rc = 0, rc = 0;
      auto step = [&](int i, uint32_t d) {
        load += static_cast<int64_t>(d);
        while (head < tail && load - front_l > a.Q) {
          if (++head < tail) {
            front_f = f[head];
            front_l = ld[head];
            front_i = dq[head];
            front_rc = rcs[head];
          }
        }
        int32_t cut = -1;
        if (head >= tail) {
          v = kInfD;
          rc = 0;
        } else {
          v = __dadd_rn(__dadd_rn(front_f, dist[i]), ret[i]);
          cut = v < kInfD ? front_i : -1;
          rc = v < kInfD ? front_rc + 1 : 0;
        }
        if (FULL) {
          Vout[static_cast<uint64_t>(i) * kTile] = v;
          Cout[static_cast<uint64_t>(i) * kTile] = cut;
        }
        if (i < n) {
          const double fi = __dsub_rn(__dadd_rn(v, c0[i]), dist[i + 1]);
          while (tail > head && back_f > fi) {
            --tail;
            back_f = tail > head ? f[tail - 1] : -kInfD;
          }
          f[tail] = fi;
          ld[tail] = load;
          dq[tail] = i;
          rcs[tail] = rc;
          if (tail == head) {
            front_f = fi;
            front_l = load;
            front_i = i;
            front_rc = rc;
          }
          ++tail;
          back_f = fi;
        }
      };
      // demands are loaded one chunk of 4 positions ahead of their use
      auto dem4 = [&](int i0, uint32_t (&dd)[4]) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dd[j] = i0 + j <= n ? demand_at(a, SRC, stream, tile_base, col[i0 + j]) : 0u;
      };
      uint32_t dc[4], dn[4];
      dem4(1, dc);
      for (int i0 = 1; i0 <= n; i0 += 4) {
        dem4(i0 + 4, dn);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (i0 + j <= n) step(i0 + j, dc[j]);
#pragma unroll
        for (int j = 0; j < 4; ++j) dc[j] = dn[j];
      }
      if (a.totals) a.totals[static_cast<uint64_t>(k) * a.m_total + w] = v;
      if (FULL) {
        const bool fin = v < kInfD;
        a.route_count[w] = fin ? rc : 0;
        a.feasible[w] = fin ? 1 : 0;
      }
      agg_item_global(a.agg + static_cast<uint64_t>(k) * kAggWords, v, true);
      return;
    }
    ld[0] = 0;
    for (int i = 1; i <= n; ++i)
      ld[i] = ld[i - 1] + static_cast<int64_t>(demand_at(a, SRC, stream, tile_base, col[i]));
    f[0] = f0;
    rcs[0] = 0;
    if (!a.hard && a.pen_lmax > 0 && ld[n] <= static_cast<int64_t>(a.pen_lmax)) {
      // penalized, exact integral data: the O(n) decomposition of
      // split_penal.cuh without its ring limits -- window A = {L_i - L_p
      // <= Q} (deque of f, earliest minimum) and prefix B before it (running
      // minimum of g(p) = f(p) - beta L_p); B wins ties (earlier indices).
      // Every value is an integer below 2^31, so each fp64 op is exact and
      // equals the reference's ((f + dist_i) + ret_i) + beta * excess.
      // The deque's front (f, position, routes), its back f and the B
      // candidate's routes live in registers: a position reads global
      // scratch only when the window start advances (f, load of the leaving
      // position) or an entry pops.
      int head = 0, tail = 0, lo = 0, bidx = -1;
      double bmin = kInfD;
      int32_t brc = 0;
      dq[tail++] = 0;
      double front_f = f0, back_f = f0;
      int32_t front_p = 0, front_rc = 0;
      int64_t lo_ld = 0;  // ld[lo]
      const double beta = a.beta;
      for (int i = 1; i <= n; ++i) {
        const int64_t li = ld[i];
        while (lo < i && li - lo_ld > a.Q) {
          const double g = f[lo] - beta * static_cast<double>(lo_ld);
          if (g < bmin) {
            bmin = g;
            bidx = lo;
            brc = rcs[lo];
          }
          ++lo;
          lo_ld = ld[lo];
        }
        if (front_p < lo) {
          do {
            ++head;
            front_p = head < tail ? dq[head] : 0x7fffffff;
          } while (front_p < lo);
          if (head < tail) {
            front_f = f[front_p];
            front_rc = rcs[front_p];
          }
        }
        const double candA = head < tail ? (front_f + dist[i]) + ret[i] : kInfD;
        const double candB = bidx >= 0 ? ((bmin + dist[i]) + ret[i]) +
                                             beta * static_cast<double>(li - a.Q)
                                       : kInfD;
        const bool useB = candB <= candA;
        v = useB ? candB : candA;
        const int32_t bestp = useB ? bidx : front_p;
        const int32_t rci = (useB ? brc : front_rc) + 1;
        rcs[i] = rci;
        if (FULL) {
          Vout[static_cast<uint64_t>(i) * kTile] = v;
          Cout[static_cast<uint64_t>(i) * kTile] = bestp;
        }
        if (i < n) {
          const double fi = (v + c0[i]) - dist[i + 1];
          while (tail > head && back_f > fi) {
            --tail;
            back_f = tail > head ? f[dq[tail - 1]] : -kInfD;
          }
          dq[tail] = i;
          f[i] = fi;
          if (tail == head) {
            front_f = fi;
            front_p = i;
            front_rc = rci;
          }
          ++tail;
          back_f = fi;
        }
      }
    } else {
      for (int i = 1; i <= n; ++i) {
        double best = kInfD;
        int32_t bestp = -1;
        for (int p = 0; p < i; ++p) {
          const double fp = f[p];
          if (!(fp < kInfD)) continue;
          const int64_t excess = ld[i] - ld[p] - a.Q;
          double cand = __dadd_rn(__dadd_rn(fp, dist[i]), ret[i]);
          if (excess > 0) {
            if (a.hard) continue;
            cand = __dadd_rn(cand, __dmul_rn(a.beta, static_cast<double>(excess)));
          }
          if (cand < best) {
            best = cand;
            bestp = p;
          }
        }
        v = best;
        rcs[i] = bestp >= 0 ? rcs[bestp] + 1 : 0;
        if (FULL) {
          Vout[static_cast<uint64_t>(i) * kTile] = best;
          Cout[static_cast<uint64_t>(i) * kTile] = bestp;
        }
        if (i < n) f[i] = __dsub_rn(__dadd_rn(best, c0[i]), dist[i + 1]);
      }
    }
    if (a.totals) a.totals[static_cast<uint64_t>(k) * a.m_total + w] = v;
    if (FULL) {
      const bool fin = v < kInfD;
      a.route_count[w] = fin ? rcs[n] : 0;
      a.feasible[w] = fin ? 1 : 0;
    }
    agg_item_global(a.agg + static_cast<uint64_t>(k) * kAggWords, v, true);
  };
  if (!list_mode) {
    for (uint64_t item = gtid; item < n_range_items; item += nthreads)
      run_item(static_cast<uint32_t>(item / a.m_wave), item % a.m_wave);
    return;
  }
  const uint64_t cnt = *a.ovf_count;
  const uint64_t n_list = min(cnt, static_cast<uint64_t>(a.ovf_cap));
  for (uint64_t item = gtid; item < n_list; item += nthreads) {
    const unsigned long long it = a.ovf_items[item];
    run_item(static_cast<uint32_t>(it >> 40), it & ((1ULL << 40) - 1));
  }
  if (cnt > a.ovf_cap) {
    // the list was full: the remaining items are flagged in the bitmap
    // (bit = k * m_wave + wl).  Lane j of a warp takes bit j of a word (an
    // item per thread -- not a word per thread, which ran 32 items in
    // sequence), and lane 0 clears the word once the warp has read it, so
    // the bitmap is all-zero again for the next wave / call
    const uint64_t words = (static_cast<uint64_t>(a.k) * a.m_wave + 31) / 32;
    const uint64_t gwarp = gtid >> 5, nwarps = nthreads >> 5;
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t wd = gwarp; wd < words; wd += nwarps) {
      const uint32_t bits = a.ovf_bits[wd];
      __syncwarp();
      if (!bits) continue;
      if (lane == 0) a.ovf_bits[wd] = 0u;
      if ((bits >> lane) & 1u) {
        const uint64_t item = wd * 32 + lane;
        run_item(static_cast<uint32_t>(item / a.m_wave), item % a.m_wave);
      }
    }
  }
}

// ---- host ----------------------------------------------------------------
// Tour-only tables, written in place into one staging blob (one H2D copy);
// sections 16-byte aligned.  Per tour q, positions i = 0..n:
//   dist/ret/c0/col [k][n+1]   (generic / quadratic kernels)
//   ccol [k][npad]             (K1 / K2-int column table, slot s = position s+1)
//   itab [k][2][npad] int32    (exact integer path) | dtab [k][npad][4] fp64
//   f0d [k], f0i [k]           (f(0))
struct TableLayout {
  int npad = 0;
  size_t o_dist, o_ret, o_c0, o_col, o_ccol, o_f0d, o_f0i, o_tab, bytes;
  TableLayout(int n, uint32_t k) {
    const size_t n1 = static_cast<size_t>(n) + 1;
    npad = ((n + 3) / 4) * 4 + 4;
    size_t off = 0;
    auto sec = [&off](size_t bytes) {
      const size_t o = (off + 15) & ~size_t(15);
      off = o + bytes;
      return o;
    };
    o_dist = sec(k * n1 * 8);
    o_ret = sec(k * n1 * 8);
    o_c0 = sec(k * n1 * 8);
    o_col = sec(k * n1 * 4);
    o_ccol = sec(static_cast<size_t>(k) * npad * 4);
    o_f0d = sec(static_cast<size_t>(k) * 8);
    o_f0i = sec(static_cast<size_t>(k) * 4);
    o_tab = sec(static_cast<size_t>(k) * 4 * npad * 8);  // itab or dtab, whichever applies
    bytes = (off + 15) & ~size_t(15);
  }
};

struct TourTables {
  bool intv = false;  // every tour admits the exact integer path (itab at o_tab)
  bool ident = false; // every tour is the identity (contiguous demand rows)
  double costbound = 0.0;  // max over tours of dist_n + sum(c0 + ret) + max c0
};

// x (finite, >= 0) is an integer.  Branch-free and inline: std::floor is a
// libm call on the baseline x86-64 target, and it dominated the table build
// for large K (3 calls per position).  Below 2^52, adding and removing 2^52
// rounds x to an integer (round-to-nearest), unchanged iff x was one; every
// double from 2^52 up is an integer.
inline bool is_whole(double x) {
  constexpr double k52 = 4503599627370496.0;
  return (x >= k52) | (((x + k52) - k52) == x);  // IEEE: not folded without -ffast-math
}

// The instance checks other than the cost matrix scan (split.cpp:128-138).
void validate_instance_scalars(const scendp_routing* inst) {
  if (inst->capacity <= 0) fail(SCENDP_ERR_INVALID_ARGUMENT, "capacity Q must be > 0");
  if (!inst->hard && !(inst->penalty_beta >= 0.0))
    fail(SCENDP_ERR_INVALID_ARGUMENT, "penalty beta must be >= 0");
}

void validate_instance(const scendp_routing* inst) {
  if (!inst) fail(SCENDP_ERR_INVALID_ARGUMENT, "instance is null");
  const int n = inst->n;
  if (n < 1) fail(SCENDP_ERR_INVALID_ARGUMENT, "instance needs at least one customer");
  if (inst->capacity <= 0) fail(SCENDP_ERR_INVALID_ARGUMENT, "capacity Q must be > 0");
  if (!inst->costs) fail(SCENDP_ERR_INVALID_ARGUMENT, "cost matrix must be (n+2) x (n+2)");
  const size_t side = static_cast<size_t>(n) + 2;
  // branch-free (vectorized) scan; the messages follow the reference's
  // row-major check order (split.cpp:148-156): the first offending entry
  // decides which one is reported
  const double* c = inst->costs;
  const size_t cells = side * side;
  unsigned good = 1u;
  for (size_t e = 0; e < cells; ++e)
    good &= static_cast<unsigned>(c[e] >= 0.0) & static_cast<unsigned>(c[e] <= 1.7976931348623157e308);
  bool bad = good == 0u;
  for (size_t x = 0; x < side; ++x) bad |= c[x * side + x] != 0.0;
  if (bad) {
    for (size_t x = 0; x < side; ++x)
      for (size_t y = 0; y < side; ++y) {
        const double v = c[x * side + y];
        if (!std::isfinite(v) || v < 0.0)
          fail(SCENDP_ERR_INVALID_ARGUMENT, "cost matrix entries must be finite and >= 0");
        if (x == y && v != 0.0) fail(SCENDP_ERR_INVALID_ARGUMENT, "cost matrix diagonal must be 0");
      }
  }
  if (!inst->hard && !(inst->penalty_beta >= 0.0))
    fail(SCENDP_ERR_INVALID_ARGUMENT, "penalty beta must be >= 0");
}

// seen[c] == stamp marks customer c as visited by this tour; one array for
// all tours of a call (stamp = tour index + 1), no clearing per tour
void validate_tour(const int32_t* tour, int n, std::vector<uint32_t>& seen, uint32_t stamp) {
  for (int i = 0; i < n; ++i) {
    const int c = tour[i];
    if (c < 1 || c > n || seen[c] == stamp)
      fail(SCENDP_ERR_INVALID_ARGUMENT, "tour is not a permutation of 1.." + std::to_string(n));
    seen[c] = stamp;
  }
}

// Tour-only prefix constants, in the reference's sequential order
// (fill_prefixes, split.cpp:24-39), built straight into `blob` (layout L).
// The integer-path check: all tour costs integral and every partial sum
// < 2^29, so each fp64 op of the reference is exact and integer adds
// reproduce it bit for bit.
void build_tables(const scendp_routing* inst, const int32_t* tours, uint32_t k,
                  const TableLayout& L, char* blob, TourTables& t) {
  const int n = inst->n, side = n + 2, npad = L.npad;
  const size_t n1 = static_cast<size_t>(n) + 1;
  const double* c = inst->costs;
  auto D = [&](size_t o) { return reinterpret_cast<double*>(blob + o); };
  double* dist_all = D(L.o_dist);
  double* ret_all = D(L.o_ret);
  double* c0_all = D(L.o_c0);
  uint32_t* col_all = reinterpret_cast<uint32_t*>(blob + L.o_col);
  uint32_t* ccol_all = reinterpret_cast<uint32_t*>(blob + L.o_ccol);
  double* f0d = D(L.o_f0d);
  int32_t* f0i = reinterpret_cast<int32_t*>(blob + L.o_f0i);
  // tours are independent: large K (the SAA candidate sweeps) is split over
  // host threads, each with its own flags, combined after the join
  const unsigned parts = static_cast<unsigned>(std::min<uint64_t>(
      std::max(1u, std::min(16u, std::thread::hardware_concurrency())),
      std::max<uint64_t>(1, static_cast<uint64_t>(k) * n1 / 2048)));
  auto for_tours = [&](auto&& body) {
    parallel_parts(static_cast<int>(parts), [&](int t) {
      body(static_cast<uint32_t>(uint64_t{k} * t / parts),
           static_cast<uint32_t>(uint64_t{k} * (t + 1) / parts), static_cast<unsigned>(t));
    });
  };
  // an all-integer matrix makes every prefix integral (a rounded sum of
  // integers is an integer): for many tours one scan of the (n+2)^2 entries
  // replaces the 3 tests per tour position
  bool matrix_whole = false;
  if (static_cast<uint64_t>(k) * n1 * 3 > static_cast<uint64_t>(side) * side) {
    unsigned w = 1u;
    for (size_t e = 0; e < static_cast<size_t>(side) * side; ++e) w &= static_cast<unsigned>(is_whole(c[e]));
    matrix_whole = w != 0u;
  }
  std::vector<char> p_intv(parts, 1), p_ident(parts, 1);
  std::vector<double> p_bound(parts, 0.0);
  for_tours([&](uint32_t q0, uint32_t q1, unsigned part) {
    bool intv = true, ident = true;
    double costbound = 0.0;
    for (uint32_t q = q0; q < q1; ++q) {
      const int32_t* sq = tours + static_cast<size_t>(q) * n;
      double* dist = dist_all + q * n1;
      double* ret = ret_all + q * n1;
      double* c0 = c0_all + q * n1;
      uint32_t* col = col_all + q * n1;
      uint32_t* ccol = ccol_all + static_cast<size_t>(q) * npad;
      dist[0] = 0.0;
      dist[1] = 0.0;
      for (int i = 2; i <= n; ++i) dist[i] = dist[i - 1] + c[sq[i - 2] * side + sq[i - 1]];
      ret[0] = 0.0;
      col[0] = 0u;
      for (int i = 1; i <= n; ++i) {
        ret[i] = c[sq[i - 1] * side + (n + 1)];
        col[i] = static_cast<uint32_t>(sq[i - 1] - 1);
        ccol[i - 1] = col[i];
        ident &= sq[i - 1] == i;
      }
      for (int i = n; i < npad; ++i) ccol[i] = 0u;
      for (int i = 0; i < n; ++i) c0[i] = c[0 * side + sq[i]];
      c0[n] = 0.0;
      double bound = dist[n], cmax = 0.0;
      bool integral = true;
      for (int i = 0; i <= n; ++i) {
        if (!matrix_whole) integral &= is_whole(dist[i]) & is_whole(ret[i]) & is_whole(c0[i]);
        bound += ret[i] + c0[i];
        cmax = std::max(cmax, c0[i]);
      }
      bound += cmax;
      intv &= integral && bound < static_cast<double>(1 << 29);
      costbound = std::max(costbound, bound);
      f0d[q] = (0.0 + c0[0]) - dist[1];
    }
    p_intv[part] = intv;
    p_ident[part] = ident;
    p_bound[part] = costbound;
  });
  bool intv = true, ident = true;
  double costbound = 0.0;
  for (unsigned t = 0; t < parts; ++t) {
    intv &= p_intv[t] != 0;
    ident &= p_ident[t] != 0;
    costbound = std::max(costbound, p_bound[t]);
  }
  // per-position K1/K2 tables: integer A/B when every tour admits it, else
  // the fp64 quadruple
  for_tours([&](uint32_t q0, uint32_t q1, unsigned) {
    for (uint32_t q = q0; q < q1; ++q) {
      const double* dist = dist_all + q * n1;
      const double* ret = ret_all + q * n1;
      const double* c0 = c0_all + q * n1;
      if (intv) {
        f0i[q] = static_cast<int32_t>(f0d[q]);
        int32_t* it = reinterpret_cast<int32_t*>(blob + L.o_tab) + static_cast<size_t>(q) * 2 * npad;
        for (int i = 1; i <= n; ++i) {
          it[0 * npad + (i - 1)] = static_cast<int32_t>(dist[i] + ret[i]);
          it[1 * npad + (i - 1)] = i < n ? static_cast<int32_t>(c0[i] - dist[i + 1]) : 0;
        }
        for (int i = n; i < npad; ++i) it[i] = it[npad + i] = 0;
      } else {
        f0i[q] = 0;
        // interleaved per position: (dist, ret, c0, dist_next) of slot s at
        // dt[4 s .. 4 s + 3] (two 128-bit shared loads per K1 step)
        double* dt = D(L.o_tab) + static_cast<size_t>(q) * 4 * npad;
        for (int i = 1; i <= n; ++i) {
          double* e = dt + 4 * static_cast<size_t>(i - 1);
          e[0] = dist[i];
          e[1] = ret[i];
          e[2] = c0[i];
          e[3] = i < n ? dist[i + 1] : 0.0;
        }
        for (int i = n; i < npad; ++i) dt[4 * i] = dt[4 * i + 1] = dt[4 * i + 2] = dt[4 * i + 3] = 0.0;
      }
    }
  });
  t.intv = intv;
  t.ident = ident;
  t.costbound = costbound;
}

constexpr int kMaxQuadSmem = 200 * 1024;
constexpr int kGenericThreads = 64;
constexpr int kGenericBlocksPerSm = 2;

int quad_threads(int n) {
  // largest multiple of 32 (<= 256) whose arrays fit in ~kMaxQuadSmem
  const size_t per_thread = static_cast<size_t>(n) * (sizeof(double) + 2 * sizeof(uint32_t));
  const size_t avail = kMaxQuadSmem - tour_smem_bytes(n) - 64;
  int t = static_cast<int>(avail / per_thread / 32) * 32;
  return std::min(t, 256);
}

// cudaFuncSetAttribute only when a (device, kernel) needs more dynamic
// shared memory than already granted (it is a driver call per launch
// otherwise).
template <typename K>
void set_smem(K kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> granted;
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  const auto key = std::make_pair(dev, reinterpret_cast<const void*>(kernel));
  std::lock_guard<std::mutex> g(mu);
  auto it = granted.find(key);
  if (it != granted.end() && it->second >= bytes) return;
  CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
  granted[key] = bytes;
}

// The overflow (hand-off) pass of a wave: list mode of the generic kernel.
template <bool FULL, int KSRC>
void launch_overflow_pass(scendp_ctx* ctx, const SplitArgs& a, char* generic_scratch,
                          uint64_t generic_stride, int generic_blocks) {
  constexpr int SRC = KSRC == kSrcGenU32 ? kSrcGen : KSRC;
  // programmatic dependent launch: the pass's CTAs are scheduled while the
  // primary's last CTAs run (the primary triggers early) and wait in
  // griddepcontrol.wait, so the usually empty pass costs ~no launch gap
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(generic_blocks));
  cfg.blockDim = dim3(kGenericThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, split_generic_kernel<FULL, SRC>, a, 1, uint64_t{0},
                                generic_scratch, generic_stride));
  CUDA_CHECK(cudaGetLastError());
  ctx->count_launch();
}

// defer_overflow: the caller reads the hand-off counter back (it syncs
// anyway) and runs the overflow pass only when it is non-zero.
template <bool FULL, int KSRC>
void launch_wave(scendp_ctx* ctx, const SplitArgs& a, bool linear, char* generic_scratch,
                 uint64_t generic_stride, int generic_blocks, bool defer_overflow = false) {
  // K1 takes the specialized source; every other kernel the generic one
  constexpr int SRC = KSRC == kSrcGenU32 ? kSrcGen : KSRC;
  const int n = a.n;
  // deque form needs Q < 2^31 (u32 window arithmetic); the quadratic form
  // needs its per-thread arrays to fit in shared memory
  const bool use_generic_range =
      linear ? a.Q >= (int64_t{1} << 31) : quad_threads(n) < 32;
  const bool small_tables = tour_smem_bytes(n) <= 48 * 1024 &&
                            static_cast<size_t>(a.npad) * 36 <= 96 * 1024;
  const int tok = ctx->timing_begin(0);
  // penalized with integral data: exact O(n) form (pen_lmax > 0 marks it)
  if (!linear && !a.hard && a.pen_lmax > 0 && small_tables) {
    const int T = kPenThreads;
    const size_t smem = static_cast<size_t>(a.npad) * ((a.ident ? 0 : 4) + 2 * 4) +
                        static_cast<size_t>(T) * (a.pen_bits ? penal_bits_ring_bytes(FULL, a.n >= 100 ? 64 : 32)
                                                             : penal_ring_bytes(FULL));
    dim3 grid(static_cast<unsigned>((a.m_wave + T - 1) / T), a.k);
    SplitArgs ab = a;
    if (a.pen_bits) {
      // up to 8 scenario blocks per CTA while >= 8 waves of CTAs remain (the
      // tour tables and the aggregate flush are per CTA: C5 11.52 -> 11.11
      // ms with 8; 4: 11.16 ms)
      const uint64_t blocks = (a.m_wave + T - 1) / T;
      const uint64_t slots = static_cast<uint64_t>(ctx->sm_count) * 8;
      int units = 8;
      while (units > 1 && static_cast<uint64_t>(a.k) * ((blocks + units - 1) / units) < 8 * slots)
        units /= 2;
      ab.pen_units = units;
      grid.x = static_cast<unsigned>((blocks + units - 1) / units);
    }
    auto go = [&](auto kernel) {
      set_smem(kernel, smem);
      kernel<<<grid, T, smem, ctx->stream>>>(ab);
    };
    if (a.pen_bits) {
      auto bits = [&](auto ident, auto pr) {
        constexpr bool I = decltype(ident)::value;
        constexpr int PR = decltype(pr)::value;
        switch (a.Q >> 5) {
          case 0: go(split_penal_bits_kernel<FULL, SRC, I, 1, PR>); break;
          case 1: go(split_penal_bits_kernel<FULL, SRC, I, 2, PR>); break;
          case 2: go(split_penal_bits_kernel<FULL, SRC, I, 3, PR>); break;
          default: go(split_penal_bits_kernel<FULL, SRC, I, 4, PR>); break;
        }
      };
      using P32 = std::integral_constant<int, 32>;
      using P64 = std::integral_constant<int, 64>;
      if (a.n >= 100) {
        if (a.ident) bits(std::true_type{}, P64{});
        else bits(std::false_type{}, P64{});
      } else {
        if (a.ident) bits(std::true_type{}, P32{});
        else bits(std::false_type{}, P32{});
      }
    } else {
      if (a.ident) go(split_penal_kernel<FULL, SRC, true>);
      else go(split_penal_kernel<FULL, SRC, false>);
    }
  } else if (use_generic_range || !small_tables) {
    const uint64_t items = static_cast<uint64_t>(a.k) * a.m_wave;
    split_generic_kernel<FULL, SRC><<<generic_blocks, kGenericThreads, 0, ctx->stream>>>(
        a, 0, items, generic_scratch, generic_stride);
    CUDA_CHECK(cudaGetLastError());
    ctx->count_launch();
    ctx->timing_end(tok);
    return;
  } else if (linear) {
    const bool intv = a.itab != nullptr;
    const int T = k1_threads(intv);
    const size_t vt = intv ? 4 : 8;
    // column table (non-identity tours), position tables, per-thread rings
    // (generated demands on a column-table tour: the column table holds
    // row * gamma as u64)
    const size_t col_bytes = a.ident ? 0 : KSRC == kSrcTiled ? 4 : 8;
    const size_t smem = static_cast<size_t>(a.npad) * (col_bytes + (intv ? 2 : 4) * vt) +
                        static_cast<size_t>(k1_ring(a.ident)) * T * (vt + 4 + (FULL ? 8 : 0));
    dim3 grid(static_cast<unsigned>((a.m_wave + T - 1) / T), a.k);
    auto go = [&](auto kernel) {
      set_smem(kernel, smem);
      kernel<<<grid, T, smem, ctx->stream>>>(a);
    };
    if (intv) {
      if (a.ident) go(split_linear_kernel<FULL, KSRC, true, true>);
      else go(split_linear_kernel<FULL, KSRC, true, false>);
    } else {
      if (a.ident) go(split_linear_kernel<FULL, KSRC, false, true>);
      else go(split_linear_kernel<FULL, KSRC, false, false>);
    }
  } else {
    const int T = quad_threads(n);
    const size_t smem = ((tour_smem_bytes(n) + 15) & ~size_t(15)) +
                        static_cast<size_t>(n) * T * (sizeof(double) + 2 * sizeof(uint32_t));
    set_smem(split_quadratic_kernel<FULL, SRC>, smem);
    dim3 grid(static_cast<unsigned>((a.m_wave + T - 1) / T), a.k);
    split_quadratic_kernel<FULL, SRC><<<grid, T, smem, ctx->stream>>>(a);
  }
  CUDA_CHECK(cudaGetLastError());
  ctx->count_launch();
  // scenarios whose deque overflowed (or whose u32 load wrapped); the
  // timing event follows the pass, so nothing separates it from the DP
  // kernel (a programmatic dependent launch needs them adjacent)
  if (!defer_overflow)
    launch_overflow_pass<FULL, KSRC>(ctx, a, generic_scratch, generic_stride, generic_blocks);
  ctx->timing_end(tok);
}

// Generic (hand-off) kernel scratch: latency-bound (dependent global-scratch
// accesses), so as many threads as ~512 MB of scratch allows (an eighth of
// scratch_limit when one is set), 2..16 CTAs/SM.  (64 MB until round 2:
// 2 CTAs/SM at n = 200 -- a zero-heavy demand set that sends most scenarios
// to this pass ran 5-8x slower.)
struct GenericLayout {
  uint64_t stride;
  int blocks;
  uint64_t bytes() const { return stride * static_cast<uint64_t>(blocks) * kGenericThreads; }
};

GenericLayout generic_layout(const scendp_ctx* ctx, int n) {
  const uint64_t n1 = static_cast<uint64_t>(n) + 1;
  GenericLayout g;
  g.stride = ((n1 * (8 + 8 + 4 + 4)) + 127) & ~uint64_t{127};
  const uint64_t per_sm = static_cast<uint64_t>(ctx->sm_count) * kGenericThreads * g.stride;
  uint64_t cap = uint64_t{512} << 20;
  if (ctx->opts.scratch_limit) cap = std::min(cap, ctx->opts.scratch_limit / 8);
  g.blocks = ctx->sm_count *
             static_cast<int>(std::clamp<uint64_t>(cap / per_sm, kGenericBlocksPerSm, 16));
  return g;
}

// Hand-off list capacity and bitmap bytes of a wave of `items` items.
inline uint32_t handoff_cap(uint64_t items) {
  return static_cast<uint32_t>(std::min<uint64_t>(std::max<uint64_t>(items / 128, 1u << 16), 1u << 26));
}
inline uint64_t handoff_bits_bytes(uint64_t items) {
  return (((items + 31) / 32) * 4 + 15) & ~uint64_t{15};
}

// Device footprint model of one scendp_split_eval call (the device analogue
// of split_per_scenario_bytes / adjust_batch_size, split.cpp:287-301,
// engine.cpp:7-20): bytes that do not depend on the wave, bytes per
// scenario of a wave, and the wave the context's budget allows.  The terms
// are exactly the scratch blocks reserve_split_wave requests.
struct SplitFootprint {
  uint64_t fixed = 0, per_scenario = 0, wave = 0, budget = 0;
};

SplitFootprint split_footprint(scendp_ctx* ctx, int n, uint32_t k, const scendp_scenarios* sc,
                               uint32_t flags, const scendp_split_out* out, uint64_t table_bytes,
                               const GenericLayout& gl) {
  const uint64_t n1 = static_cast<uint64_t>(n) + 1, K = k;
  const bool full = (flags & SCENDP_SPLIT_FULL) != 0;
  const bool host_out = out->mem_kind == SCENDP_MEM_HOST;
  SplitFootprint f;
  f.fixed = table_bytes + K * sizeof(scendp_agg_raw) + 16 + gl.bytes() + (uint64_t{1} << 16) * 8;
  uint64_t in_fixed = 0;
  f.per_scenario = stage_footprint(sc, &in_fixed);
  f.fixed += in_fixed;
  f.per_scenario += K / 8 + 1 + K / 16 + 1;  // hand-off bitmap + list above its floor
  if (out->totals && host_out && !mapped_host_alias(out->totals)) f.per_scenario += K * 8;
  if (full && out->mem_kind != SCENDP_MEM_DEVICE_TILED) f.per_scenario += 12 * n1;  // tiled V, cuts
  if (full && host_out) f.per_scenario += 12 * n1 + 5;  // reference-layout V, cuts; rc, feasible
  f.wave = ctx->wave_for_model(sc->count, f.fixed, f.per_scenario, &f.budget);
  return f;
}

// Scratch blocks of one split wave (reserved before its kernels run).
struct SplitWaveBufs {
  char* handoff = nullptr;
  uint64_t bits_bytes = 0;
  uint32_t ovf_cap = 0;
  char* generic = nullptr;
  double* totals = nullptr;
  double* V = nullptr;
  int32_t* cuts = nullptr;
  double* V_ref = nullptr;
  int32_t* C_ref = nullptr;
  int32_t* rc = nullptr;
  uint8_t* feas = nullptr;
};

SplitWaveBufs reserve_split_wave(scendp_ctx* ctx, int n, uint32_t k, const scendp_scenarios* sc,
                                 bool full, const scendp_split_out* out, bool call_totals,
                                 uint64_t table_bytes, const GenericLayout& gl, uint64_t mw,
                                 uint64_t wave) {
  (void)table_bytes;
  const uint64_t n1 = static_cast<uint64_t>(n) + 1, tiles = (mw + 31) / 32;
  const bool host_out = out->mem_kind == SCENDP_MEM_HOST;
  SplitWaveBufs b;
  reserve_stage(ctx, sc, mw);
  const uint64_t items = static_cast<uint64_t>(k) * std::max(mw, wave);
  b.ovf_cap = handoff_cap(items);
  b.bits_bytes = handoff_bits_bytes(items);
  b.handoff = static_cast<char*>(ctx->scratch_get(kScrHandoff, b.bits_bytes + b.ovf_cap * 8ull));
  b.generic = static_cast<char*>(ctx->scratch_get(kScrFallback, gl.bytes()));
  if (out->totals && !call_totals)
    b.totals = static_cast<double*>(ctx->scratch_get(kScrTotals, static_cast<uint64_t>(k) * mw * 8));
  if (full && out->mem_kind != SCENDP_MEM_DEVICE_TILED) {
    b.V = static_cast<double*>(ctx->scratch_get(kScrOut1, tiles * 32 * n1 * 8));
    b.cuts = static_cast<int32_t*>(ctx->scratch_get(kScrOut2, tiles * 32 * n1 * 4));
  }
  if (full && host_out) {
    b.V_ref = static_cast<double*>(ctx->scratch_get(kScrOut5, mw * n1 * 8));
    b.C_ref = static_cast<int32_t*>(ctx->scratch_get(kScrOut6, mw * n1 * 4));
    b.rc = static_cast<int32_t*>(ctx->scratch_get(kScrOut3, mw * 4));
    b.feas = static_cast<uint8_t*>(ctx->scratch_get(kScrOut4, mw));
  }
  return b;
}

// Per-wave totals [k][mw] -> host [k][m] at column w0.
void copy_totals_back(scendp_ctx* ctx, double* host, const double* wave_totals, uint32_t k,
                      uint64_t m, uint64_t w0, uint64_t mw) {
  if (k == 1 || mw == m) {
    download(ctx, host + w0, wave_totals, static_cast<uint64_t>(k) * mw * 8);
  } else {
    CUDA_CHECK(cudaMemcpy2DAsync(host + w0, m * 8, wave_totals, mw * 8, mw * 8, k,
                                 cudaMemcpyDeviceToHost, ctx->stream));
    ctx->stats.d2h_bytes += static_cast<uint64_t>(k) * mw * 8;
  }
}

}  // namespace

// SCENDP_HOST_TRACE=1: per-call host-side phase times (microseconds) on
// stderr -- validation, staging buffer, table build, upload, launches,
// completion.
struct HostTrace {
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  char buf[256];
  int len = 0;
  HostTrace() : on(std::getenv("SCENDP_HOST_TRACE") != nullptr) {
    if (on) t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    len += std::snprintf(buf + len, sizeof(buf) - len, " %s=%.1f", what,
                         std::chrono::duration<double, std::micro>(now - last).count());
    last = now;
  }
  ~HostTrace() {
    if (on) std::fprintf(stderr, "split_eval host us:%s\n", buf);
  }
};

extern "C" scendp_status scendp_split_eval(scendp_ctx* ctx, const scendp_routing* inst,
                                           const int32_t* tours, uint32_t k_tours,
                                           const scendp_scenarios* sc, uint32_t flags,
                                           const scendp_split_out* out) {
  HostTrace trace;
  NvtxRange nvtx("scendp_split_eval");
  return guard([&] {
    if (!ctx) fail(SCENDP_ERR_INVALID_ARGUMENT, "ctx is null");
    if (!sc || !out) fail(SCENDP_ERR_INVALID_ARGUMENT, "scenarios/out is null");
    // the scan of the (n+2)^2 matrix is skipped when it equals the last one
    // that passed (glibc's vectorized memcmp is several times faster than
    // the checks); the rest of the instance is validated every call
    const size_t cells = (static_cast<size_t>(inst ? inst->n : 0) + 2) * (static_cast<size_t>(inst ? inst->n : 0) + 2);
    if (inst && inst->n >= 1 && inst->costs && ctx->valid_costs.size() == cells &&
        std::memcmp(ctx->valid_costs.data(), inst->costs, cells * sizeof(double)) == 0) {
      validate_instance_scalars(inst);
    } else {
      validate_instance(inst);
      // keep a copy for the memcmp only once a matrix is passed again (the
      // same pointer as the last validated one): callers that hand a new
      // matrix every call do not pay the copy (very large matrices: never)
      if (cells <= (size_t{1} << 20) && inst->costs == ctx->last_costs_ptr)
        ctx->valid_costs.assign(inst->costs, inst->costs + cells);
      else
        ctx->valid_costs.clear();
      ctx->last_costs_ptr = inst->costs;
    }
    const int n = inst->n;
    if (!tours || k_tours == 0) fail(SCENDP_ERR_INVALID_ARGUMENT, "need at least one tour");
    if (k_tours >= (1u << 23)) fail(SCENDP_ERR_UNSUPPORTED, "too many tours per call");
    {
      std::vector<uint32_t> seen(static_cast<size_t>(n) + 1, 0u);
      for (uint32_t q = 0; q < k_tours; ++q)
        validate_tour(tours + static_cast<size_t>(q) * n, n, seen, q + 1);
    }
    if (sc->rows != static_cast<uint64_t>(n))
      fail(SCENDP_ERR_INVALID_ARGUMENT, "demand column has " + std::to_string(sc->rows) +
                                            " entries, instance has " + std::to_string(n) +
                                            " customers");
    const bool full = (flags & SCENDP_SPLIT_FULL) != 0;
    if (full && k_tours != 1) fail(SCENDP_ERR_INVALID_ARGUMENT, "full solutions need k_tours == 1");
    if (full && (!out->values || !out->cuts || !out->route_count || !out->feasible))
      fail(SCENDP_ERR_INVALID_ARGUMENT, "full mode needs values, cuts, route_count, feasible");
    // hard mode follows the deque form (batched_expected_split, split.cpp:
    // 316-318); penalized or SCENDP_QUADRATIC -> quadratic form
    const bool linear = inst->hard && !(flags & SCENDP_QUADRATIC);
    const uint64_t m = sc->count;
    const uint32_t k = k_tours;
    trace.mark("validate");
    CUDA_CHECK(cudaSetDevice(ctx->device));

    // tour tables, built in the context's pinned staging buffer (the
    // previous call's upload from it has finished) and uploaded in one
    // async copy -- unless they equal the tables already resident on the
    // device (same instance and tours as the previous call; small K only,
    // where the comparison is cheap)
    TourTables tt;
    const TableLayout L(n, k);
    const size_t n1 = static_cast<size_t>(n) + 1;
    char* stage = static_cast<char*>(ctx->pinned_tables(L.bytes));
    trace.mark("stage");
    build_tables(inst, tours, k, L, stage, tt);
    trace.mark("build");
    const size_t used = tt.intv ? L.o_tab + static_cast<size_t>(k) * 2 * L.npad * 4 : L.bytes;
    char* dtab = static_cast<char*>(ctx->scratch_get(kScrTours, L.bytes));
    constexpr size_t kCacheBytes = 256 << 10;
    const bool cacheable = used <= kCacheBytes;
    if (!cacheable || dtab != ctx->tours_dev || ctx->tours_blob.size() != used ||
        std::memcmp(ctx->tours_blob.data(), stage, used) != 0) {
      ctx->copy(dtab, stage, used, cudaMemcpyHostToDevice);
      ctx->tables_uploaded();
      if (cacheable) {
        ctx->tours_blob.assign(stage, stage + used);
        ctx->tours_dev = dtab;
      } else {
        ctx->tours_blob.clear();
        ctx->tours_dev = nullptr;
      }
    }
    const size_t o_dist = L.o_dist, o_ret = L.o_ret, o_c0 = L.o_c0, o_col = L.o_col,
                 o_ccol = L.o_ccol, o_f0d = L.o_f0d, o_f0i = L.o_f0i;
    const size_t o_itab = L.o_tab, o_dtab = L.o_tab;
    const double* d_dist = reinterpret_cast<const double*>(dtab + o_dist);
    const double* d_ret = reinterpret_cast<const double*>(dtab + o_ret);
    const double* d_c0 = reinterpret_cast<const double*>(dtab + o_c0);
    const uint32_t* d_col = reinterpret_cast<const uint32_t*>(dtab + o_col);

    trace.mark("tables");
    // aggregates
    // raw aggregates [k] followed by the overflow counter of the first wave:
    // one memset clears both
    char* aggbuf = static_cast<char*>(ctx->agg_buffer(k * sizeof(scendp_agg_raw) + 16));
    auto* d_agg = reinterpret_cast<unsigned long long*>(aggbuf);
    unsigned int* d_ovf_count = reinterpret_cast<unsigned int*>(aggbuf + k * sizeof(scendp_agg_raw));
    CUDA_CHECK(cudaMemsetAsync(aggbuf, 0, k * sizeof(scendp_agg_raw) + 16, ctx->stream));

    // outputs: the caller's device buffers (tiled or reference layout) and
    // page-locked host totals (stored by the kernels over PCIe) are written in
    // place at each wave's offset; whatever is bound for pageable host memory
    // goes through per-wave scratch and is copied back after its wave
    const bool out_dev_tiled = out->mem_kind == SCENDP_MEM_DEVICE_TILED;
    const bool out_dev_ref = out->mem_kind == SCENDP_MEM_DEVICE;
    const bool host_out = out->mem_kind == SCENDP_MEM_HOST;
    double* zc_totals = nullptr;
    if (out->totals && host_out) zc_totals = static_cast<double*>(mapped_host_alias(out->totals));
    double* call_totals = !out->totals ? nullptr : host_out ? zc_totals : out->totals;

    // device footprint model (fixed + per-scenario bytes) -> wave size under
    // the context's budget (scratch_limit, else the free device memory)
    const GenericLayout gl = generic_layout(ctx, n);
    const SplitFootprint fpm = split_footprint(ctx, n, k, sc, flags, out, L.bytes, gl);
    uint64_t wave = fpm.wave;

    // a call that syncs anyway, in one wave, cost-only, on one GPU reads the
    // hand-off counter back with the aggregates and skips the (almost
    // always empty) overflow pass -- one launch less per call
    const bool want_agg = out->agg || out->agg_raw;
    const bool syncs = !(flags & SCENDP_ASYNC) || (host_out && out->totals) || want_agg;
    bool defer_ovf = false;
    SplitArgs last_a{};
    int last_src = kSrcTiled;
    char* gen_scratch = nullptr;
    // hand-off bitmap bytes known all-zero (in stream order); the context's
    // record stays "dirty" until every hand-off pass of the call is enqueued,
    // so an error exit in between leaves the bitmap to the next call's memset
    uint64_t known_clean = ctx->scratch_gen[kScrHandoff] == ctx->ovf_gen ? ctx->ovf_clean : 0;
    ctx->ovf_clean = 0;
    double* w_tot = nullptr;  // per-wave scratch totals [k][mw] (pageable host totals)
    for (uint64_t w0 = 0; w0 < m;) {
      const uint64_t mw = std::min(wave, m - w0);
      // every scratch block of this wave is reserved before its kernels are
      // enqueued: out of device memory halves the wave and retries
      SplitWaveBufs wb;
      try {
        // (hand-off bitmap and list sized for the full wave, so every wave
        // of the call places its list at the same offset)
        wb = reserve_split_wave(ctx, n, k, sc, full, out, call_totals != nullptr, L.bytes, gl, mw,
                                wave);
      } catch (const Error& e) {
        if (e.status != SCENDP_ERR_OUT_OF_MEMORY || wave <= 32) throw;
        wave = std::max<uint64_t>(32, (wave / 2) & ~uint64_t{31});
        release_wave_scratch(ctx);
        ++ctx->oom_retries;
        continue;
      }
      ctx->last_wave = wave;
      gen_scratch = wb.generic;
      w_tot = wb.totals;
      // overflow items for the generic kernel: a list sized for ~1% of the
      // wave's items (the rates seen at the BASELINE shapes are <= 0.3%), and
      // a bitmap of every item for the rest -- kept all-zero at rest (the
      // generic kernel clears what it processes; the bytes after it hold the
      // list, so only the part known clean is skipped when it grows)
      if (ctx->scratch_gen[kScrHandoff] != ctx->ovf_gen) {  // a new block
        ctx->ovf_gen = ctx->scratch_gen[kScrHandoff];
        known_clean = 0;
      }
      if (known_clean < wb.bits_bytes)
        CUDA_CHECK(cudaMemsetAsync(wb.handoff + known_clean, 0, wb.bits_bytes - known_clean,
                                   ctx->stream));
      // after this wave's pass: its bits are clear, its list (right after
      // the bitmap) is not
      known_clean = wb.bits_bytes;

      scendp_scenarios sw = *sc;
      sw.count = mw;
      sw.first_index = sc->first_index + w0;
      if (sc->mem_kind == SCENDP_MEM_DEVICE_TILED) sw.data = sc->data + (w0 / 32) * n * 32;
      else if (sc->mem_kind == SCENDP_MEM_HOST || sc->mem_kind == SCENDP_MEM_DEVICE)
        sw.data = sc->data + w0 * static_cast<uint64_t>(n);
      GenParams gp{};
      bool fused = false;
      const uint32_t* tiled = stage_scenarios(ctx, &sw, true, &gp, &fused);
      SplitArgs a{};
      a.n = n;
      a.Q = inst->capacity;
      a.hard = inst->hard;
      a.linear = linear;
      a.beta = inst->penalty_beta;
      a.k = k;
      a.m_wave = mw;
      // outputs are addressed wave-locally: call-level destinations are
      // passed at the wave's offset (waves start on 32-scenario tiles)
      a.w_base = 0;
      a.m_total = call_totals ? m : mw;
      a.dist = d_dist;
      a.ret = d_ret;
      a.c0 = d_c0;
      a.col = d_col;
      a.npad = L.npad;
      a.ident = tt.ident ? 1 : 0;
      // K2-int eligibility: integral tour costs (tt.intv) and an integral
      // beta; loads up to pen_lmax keep every sum exact and inside int32
      // (|values| <= 2 (costbound + beta * L) < 2^30); larger loads are
      // detected per scenario and re-run on the generic fp64 path
      a.pen_lmax = 0;
      // (the kernel's 16-bit rings need Q < 2^15 and n < 2^16)
      if (!inst->hard && tt.intv && !(flags & SCENDP_QUADRATIC) && inst->capacity < 32768 &&
          n < 65536 &&
          inst->penalty_beta == std::floor(inst->penalty_beta) && inst->penalty_beta >= 0.0 &&
          inst->penalty_beta <= 1048576.0) {
        const double room = static_cast<double>(1 << 29) - tt.costbound;
        const double lm = inst->penalty_beta > 0.0 ? room / inst->penalty_beta : 2147483647.0;
        a.pen_lmax = static_cast<uint32_t>(std::min(lm, 2147483647.0 - static_cast<double>(inst->capacity)));
      }
      a.pen_bits = 0;
      a.ccol = reinterpret_cast<const uint32_t*>(dtab + o_ccol);
      a.itab = tt.intv ? reinterpret_cast<const int32_t*>(dtab + o_itab) : nullptr;
      a.dtab = reinterpret_cast<const double*>(dtab + o_dtab);
      a.f0d = reinterpret_cast<const double*>(dtab + o_f0d);
      a.f0i = reinterpret_cast<const int32_t*>(dtab + o_f0i);
      a.tiled = tiled;
      a.gen = gp;
      a.totals = !out->totals ? nullptr : call_totals ? call_totals + w0 : wb.totals;
      if (full) {
        const uint64_t toff = (w0 / 32) * n1 * 32;
        a.V = out_dev_tiled ? out->values + toff : wb.V;
        a.cuts = out_dev_tiled ? out->cuts + toff : wb.cuts;
        a.route_count = host_out ? wb.rc : out->route_count + w0;
        a.feasible = host_out ? wb.feas : out->feasible + w0;
      }
      a.agg = d_agg;
      a.ovf_count = d_ovf_count;
      a.ovf_items = reinterpret_cast<unsigned long long*>(wb.handoff + wb.bits_bytes);
      a.ovf_cap = wb.ovf_cap;
      a.ovf_bits = reinterpret_cast<uint32_t*>(wb.handoff);
      if (w0 > 0) CUDA_CHECK(cudaMemsetAsync(d_ovf_count, 0, 4, ctx->stream));
      const bool u32 = fused && gp.kind == SCENDP_DIST_UNIFORM && gp.span32 != 0;
      // K2-bits (window bitmap) when Q <= 127 and every demand of the wave is
      // known to lie in [1, min(31, Q)]: from the distribution for generated
      // demands, else from one pass over the materialized wave (a 4-byte
      // read-back; the penalized pass it selects for runs ~100x longer)
      if (!linear && !inst->hard && a.pen_lmax > 0 && inst->capacity <= 127 &&
          !std::getenv("SCENDP_K2_NO_BITS")) {
        const uint32_t dhi = static_cast<uint32_t>(std::min<int64_t>(31, inst->capacity));
        if (fused) {
          a.pen_bits = gp.kind == SCENDP_DIST_UNIFORM && gp.lo >= 1 &&
                       static_cast<uint64_t>(gp.lo) + gp.span - 1 <= dhi;
        } else {
          unsigned int* d_out = d_ovf_count + 2;
          CUDA_CHECK(cudaMemsetAsync(d_out, 0, 4, ctx->stream));
          const int blocks = std::max(1, std::min<int>(ctx->sm_count * 8,
              static_cast<int>((((mw + 31) / 32) * n * 32 / 4 + 255) / 256)));
          demand_range_kernel<<<blocks, 256, 0, ctx->stream>>>(tiled, static_cast<uint32_t>(n), mw,
                                                               1u, dhi, d_out);
          CUDA_CHECK(cudaGetLastError());
          ctx->count_launch();
          unsigned int outside = 1;
          CUDA_CHECK(cudaMemcpyAsync(&outside, d_out, 4, cudaMemcpyDeviceToHost, ctx->stream));
          CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
          a.pen_bits = outside == 0;
        }
      }
      last_a = a;
      last_src = u32 ? kSrcGenU32 : fused ? kSrcGen : kSrcTiled;
      defer_ovf = syncs && !full && w0 == 0 && mw == m && !ctx->nccl_comm;
      const uint64_t gstride = gl.stride;
      const int gblocks = gl.blocks;
      if (full) {
        if (u32) launch_wave<true, kSrcGenU32>(ctx, a, linear, gen_scratch, gstride, gblocks);
        else if (fused) launch_wave<true, kSrcGen>(ctx, a, linear, gen_scratch, gstride, gblocks);
        else launch_wave<true, kSrcTiled>(ctx, a, linear, gen_scratch, gstride, gblocks);
      } else {
        if (u32) launch_wave<false, kSrcGenU32>(ctx, a, linear, gen_scratch, gstride, gblocks, defer_ovf);
        else if (fused) launch_wave<false, kSrcGen>(ctx, a, linear, gen_scratch, gstride, gblocks, defer_ovf);
        else launch_wave<false, kSrcTiled>(ctx, a, linear, gen_scratch, gstride, gblocks, defer_ovf);
      }
      // per-wave copies back (a deferred hand-off pass -- single wave only --
      // still writes totals: that wave's copy follows it below)
      if (!defer_ovf && out->totals && !call_totals) copy_totals_back(ctx, out->totals, wb.totals, k, m, w0, mw);
      if (full && !out_dev_tiled) {
        // tiled -> reference layout [mw][n+1], into the caller's device
        // buffer at the wave's rows or through scratch to host memory
        double* V_ref = out_dev_ref ? out->values + w0 * n1 : wb.V_ref;
        int32_t* C_ref = out_dev_ref ? out->cuts + w0 * n1 : wb.C_ref;
        launch_from_tiled<double>(ctx, wb.V, n1, mw, V_ref);
        launch_from_tiled<int32_t>(ctx, wb.cuts, n1, mw, C_ref);
        if (host_out) {
          download(ctx, out->values + w0 * n1, V_ref, mw * n1 * 8);
          download(ctx, out->cuts + w0 * n1, C_ref, mw * n1 * 4);
          ctx->copy(out->route_count + w0, wb.rc, mw * 4, cudaMemcpyDeviceToHost);
          ctx->copy(out->feasible + w0, wb.feas, mw, cudaMemcpyDeviceToHost);
        }
      }
      w0 += mw;
    }

    trace.mark("launch");
    // deferred overflow pass: aggregates + hand-off counter in one read
    const uint64_t agg_bytes = static_cast<uint64_t>(k) * sizeof(scendp_agg_raw);
    char* h_aggc = nullptr;
    if (defer_ovf && m > 0) {
      h_aggc = static_cast<char*>(ctx->pinned_agg(agg_bytes + 16));
      ctx->copy(h_aggc, aggbuf, agg_bytes + 16, cudaMemcpyDeviceToHost);
      ctx->sync();
      uint32_t handed_off = 0;
      std::memcpy(&handed_off, h_aggc + agg_bytes, 4);
      if (handed_off > 0) {
        const uint64_t gstride = gl.stride;
        const int gblocks = gl.blocks;
        if (last_src == kSrcGenU32)
          launch_overflow_pass<false, kSrcGenU32>(ctx, last_a, gen_scratch, gstride, gblocks);
        else if (last_src == kSrcGen)
          launch_overflow_pass<false, kSrcGen>(ctx, last_a, gen_scratch, gstride, gblocks);
        else
          launch_overflow_pass<false, kSrcTiled>(ctx, last_a, gen_scratch, gstride, gblocks);
        h_aggc = nullptr;  // aggregates changed: read them again below
      }
      if (out->totals && !call_totals) copy_totals_back(ctx, out->totals, w_tot, k, m, 0, m);
    }
    ctx->ovf_clean = known_clean;  // every hand-off pass is enqueued
    // the single collective: per-candidate raw aggregates, K x 16 u64
    ctx->allreduce_agg(d_agg, static_cast<uint64_t>(k) * kAggWords);
    if (out->totals && zc_totals) ctx->stats.d2h_bytes += k * m * 8;  // stored by the kernels
    scendp_agg_raw* h_raw = nullptr;
    if (want_agg) {
      h_raw = static_cast<scendp_agg_raw*>(ctx->pinned_agg(agg_bytes + 16));
      if (!h_aggc) ctx->agg_readback(h_raw, d_agg, agg_bytes);
    }
    if (syncs || (host_out && full)) ctx->sync();
    trace.mark("sync");
    if (want_agg) {
      if (out->agg_raw) std::memcpy(out->agg_raw, h_raw, k * sizeof(scendp_agg_raw));
      if (out->agg) finalize_agg(h_raw, 1, k, out->agg);
    }
  });
}

extern "C" scendp_status scendp_split_footprint(scendp_ctx* ctx, const scendp_routing* inst,
                                                uint32_t k_tours, const scendp_scenarios* sc,
                                                uint32_t flags, const scendp_split_out* out,
                                                scendp_footprint* fp) {
  return guard([&] {
    if (!ctx || !inst || !sc || !out || !fp) fail(SCENDP_ERR_INVALID_ARGUMENT, "null argument");
    if (inst->n < 1 || k_tours == 0) fail(SCENDP_ERR_INVALID_ARGUMENT, "need n >= 1 and a tour");
    CUDA_CHECK(cudaSetDevice(ctx->device));
    const TableLayout L(inst->n, k_tours);
    const SplitFootprint f = split_footprint(ctx, inst->n, k_tours, sc, flags, out, L.bytes,
                                             generic_layout(ctx, inst->n));
    fp->fixed_bytes = f.fixed;
    fp->per_scenario_bytes = f.per_scenario;
    fp->wave = f.wave;
    fp->budget = f.budget;
  });
}
