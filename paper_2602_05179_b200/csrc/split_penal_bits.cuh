// split_penal_bits.cuh -- K2-bits: the penalized O(n) split (split_penal.cuh)
// with the window start counted from a register bitmap instead of walked.
// Included by split.cu after split_penal.cuh.  Reference:
// split_core_quadratic, proj/src/split.cpp:45-75.
//
// Same decomposition as K2-int (window A = {L_i - L_p <= Q}: the deque front;
// prefix B = [0, lo): PM(lo-1) + beta (L_i - Q)); what changes is how lo, the
// number of positions whose load is below the threshold T_i = L_i - Q, is
// kept.  When every demand of a scenario is in [1, 31] the loads are
// strictly increasing, so each position owns one load value, and a 128-bit
// register bitmap R holds the positions inside the window relative to the
// threshold: bit k <-> load T + k.  Per position i (d = d_i, T' = T + d):
//   * the positions leaving the window are those with loads in [T, T'):
//     bits 0 .. d-1, so lo += popc(R & (2^d - 1));
//   * R >>= d (the threshold moved by d);
//   * position i, load L_i = T' + Q, enters at bit Q (Q <= 127; the kernel
//     is instantiated per bitmap width W = Q/32 + 1 words, so bit Q is in
//     the top word: one OR).
// Branch-free, no per-lane loop: the round-1 kernel walked the window start
// through a ring of loads, a data-dependent loop under SIMT divergence
// (K2).  The ring of loads is gone (2 B per position per
// thread), so more CTAs fit on an SM.  A demand outside [1, 31] (a zero
// demand merges load values; d > 31 spans bitmap words) sends the scenario
// to the generic kernel, like a ring overflow; the host takes this kernel
// only when the call's demands are known to lie in [1, 31] and Q <= 127.
#pragma once

// Host side: bytes of the K2-bits rings per thread (split.cu sizes the CTA):
// deque f (4) [| rc (4)] and positions (2); PM ring (4) [| index, rc (8)].
// PR: prefix-minimum ring slots per thread (it holds [lo-1, i+4]).  32 keeps
// 7 CTAs/SM; 64 (5 CTAs/SM) removes the hand-offs of long windows, which
// grow with n: measured C5 (n = 50) 11.4 ms + 0.33 ms hand-off pass with 32
// vs 14.3 ms with 64; C2 penalized (n = 200, 2x10^5) 0.61 ms per call with
// 32 (7.5 % of scenarios handed off) vs 0.25 ms with 64.  The host takes 64
// for n >= 100.
__host__ __device__ constexpr int penal_bits_ring_bytes(bool full, int pr) {
  return kRing * (4 + 2 + (full ? 4 : 0)) + pr * (4 + (full ? 8 : 0));
}

template <int OFF>
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1+%2];" : "=h"(v) : "r"(a), "n"(OFF));
  return v;
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(static_cast<unsigned short>(v)));
}

// W: bitmap words, Q in [32 (W-1), 32 W) -- the entry bit Q then always sits
// in the top word (one OR per position, W funnel shifts)
template <bool FULL, int SRC, bool IDENT, int W, int PR>
__global__ void __launch_bounds__(kPenThreads)
split_penal_bits_kernel(SplitArgs a) {
  constexpr int T = kPenThreads;
  constexpr int kBPosRing = PR;
  constexpr int kBPosMaskH = kBPosRing * kH - 1;
  extern __shared__ __align__(16) char smem[];
  __shared__ unsigned long long s_agg[kAggSlots];
  const uint32_t k = blockIdx.y;
  const int n = a.n;
  const int npad = a.npad;
  const int tid = threadIdx.x;
  // thread-minor rings, 4-byte arrays first: deque f [| rc], PM [| PM index
  // | PM rc]; then the 2-byte deque positions.  Counters are byte offsets of
  // 2-byte slots (at16 / at32 of split_penal.cuh).
  int32_t* dq_f = reinterpret_cast<int32_t*>(smem) + tid;
  int32_t* dq_r = dq_f + kRing * T;                                            // FULL
  int32_t* ps_pm = dq_f + (FULL ? 2 : 1) * kRing * T;
  int32_t* ps_pi = ps_pm + kBPosRing * T;                                       // FULL
  int32_t* ps_pr = ps_pi + kBPosRing * T;                                       // FULL
  uint16_t* dq_p = reinterpret_cast<uint16_t*>(ps_pm - tid + (FULL ? 3 : 1) * kBPosRing * T) + tid;
  uint32_t* s_col = reinterpret_cast<uint32_t*>(smem + T * penal_bits_ring_bytes(FULL, PR));
  int32_t* s_tab = reinterpret_cast<int32_t*>(s_col + (IDENT ? 0 : npad));  // A | B
  {
    const uint32_t* gcol = a.ccol + static_cast<uint64_t>(k) * npad;
    if (!IDENT)
      for (int x = threadIdx.x; x < npad; x += T) s_col[x] = gcol[x];
    const int32_t* g = a.itab + static_cast<uint64_t>(k) * 2 * npad;
    for (int x = threadIdx.x; x < 2 * npad; x += T) s_tab[x] = g[x];
  }
  agg_cta_init(s_agg);
  __syncthreads();

  uint32_t Qc = static_cast<uint32_t>(a.Q);  // host: Q <= 127
  Qc += static_cast<uint32_t>(a.m_total >> 62);  // + 0, keeps Q in a register
  const int32_t beta = static_cast<int32_t>(a.beta);
  const uint32_t lmax = a.pen_lmax;  // loads above this leave the exact range
  // bit Q of the bitmap: bit Q & 31 of the top word W-1 (host: Q >> 5 == W-1)
  const uint32_t qb = 1u << (Qc & 31);

  // a.pen_units blocks of T scenarios per CTA (the tour tables and the
  // aggregate flush are per CTA)
  for (int unit = 0; unit < a.pen_units; ++unit) {
  const uint64_t wl = (blockIdx.x * static_cast<uint64_t>(a.pen_units) + unit) * T + tid;
  const bool active = wl < a.m_wave;
  const uint64_t w = a.w_base + wl;
  int32_t v = 0;
  bool ok = true;
  int32_t rc = 0;
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
    // position 0: f(0) = (0.0 + c(0, s_1)) - dist[1], L_0 = 0, g(0) = f(0)
    const int32_t f0 = a.f0i[k];
    ps_pm[0] = f0;
    if (FULL) {
      ps_pi[0] = 0;
      ps_pr[0] = 0;
    }
    // deque: -inf sentinel in slot 0, entry p = 0 in slot 1 (K1 layout).  As
    // in K1 the ring is not circular and its ends are 32-bit shared
    // addresses of f-plane slots (one LDS/STS with an immediate offset per
    // access, rc plane at +kDqPlane); the 2-byte position plane of a slot is
    // at (f address >> 1) + pofs.  Live entries move back to the bottom when
    // a chunk's pushes would run past the end (rare: the head advances only
    // by window evictions of the front).
    constexpr int kDqStep = T * 4, kDqPlane = kRing * kDqStep;
    const uint32_t fbase = smem_addr(dq_f);
    const uint32_t pofs = smem_addr(dq_p) - (fbase >> 1);
    auto pa = [&](uint32_t fa) { return (fa >> 1) + pofs; };
    dq_f[0] = INT32_MIN;
    dq_f[T] = f0;
    dq_p[T] = 0;
    if (FULL) dq_r[T] = 0;
    uint32_t head = fbase + kDqStep, tail = fbase + 2 * kDqStep;
    int32_t front_f = f0, back_f = f0;
    int front_p = 0;                    // position of the deque front
    int32_t front_rc = 0;
    int lo_c = 0;                       // window start lo, as a position counter (lo * kH)
    int32_t bmin = kPenInf;             // PM(lo - 1); kPenInf while lo == 0
    int32_t bidx = -1, brc = 0;
    int32_t pm = f0, pm_i = 0, pm_rc = 0;  // running prefix minimum of g
    uint32_t load = 0;
    // window bitmap: bit j <-> load T + j (T = load - Q); position 0 (load 0)
    // sits at bit Q
    uint32_t R[W];
#pragma unroll
    for (int j = 0; j < W; ++j) R[j] = j == W - 1 ? qb : 0u;

    // one DP position (i_c = i * kH); d in [1, 31] and ring room are checked
    // per chunk by the caller
    auto step = [&](int i, int i_c, uint32_t d, int32_t Ai, int32_t Bi, auto push_tag) {
      constexpr bool PUSH = decltype(push_tag)::value;
      load += d;
      // positions whose load fell below the new threshold: bits 0 .. d-1
      const int leave = __popc(R[0] & ((1u << d) - 1u));
#pragma unroll
      for (int j = 0; j < W - 1; ++j) R[j] = __funnelshift_r(R[j], R[j + 1], d);
      R[W - 1] >>= d;
      // (unconditional: a branch on leave > 0 measured 12.19 vs 12.15 ms)
      {
        lo_c += leave * kH;
        const int pc = lo_c - kH;  // lo - 1
        if (lo_c > 0) bmin = at32(ps_pm, pc, kBPosMaskH);
        if (FULL) {
          bidx = at32(ps_pi, pc, kBPosMaskH);
          brc = at32(ps_pr, pc, kBPosMaskH);
        }
        // deque entries before lo leave from the front (entry i-1 stays:
        // d_i <= 31 < ... its load is >= T' since d_i <= Q); the vacated slot
        // becomes the -inf sentinel below the head
        const int lo = static_cast<int>(static_cast<unsigned>(lo_c) / kH);
        if (front_p < lo) {
          do {
            sts32<0>(head, static_cast<uint32_t>(INT32_MIN));
            head += kDqStep;
            front_p = static_cast<int>(lds16<0>(pa(head)));
          } while (front_p < lo);
          front_f = static_cast<int32_t>(lds32<0>(head));
          if (FULL) front_rc = static_cast<int32_t>(lds32<kDqPlane>(head));
        }
      }
      // candidates: window A (deque front) and prefix B (prefix minimum)
      const int32_t candA = front_f + Ai;
      const int32_t candB = lo_c > 0 ? bmin + Ai + beta * static_cast<int32_t>(load - Qc) : kPenInf;
      const bool useB = candB <= candA;  // B's indices come first: ties go to B
      v = useB ? candB : candA;
      if (FULL) {
        rc = (useB ? brc : front_rc) + 1;
        Vout[static_cast<uint64_t>(i) * kTile] = static_cast<double>(v);
        Cout[static_cast<uint64_t>(i) * kTile] = useB ? bidx : front_p;
      }
      if constexpr (PUSH) {
        const int32_t fi = v + Bi;
        const int32_t g = fi - beta * static_cast<int32_t>(load);
        if (g < pm) {  // strict: the earliest minimum stays
          pm = g;
          if (FULL) {
            pm_i = i;
            pm_rc = rc;
          }
        }
        at32(ps_pm, i_c, kBPosMaskH) = pm;
        if (FULL) {
          at32(ps_pi, i_c, kBPosMaskH) = pm_i;
          at32(ps_pr, i_c, kBPosMaskH) = pm_rc;
        }
        // position i enters the window bitmap at bit Q (load T' + Q)
        R[W - 1] |= qb;
        // strict pop (sentinel-terminated), then push (K1 deque); the deque
        // is non-empty here, so it can only empty by popping
        if (back_f > fi) {
          do {
            tail -= kDqStep;
            back_f = static_cast<int32_t>(lds32<-kDqStep>(tail));
          } while (back_f > fi);
          if (tail == head) {
            front_f = fi;
            front_p = i;
            if (FULL) front_rc = rc;
          }
        }
        sts32<0>(tail, static_cast<uint32_t>(fi));
        sts16(pa(tail), static_cast<uint32_t>(i));
        if (FULL) sts32<kDqPlane>(tail, static_cast<uint32_t>(rc));
        tail += kDqStep;
        back_f = fi;
      }
    };
    auto load4 = [&](int s0, uint32_t (&dd)[4]) {
      uint4 cr = make_uint4(s0, s0 + 1, s0 + 2, s0 + 3);
      if (!IDENT) cr = *reinterpret_cast<const uint4*>(s_col + s0);
      const uint32_t rows[4] = {cr.x, cr.y, cr.z, cr.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        dd[j] = s0 + j < n ? demand_at(a, SRC, stream, tile_base, rows[j]) : 1u;
    };
    auto tab4 = [&](int s0, int4& A4, int4& B4) {
      A4 = *reinterpret_cast<const int4*>(s_tab + s0);
      B4 = *reinterpret_cast<const int4*>(s_tab + npad + s0);
    };
    using Push = std::true_type;
    using Last = std::false_type;
    // room for 4 pushes: the PM ring must hold [lo-1, i] for every i of the
    // chunk, the deque its live entries + 4 + the sentinel slot
    auto room = [&](int s0) {
      if ((s0 + 4) * kH - lo_c > (kBPosRing - 2) * kH) return false;
      if (tail + 4 * kDqStep <= fbase + kDqPlane) return true;
      // compact: the sentinel and the live entries back to slots 0..len
      const uint32_t len = (tail - head) / kDqStep;
      if (len + 5 > static_cast<uint32_t>(kRing)) return false;
      uint32_t dst = fbase + kDqStep;
      for (uint32_t src = head; src < tail; src += kDqStep, dst += kDqStep) {
        sts32<0>(dst, lds32<0>(src));
        sts16(pa(dst), lds16<0>(pa(src)));
        if (FULL) sts32<kDqPlane>(dst, lds32<kDqPlane>(src));
      }
      sts32<0>(fbase, static_cast<uint32_t>(INT32_MIN));
      head = fbase + kDqStep;
      tail = dst;
      return true;
    };
    // every demand of the chunk in [1, 31] (and <= Q: 31 < Q is not
    // required -- Q >= 1 and d <= Q keeps entry i-1 in the window, checked)
    auto dem_ok = [&](const uint32_t (&dd)[4]) {
      const uint32_t mx = max(max(dd[0], dd[1]), max(dd[2], dd[3]));
      const uint32_t mn = min(min(dd[0], dd[1]), min(dd[2], dd[3]));
      return mn >= 1u && mx <= min(31u, Qc);
    };
    const int npush = n - 1;
    uint32_t dc[4], dn[4] = {1u, 1u, 1u, 1u};
    load4(0, dc);
    int s0 = 0;
    for (; s0 + 4 <= npush; s0 += 4) {
      if (s0 + 4 < n) load4(s0 + 4, dn);
      if (!dem_ok(dc) || !room(s0)) {
        ok = false;
        break;
      }
      int4 A4, B4;
      tab4(s0, A4, B4);
      step(s0 + 1, (s0 + 1) * kH, dc[0], A4.x, B4.x, Push{});
      step(s0 + 2, (s0 + 2) * kH, dc[1], A4.y, B4.y, Push{});
      step(s0 + 3, (s0 + 3) * kH, dc[2], A4.z, B4.z, Push{});
      step(s0 + 4, (s0 + 4) * kH, dc[3], A4.w, B4.w, Push{});
#pragma unroll
      for (int j = 0; j < 4; ++j) dc[j] = dn[j];
    }
    if (ok) {
      if (!dem_ok(dc) || !room(s0)) {
        ok = false;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = s0 + j + 1;
          const int32_t Ai = s_tab[i - 1], Bi = s_tab[npad + i - 1];
          if (i < n) step(i, i * kH, dc[j], Ai, Bi, Push{});
          else if (i == n) step(i, i * kH, dc[j], Ai, Bi, Last{});
        }
      }
    }
    if (ok && load > lmax) ok = false;  // values may have left the exact range
    if (!ok) {
      push_overflow(a, k, wl);
    } else {
      if (a.totals) a.totals[static_cast<uint64_t>(k) * a.m_total + w] = static_cast<double>(v);
      if (FULL) {
        a.route_count[w] = rc;
        a.feasible[w] = 1;
      }
    }
  }
  const double vout = active && ok ? static_cast<double>(v) : 0.0;
  __syncwarp();
  agg_warp_add(s_agg, agg_pieces(vout, true), active && ok);
  }
  __syncthreads();
  agg_cta_flush(s_agg, a.agg + static_cast<uint64_t>(k) * kAggWords);
}
