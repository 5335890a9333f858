// split_linear.cuh -- K1: hard capacities, O(n) monotone deque
// (reference split_core_linear, proj/src/split.cpp:77-118).  Included by
// split.cu (shares SplitArgs / demand_at / push_overflow).
//
// The kernel is issue-bound (its DRAM traffic equals the algorithmic 4n+8
// bytes per scenario), so the step is written for instruction count:
//  * tour constants arrive as 128-bit broadcast loads once per 4 positions
//    (chunked SoA tables in shared memory);
//  * the deque's front entry (f, load, idx, routes) and back f-value live in
//    registers; the per-thread ring in shared memory is read only when an end
//    moves (eviction / pop) and written once per push;
//  * the deque is never empty at the start of a position (position i-1 was
//    just pushed) and, unless d_i > Q, entry i-1 survives the eviction, so
//    the common path carries no emptiness tests: the rare "window emptied"
//    and "popped empty" cases are handled inside the eviction / pop bodies;
//  * ring overflow is checked once per chunk (<= 11 entries before a chunk
//    of 4 pushes cannot reach 16).
//
// Value type VT: double (the reference's arithmetic verbatim), or int32 when
// the host proved every tour cost is an integer and every partial sum stays
// below 2^29.  Then every fp64 operation of the reference is exact, and
//   V(i) = f(front) + (dist_i + ret_i),  f(i) = V(i) + (c0_i - dist_{i+1})
// reproduce its doubles bit for bit with one integer add each.  +inf is the
// class of values >= 2^29 (an emptied window yields 2^30 and inf-class values
// never decrease below 2^30 - dist_n).  Inf-class entries can
// only occupy the back of the deque, so the finite prefix -- which alone
// decides V and the cuts -- is identical to the reference's.
#pragma once

constexpr int32_t kIntInf = 1 << 30;      // value of an emptied window
constexpr int32_t kIntFinite = 1 << 29;   // v < kIntFinite  <=>  finite
constexpr int kK1Threads = 128;           // CTA size (ring stride)
constexpr int kK1Prefetch = 2;            // demand chunks in flight ahead
constexpr int kRingSpan = kRing * kK1Threads;  // ring elements per array
constexpr int kStep = kK1Threads * 4;           // counters: byte offsets of 4-byte slots
constexpr int kMask = kRing * kStep - 1;

// Ring slot at counter c (bytes for 4-byte elements, scaled for wider ones).
template <typename E>
__device__ __forceinline__ E& ring_at(E* base, int c) {
  return *reinterpret_cast<E*>(reinterpret_cast<char*>(base) + (sizeof(E) / 4) * (c & kMask));
}

template <typename VT>
struct K1State {
  uint32_t load;
  int head, tail;  // slot * kStep (byte offsets), unbounded, masked on access
  VT front_f, back_f, v;
  uint32_t front_l;
  int32_t front_i, front_rc, rc;
};

template <typename VT>
__device__ __forceinline__ bool k1_finite(VT v) {
  if constexpr (std::is_same<VT, int32_t>::value) return v < kIntFinite;
  else return v < kInfD;
}

template <typename VT>
__device__ __forceinline__ double k1_to_double(VT v) {
  if constexpr (std::is_same<VT, int32_t>::value)
    return v < kIntFinite ? static_cast<double>(v) : kInfD;
  else return v;
}

template <typename VT>
__device__ __forceinline__ VT k1_inf() {
  if constexpr (std::is_same<VT, int32_t>::value) return kIntInf;
  else return kInfD;
}

template <typename VT>
__device__ __forceinline__ VT k1_neg_inf() {
  if constexpr (std::is_same<VT, int32_t>::value) return INT32_MIN;
  else return -kInfD;
}

// One DP position.  PUSH = (i < n).  Ring slot s of this thread lives at
// ring_at(rf, s) (rf/rl/ri/rr are per-thread base pointers).
//
// SAFE = false is the fast form for a position with d_i <= Q (checked per
// chunk): entry i-1, at the back, then survives the eviction, so the window
// never empties and the eviction loop needs no emptiness test; and since the
// deque is non-empty before the pops, it can only become empty by popping,
// so the "popped empty" front update lives inside the (rarer) pop branch.
// SAFE = true handles any d_i (window emptied when d_i > Q).
// NOEVICT (with SAFE = false): the caller proved no eviction can happen at
// this position (see the chunk loop), so the window test is skipped.
template <typename VT, bool FULL, bool PUSH, bool SAFE = true, bool NOEVICT = false>
__device__ __forceinline__ void k1_step(K1State<VT>& s, int i, uint32_t d, uint32_t Qc, VT t0,
                                        VT t1, VT t2, VT t3, VT* __restrict__ rf,
                                        uint32_t* __restrict__ rl, int32_t* __restrict__ ri,
                                        int32_t* __restrict__ rr, double* Vout, int32_t* Cout) {
  s.load += d;
  // evict predecessors whose route (p, i] exceeds Q (split.cpp:93-96); the
  // evicted slot becomes the -inf sentinel below the new head
  if constexpr (SAFE) {
    if (d > Qc) {
      // every route into i carries d_i > Q: the window empties.  Decided on
      // d itself -- the u32 difference load - front_l wraps once d_i >=
      // 2^32 - Q (loads are int64 in the reference, split.cpp:93); with
      // d_i <= Q every window difference is < 2Q < 2^32 and exact mod 2^32
      ring_at(rf, s.tail - kStep) = k1_neg_inf<VT>();
      s.head = s.tail;
      s.back_f = k1_neg_inf<VT>();
      s.front_f = k1_inf<VT>();
      s.front_l = s.load;
      if (FULL) {
        s.front_i = -1;
        s.front_rc = -1;
      }
    }
    while (s.load - s.front_l > Qc) {
      ring_at(rf, s.head) = k1_neg_inf<VT>();
      s.head += kStep;
      if (s.head == s.tail) {
        // only when d_i > Q: every route into i overflows, V(i) = +inf.  The
        // placeholder front (inf-class f, load of position i) stands in for
        // entry i until it is pushed; the parked back value stops the pops.
        s.back_f = k1_neg_inf<VT>();
        s.front_f = k1_inf<VT>();
        s.front_l = s.load;
        if (FULL) {
          s.front_i = -1;
          s.front_rc = -1;
        }
        break;
      }
      const int hs = s.head;
      s.front_f = ring_at(rf, hs);
      s.front_l = ring_at(rl, hs);
      if (FULL) {
        s.front_i = ring_at(ri, hs);
        s.front_rc = ring_at(rr, hs);
      }
    }
  } else if constexpr (!NOEVICT) {
    if (s.load - s.front_l > Qc) {
      do {
        ring_at(rf, s.head) = k1_neg_inf<VT>();
        s.head += kStep;
        s.front_l = ring_at(rl, s.head);
      } while (s.load - s.front_l > Qc);
      const int hs = s.head;
      s.front_f = ring_at(rf, hs);
      if (FULL) {
        s.front_i = ring_at(ri, hs);
        s.front_rc = ring_at(rr, hs);
      }
    }
  }
  if constexpr (std::is_same<VT, int32_t>::value) s.v = s.front_f + t0;
  else s.v = __dadd_rn(__dadd_rn(s.front_f, t0), t1);
  if (FULL) {
    const bool fin = k1_finite(s.v);
    s.rc = fin ? s.front_rc + 1 : 0;
    Vout[static_cast<uint64_t>(i) * kTile] = k1_to_double(s.v);
    Cout[static_cast<uint64_t>(i) * kTile] = fin ? s.front_i : -1;
  }
  if (PUSH) {
    VT fi;
    if constexpr (std::is_same<VT, int32_t>::value) fi = s.v + t1;
    else fi = __dsub_rn(__dadd_rn(s.v, t2), t3);
    // strict pop: earlier candidates stay ahead on f ties (split.cpp:110-113);
    // the -inf sentinel in the slot below the head ends the loop when the
    // deque runs empty
    auto become_front = [&] {  // entry i is the only one left
      s.front_f = fi;
      s.front_l = s.load;
      if (FULL) {
        s.front_i = i;
        s.front_rc = s.rc;
      }
    };
    if constexpr (SAFE) {
      while (s.back_f > fi) {
        s.tail -= kStep;
        s.back_f = ring_at(rf, s.tail - kStep);
      }
      if (s.tail == s.head) become_front();
    } else {
      if (s.back_f > fi) {
        do {
          s.tail -= kStep;
          s.back_f = ring_at(rf, s.tail - kStep);
        } while (s.back_f > fi);
        if (s.tail == s.head) become_front();
      }
    }
    const int ts = s.tail;
    ring_at(rf, ts) = fi;
    ring_at(rl, ts) = s.load;
    if (FULL) {
      ring_at(ri, ts) = i;
      ring_at(rr, ts) = s.rc;
    }
    s.tail += kStep;
    s.back_f = fi;
  }
}

// Demands of tour slots s0..s0+3.  IDENT (identity giant tour, the
// reference's default tour, scendp_main.cpp:222-225): slot s reads customer
// row s, so the four rows are consecutive 128-byte lines (immediate offsets).
template <int SRC, bool IDENT>
__device__ __forceinline__ void k1_demand4(const SplitArgs& a, uint64_t stream,
                                           const uint32_t* tile_base, const uint32_t* s_col,
                                           int s0, uint32_t& d0, uint32_t& d1, uint32_t& d2,
                                           uint32_t& d3) {
  if constexpr (IDENT && SRC == kSrcTiled) {
    const uint32_t* p = tile_base + static_cast<uint64_t>(s0) * kTile;
    d0 = __ldg(p);
    d1 = __ldg(p + kTile);
    d2 = __ldg(p + 2 * kTile);
    d3 = __ldg(p + 3 * kTile);
  } else if constexpr (IDENT && SRC != kSrcTiled) {
    // rows s0..s0+3: consecutive SplitMix64 counters, one multiply per chunk
    const uint64_t ctr = stream + static_cast<uint64_t>(static_cast<uint32_t>(s0)) * kGamma;
    auto val = [&](uint64_t x) {
      if constexpr (SRC == kSrcGenU32) return uniform_draw32(a.gen, x);
      else return draw_value(a.gen, x);
    };
    d0 = val(mix64(ctr));
    d1 = val(mix64(ctr + kGamma));
    d2 = val(mix64(ctr + 2 * kGamma));
    d3 = val(mix64(ctr + 3 * kGamma));
  } else {
    uint4 c;
    if constexpr (IDENT) c = make_uint4(s0, s0 + 1, s0 + 2, s0 + 3);
    else c = *reinterpret_cast<const uint4*>(s_col + s0);
    d0 = demand_at(a, SRC, stream, tile_base, c.x);
    d1 = demand_at(a, SRC, stream, tile_base, c.y);
    d2 = demand_at(a, SRC, stream, tile_base, c.z);
    d3 = demand_at(a, SRC, stream, tile_base, c.w);
  }
}

template <bool FULL, int SRC, bool INTV, bool IDENT>
__global__ void __launch_bounds__(kK1Threads)
split_linear_kernel(SplitArgs a) {
  using VT = typename std::conditional<INTV, int32_t, double>::type;
  constexpr int T = kK1Threads;
  extern __shared__ __align__(16) char smem[];
  __shared__ unsigned long long s_agg[kAggSlots];
  const uint32_t k = blockIdx.y;
  const int n = a.n;
  const int npad = a.npad;  // multiple of 4, >= n + 4
  // chunked tour tables, slot s = position s+1: col | t0..t3
  uint32_t* s_col = reinterpret_cast<uint32_t*>(smem);
  VT* s_tab = reinterpret_cast<VT*>(s_col + (IDENT ? 0 : npad));  // IDENT: no column table
  constexpr int ntab = INTV ? 2 : 4;
  {
    const uint32_t* gcol = a.ccol + static_cast<uint64_t>(k) * npad;
    if (!IDENT) for (int x = threadIdx.x; x < npad; x += T) s_col[x] = gcol[x];
    if (INTV) {
      const int32_t* g = a.itab + static_cast<uint64_t>(k) * 2 * npad;
      for (int x = threadIdx.x; x < 2 * npad; x += T) reinterpret_cast<int32_t*>(s_tab)[x] = g[x];
    } else {
      const double* g = a.dtab + static_cast<uint64_t>(k) * 4 * npad;
      for (int x = threadIdx.x; x < 4 * npad; x += T) reinterpret_cast<double*>(s_tab)[x] = g[x];
    }
  }
  const int tid = threadIdx.x;
  VT* rf = reinterpret_cast<VT*>(s_tab + ntab * npad) + tid;                 // [kRing][T]
  uint32_t* rl = reinterpret_cast<uint32_t*>(rf - tid + kRingSpan) + tid;   // [kRing][T]
  int32_t* ri = reinterpret_cast<int32_t*>(rl - tid + kRingSpan) + tid;     // FULL
  int32_t* rr = ri + kRingSpan;                                             // FULL
  agg_cta_init(s_agg);
  __syncthreads();

  const uint64_t wl = blockIdx.x * static_cast<uint64_t>(T) + tid;  // wave-local
  const bool active = wl < a.m_wave;
  const uint64_t w = a.w_base + wl;                                  // call-level
  uint32_t Qc = static_cast<uint32_t>(a.Q);  // host guarantees Q < 2^31
  // keep Q in a register (opaque to the compiler): otherwise it is re-read
  // from the constant bank at every comparison, one issue slot each
  Qc += static_cast<uint32_t>(a.m_total >> 62);  // + 0, but not provably so

  K1State<VT> s;
  bool ok = true;
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
    // p = 0: f(0) = (0.0 + c(0, s_1)) - dist[1]
    s.front_f = INTV ? static_cast<VT>(a.f0i[k]) : static_cast<VT>(a.f0d[k]);
    s.back_f = s.front_f;
    s.front_l = 0u;
    s.front_i = 0;
    s.front_rc = 0;
    s.rc = 0;
    s.v = VT(0);
    s.load = 0u;
    // slot 0: -inf sentinel (always the slot below the head); slot 1: p = 0
    s.head = kStep;
    s.tail = 2 * kStep;
    rf[0] = k1_neg_inf<VT>();
    ring_at(rf, kStep) = s.front_f;
    ring_at(rl, kStep) = 0u;
    if (FULL) {
      ring_at(ri, kStep) = 0;
      ring_at(rr, kStep) = 0;
    }

    // positions 1..n-1 push; full chunks of 4 first, demands one chunk ahead
    const int npush = n - 1;
    const int nfull = npush >> 2;
    // the ring holds the sentinel + at most kRing-1 entries, so a push needs
    // <= kRing-2 live entries; a chunk pushes 4, hence <= kRing-5 at its start
    // -- otherwise the scenario takes the generic path
    constexpr int kChunkRoom = (kRing - 5) * kStep;
    auto chunk = [&](int s0, uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3) {
      // position constants for the chunk, loaded up front (latency hidden
      // behind the first steps): int32 A/B as two 128-bit loads, fp64
      // (dist, ret, c0, dist_next) interleaved per position, eight loads
      VT t0[4], t1[4], t2[4], t3[4];
      if constexpr (INTV) {
        const int4 x0 = *reinterpret_cast<const int4*>(s_tab + s0);
        const int4 x1 = *reinterpret_cast<const int4*>(s_tab + npad + s0);
        t0[0] = x0.x; t0[1] = x0.y; t0[2] = x0.z; t0[3] = x0.w;
        t1[0] = x1.x; t1[1] = x1.y; t1[2] = x1.z; t1[3] = x1.w;
#pragma unroll
        for (int j = 0; j < 4; ++j) t2[j] = t3[j] = VT(0);
      } else if constexpr (IDENT) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double2 p = *reinterpret_cast<const double2*>(s_tab + 4 * (s0 + j));
          const double2 q = *reinterpret_cast<const double2*>(s_tab + 4 * (s0 + j) + 2);
          t0[j] = p.x; t1[j] = p.y; t2[j] = q.x; t3[j] = q.y;
        }
      }
      // (fp64 with a column table and two chunks of demands in flight: each
      // position's doubles are loaded just before its step -- 64 -> 54
      // registers, measured 0.45 -> 0.37 ms at C2 with a random tour)
      auto step = [&](auto safe, auto noevict, int j, uint32_t d) {
        constexpr bool kSafe = decltype(safe)::value, kNoEvict = decltype(noevict)::value;
        if constexpr (!INTV && !IDENT) {
          const double2 p = *reinterpret_cast<const double2*>(s_tab + 4 * (s0 + j));
          const double2 q = *reinterpret_cast<const double2*>(s_tab + 4 * (s0 + j) + 2);
          k1_step<VT, FULL, true, kSafe, kNoEvict>(s, s0 + j + 1, d, Qc, p.x, p.y, q.x, q.y, rf, rl,
                                                   ri, rr, Vout, Cout);
        } else {
          k1_step<VT, FULL, true, kSafe, kNoEvict>(s, s0 + j + 1, d, Qc, t0[j], t1[j], t2[j],
                                                   t3[j], rf, rl, ri, rr, Vout, Cout);
        }
      };
      using T_ = std::true_type;
      using F_ = std::false_type;
      // fast form unless a demand of this chunk exceeds Q (window may empty);
      // front_l only grows, so if the chunk's last load stays within Q of
      // the current front no position of the chunk evicts -- decided for
      // the converged lanes together (a warp-uniform branch, no per-position
      // window test; taken for most chunks since evictions are rare)
      if (max(max(d0, d1), max(d2, d3)) <= Qc) {
        // (measured: pays off for the fp64 and full-solution forms; the lean
        // int32 cost-only form is faster with its per-position test)
        constexpr bool kSplitEvict = !std::is_same<VT, int32_t>::value || FULL;
        const uint64_t last = static_cast<uint64_t>(s.load) + d0 + d1 + d2 + d3;
        if (kSplitEvict && __all_sync(__activemask(), last - s.front_l <= Qc)) {
          step(F_{}, T_{}, 0, d0);
          step(F_{}, T_{}, 1, d1);
          step(F_{}, T_{}, 2, d2);
          step(F_{}, T_{}, 3, d3);
        } else {
          step(F_{}, F_{}, 0, d0);
          step(F_{}, F_{}, 1, d1);
          step(F_{}, F_{}, 2, d2);
          step(F_{}, F_{}, 3, d3);
        }
      } else {
        step(T_{}, F_{}, 0, d0);
        step(T_{}, F_{}, 1, d1);
        step(T_{}, F_{}, 2, d2);
        step(T_{}, F_{}, 3, d3);
      }
    };
    // demands PF chunks ahead of the chunk being processed.  PF = 1: pairs of
    // chunks with ping-pong registers (identity int32 tours read consecutive
    // rows and are issue-bound; generated demands are computed, not loaded).
    // PF = 2: a register ring indexed at compile time (the loop body is
    // unrolled over the ring) -- more loads in flight per warp for the
    // latency of out-of-order row gathers (random giant tours) and fp64.
    constexpr int PF = (SRC != kSrcTiled || (IDENT && INTV)) ? 1 : kK1Prefetch;
    if constexpr (PF == 1) {
      uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
      if (nfull > 0) k1_demand4<SRC, IDENT>(a, stream, tile_base, s_col, 0, a0, a1, a2, a3);
      int cidx = 0;
      for (; cidx + 1 < nfull; cidx += 2) {
        const int s0 = cidx * 4;
        if (s.tail - s.head > kChunkRoom) {
          ok = false;
          break;
        }
        k1_demand4<SRC, IDENT>(a, stream, tile_base, s_col, s0 + 4, b0, b1, b2, b3);
        chunk(s0, a0, a1, a2, a3);
        if (s.tail - s.head > kChunkRoom) {
          ok = false;
          break;
        }
        if (cidx + 2 < nfull)
          k1_demand4<SRC, IDENT>(a, stream, tile_base, s_col, s0 + 8, a0, a1, a2, a3);
        chunk(s0 + 4, b0, b1, b2, b3);
      }
      if (ok && cidx < nfull) {
        if (s.tail - s.head > kChunkRoom) ok = false;
        else chunk(cidx * 4, a0, a1, a2, a3);
      }
    } else {
      uint32_t db[PF + 1][4];
#pragma unroll
      for (int j = 0; j <= PF; ++j) db[j][0] = db[j][1] = db[j][2] = db[j][3] = 0u;
#pragma unroll
      for (int j = 0; j < PF; ++j)
        if (j < nfull)
          k1_demand4<SRC, IDENT>(a, stream, tile_base, s_col, 4 * j, db[j][0], db[j][1], db[j][2],
                                 db[j][3]);
      for (int cidx = 0; ok && cidx < nfull; cidx += PF + 1) {
#pragma unroll
        for (int u = 0; u <= PF; ++u) {
          const int cc = cidx + u;
          if (cc >= nfull) break;
          if (s.tail - s.head > kChunkRoom) {
            ok = false;
            break;
          }
          uint32_t(&nb)[4] = db[(u + PF) % (PF + 1)];  // chunk cc + PF's registers
          if (cc + PF < nfull)
            k1_demand4<SRC, IDENT>(a, stream, tile_base, s_col, 4 * (cc + PF), nb[0], nb[1], nb[2],
                                   nb[3]);
          chunk(4 * cc, db[u][0], db[u][1], db[u][2], db[u][3]);
        }
      }
    }
    // remaining pushing positions (< 4), then position n (no push)
    for (int i = nfull * 4 + 1; ok && i <= n; ++i) {
      if (s.tail - s.head > (kRing - 2) * kStep) {
        ok = false;
        break;
      }
      const int sl = i - 1;
      const uint32_t d = demand_at(a, SRC, stream, tile_base, IDENT ? sl : s_col[sl]);
      VT x0, x1, x2 = VT(0), x3 = VT(0);
      if constexpr (INTV) {
        x0 = s_tab[sl];
        x1 = s_tab[npad + sl];
      } else {
        x0 = s_tab[4 * sl];
        x1 = s_tab[4 * sl + 1];
        x2 = s_tab[4 * sl + 2];
        x3 = s_tab[4 * sl + 3];
      }
      if (i < n) k1_step<VT, FULL, true>(s, i, d, Qc, x0, x1, x2, x3, rf, rl, ri, rr, Vout, Cout);
      else k1_step<VT, FULL, false>(s, i, d, Qc, x0, x1, x2, x3, rf, rl, ri, rr, Vout, Cout);
    }
    if (!ok) {
      push_overflow(a, k, wl);
    } else {
      const double vd = k1_to_double(s.v);
      if (a.totals) a.totals[static_cast<uint64_t>(k) * a.m_total + w] = vd;
      if (FULL) {
        const bool fin = vd < kInfD;
        a.route_count[w] = fin ? s.rc : 0;
        a.feasible[w] = fin ? 1 : 0;
      }
    }
  }
  const double vout = active && ok ? k1_to_double(s.v) : 0.0;
  __syncwarp();
  agg_warp_add(s_agg, agg_pieces(vout, true), active && ok);
  __syncthreads();
  agg_cta_flush(s_agg, a.agg + static_cast<uint64_t>(k) * kAggWords);
}
