// split_linear.cuh -- K1: hard capacities, O(n) monotone deque
// (reference split_core_linear, proj/src/split.cpp:77-118).  Included by
// split.cu (shares SplitArgs / demand_at / push_overflow).
//
// The kernel is issue-bound (its DRAM traffic equals the algorithmic 4n+8
// bytes per scenario), so the step is written for instruction count:
//  * int32 tour constants arrive as 128-bit broadcast loads once per 4
//    positions (chunked SoA tables in shared memory), fp64 ones per position;
//  * the deque's front entry (f, load, idx, routes) and back f-value live in
//    registers; the per-thread ring in shared memory (not circular, ends
//    addressed by 32-bit shared pointers, see K1Ring) is read only when an
//    end moves (eviction / pop) and written once per push;
//  * the deque is never empty at the start of a position (position i-1 was
//    just pushed) and, unless d_i > Q, entry i-1 survives the eviction, so
//    the common path carries no emptiness tests: the rare "window emptied"
//    and "popped empty" cases are handled inside the eviction / pop bodies;
//  * ring room is checked once per chunk (k1_room: compaction, else the
//    scenario is handed off), and the window test is skipped for a whole
//    chunk when a warp vote proves that no lane evicts.
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
// CTA size: 128 for the int32 path; 256 for fp64, whose per-CTA tour table
// (32 B per position) then costs half the shared memory per warp -- 40
// instead of 32 warps per SM (C2 float 0.327 -> 0.306 ms; the int32 forms
// gain nothing, the random-tour one loses: 0.247 -> 0.261 ms)
__host__ __device__ constexpr int k1_threads(bool intv) { return intv ? 128 : 256; }
constexpr int kK1Prefetch = 2;            // demand chunks in flight ahead
// Deque slots per thread (sentinel included; any count -- the ring is not
// circular).  Identity tours: 12.  At C2 the deque holds <= 6 entries at a
// chunk start (simulated over 2000 scenarios), so 12 slots keep the 4-push
// path and let 16 instead of 12 CTAs share an SM (latency of the demand
// loads: 0.238 -> 0.227 ms; 11 slots: same, 10: hand-offs).  Column-table
// (random) tours keep longer deques: 16 (12 hands off at C2).
__host__ __device__ constexpr int k1_ring(bool ident) { return ident ? 12 : 16; }
// bytes between a thread's consecutive ring slots (4-byte planes, T threads)
// and per ring plane
template <int T>
constexpr int kStepOf = T * 4;
template <int RING, int T>
constexpr int kPlaneOf = RING * kStepOf<T>;

// The deque ring.  Every field is a plane of 4-byte slots, thread-minor
// ([slot][thread], bank-conflict-free): f (int32, or the low word of the
// fp64 value), f's high word (fp64 only), load, and for full solutions the
// predecessor index and route count.  The deque's ends are 32-bit shared-
// memory addresses of f-plane slots of this thread, so an access is one
// LDS/STS with an immediate plane offset -- no wrap mask, no base add, and
// one register per end (generic pointers would take two).  The ring is not
// circular: when a chunk's pushes would run past the last slot, the few live
// entries move back to the bottom (k1_room); the front end advances only by
// evictions, so that is rare.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int OFF>
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF));
  return v;
}
template <int OFF>
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0+%1], %2;" ::"r"(a), "n"(OFF), "r"(v));
}

template <typename VT, int RING, int T>
struct K1Ring {
  static constexpr int kPlane = kPlaneOf<RING, T>;
  static constexpr bool kInt = std::is_same<VT, int32_t>::value;
  static constexpr int kHi = 1;            // fp64 high word
  static constexpr int kL = kInt ? 1 : 2;  // load
  static constexpr int kI = kL + 1, kR = kL + 2;  // FULL
  static __device__ __forceinline__ VT f(uint32_t p) {
    if constexpr (kInt) return static_cast<int32_t>(lds32<0>(p));
    else return __hiloint2double(lds32<kHi * kPlane>(p), lds32<0>(p));
  }
  static __device__ __forceinline__ void set_f(uint32_t p, VT v) {
    if constexpr (kInt) {
      sts32<0>(p, static_cast<uint32_t>(v));
    } else {
      sts32<0>(p, static_cast<uint32_t>(__double2loint(v)));
      sts32<kHi * kPlane>(p, static_cast<uint32_t>(__double2hiint(v)));
    }
  }
  static __device__ __forceinline__ uint32_t l(uint32_t p) { return lds32<kL * kPlane>(p); }
  static __device__ __forceinline__ void set_l(uint32_t p, uint32_t v) { sts32<kL * kPlane>(p, v); }
  static __device__ __forceinline__ int32_t idx(uint32_t p) { return static_cast<int32_t>(lds32<kI * kPlane>(p)); }
  static __device__ __forceinline__ void set_idx(uint32_t p, int32_t v) { sts32<kI * kPlane>(p, static_cast<uint32_t>(v)); }
  static __device__ __forceinline__ int32_t rc(uint32_t p) { return static_cast<int32_t>(lds32<kR * kPlane>(p)); }
  static __device__ __forceinline__ void set_rc(uint32_t p, int32_t v) { sts32<kR * kPlane>(p, static_cast<uint32_t>(v)); }
  // copy every plane of slot src to slot dst
  template <bool FULL>
  static __device__ __forceinline__ void move(uint32_t dst, uint32_t src) {
    sts32<0>(dst, lds32<0>(src));
    if constexpr (!kInt) sts32<kHi * kPlane>(dst, lds32<kHi * kPlane>(src));
    set_l(dst, l(src));
    if constexpr (FULL) {
      set_idx(dst, idx(src));
      set_rc(dst, rc(src));
    }
  }
};

template <typename VT>
struct K1State {
  uint32_t load;
  uint32_t head;  // f-plane slot of the deque front (the slot below holds -inf)
  uint32_t tail;  // first free slot
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

// Make room for `pushes` more entries below the ring's end: when the tail
// would run past slot RING-1, move the sentinel and the live entries down
// to slots 0..len (rare: the head advances only by evictions).  Returns
// false when even the compacted deque has no room (the scenario then takes
// the generic path).
template <typename VT, bool FULL, int RING, int T>
__device__ __forceinline__ bool k1_room(K1State<VT>& s, uint32_t base, int pushes) {
  constexpr int kStep = kStepOf<T>;
  if (s.tail + pushes * kStep <= base + kPlaneOf<RING, T>) return true;
  using R = K1Ring<VT, RING, T>;
  const int len = static_cast<int>(s.tail - s.head) / kStep;
  if (len + 1 + pushes > RING) return false;
  uint32_t dst = base + kStep;
  for (uint32_t src = s.head; src < s.tail; src += kStep, dst += kStep)
    R::template move<FULL>(dst, src);
  R::set_f(base, k1_neg_inf<VT>());
  s.head = base + kStep;
  s.tail = dst;
  return true;
}

// One DP position.  PUSH = (i < n).
//
// SAFE = false is the fast form for a position with d_i <= Q (checked per
// chunk): entry i-1, at the back, then survives the eviction, so the window
// never empties and the eviction loop needs no emptiness test; and since the
// deque is non-empty before the pops, it can only become empty by popping,
// so the "popped empty" front update lives inside the (rarer) pop branch.
// SAFE = true handles any d_i (window emptied when d_i > Q).
// NOEVICT (with SAFE = false): the caller proved no eviction can happen at
// this position (see the chunk loop), so the window test is skipped.
// The caller guarantees a free slot at the tail (k1_room).
template <typename VT, bool FULL, bool PUSH, bool SAFE, bool NOEVICT, int RING, int T>
__device__ __forceinline__ void k1_step(K1State<VT>& s, int i, uint32_t d, uint32_t Qc, VT t0,
                                        VT t1, VT t2, VT t3, double* Vout, int32_t* Cout) {
  using R = K1Ring<VT, RING, T>;
  constexpr int kStep = kStepOf<T>;
  s.load += d;
  // evict predecessors whose route (p, i] exceeds Q (split.cpp:93-96); the
  // evicted slot becomes the -inf sentinel below the new head
  if constexpr (SAFE) {
    if (d > Qc) {
      // every route into i carries d_i > Q: the window empties.  Decided on
      // d itself -- the u32 difference load - front_l wraps once d_i >=
      // 2^32 - Q (loads are int64 in the reference, split.cpp:93); with
      // d_i <= Q every window difference is < 2Q < 2^32 and exact mod 2^32
      R::set_f(s.tail - kStep, k1_neg_inf<VT>());
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
      R::set_f(s.head, k1_neg_inf<VT>());
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
      s.front_f = R::f(s.head);
      s.front_l = R::l(s.head);
      if (FULL) {
        s.front_i = R::idx(s.head);
        s.front_rc = R::rc(s.head);
      }
    }
  } else if constexpr (!NOEVICT) {
    if (s.load - s.front_l > Qc) {
      do {
        R::set_f(s.head, k1_neg_inf<VT>());
        s.head += kStep;
        s.front_l = R::l(s.head);
      } while (s.load - s.front_l > Qc);
      s.front_f = R::f(s.head);
      if (FULL) {
        s.front_i = R::idx(s.head);
        s.front_rc = R::rc(s.head);
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
        s.back_f = R::f(s.tail - kStep);
      }
      if (s.tail == s.head) become_front();
    } else {
      if (s.back_f > fi) {
        do {
          s.tail -= kStep;
          s.back_f = R::f(s.tail - kStep);
        } while (s.back_f > fi);
        if (s.tail == s.head) become_front();
      }
    }
    R::set_f(s.tail, fi);
    R::set_l(s.tail, s.load);
    if (FULL) {
      R::set_idx(s.tail, i);
      R::set_rc(s.tail, s.rc);
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
    auto val = [&](uint64_t z) {
      if constexpr (SRC == kSrcGenU32) return mix_uniform32(a.gen, z);
      else return draw_value(a.gen, mix64(z));
    };
    d0 = val(ctr);
    d1 = val(ctr + kGamma);
    d2 = val(ctr + 2 * kGamma);
    d3 = val(ctr + 3 * kGamma);
  } else if constexpr (SRC != kSrcTiled) {
    // column-table tour, generated demands: s_col holds row * gamma (u64) per
    // slot, so each counter is one 64-bit add (no per-draw multiply)
    const ulonglong2* g = reinterpret_cast<const ulonglong2*>(s_col) + s0 / 2;
    const ulonglong2 g01 = g[0], g23 = g[1];
    auto val = [&](uint64_t z) {
      if constexpr (SRC == kSrcGenU32) return mix_uniform32(a.gen, z);
      else return draw_value(a.gen, mix64(z));
    };
    d0 = val(stream + g01.x);
    d1 = val(stream + g01.y);
    d2 = val(stream + g23.x);
    d3 = val(stream + g23.y);
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

template <typename P>
__device__ __forceinline__ double2 ldtab2(const P* p) {
  return *reinterpret_cast<const double2*>(p);
}
template <bool FULL, int SRC, bool INTV, bool IDENT>
__global__ void __launch_bounds__(k1_threads(INTV))
split_linear_kernel(SplitArgs a) {
  // the hand-off pass (launched programmatically dependent, see
  // launch_overflow_pass) may start its CTAs now; they wait for this grid
  asm volatile("griddepcontrol.launch_dependents;");
  using VT = typename std::conditional<INTV, int32_t, double>::type;
  constexpr int T = k1_threads(INTV);
  constexpr int kStep = kStepOf<T>;
  constexpr int RING = k1_ring(IDENT);
  extern __shared__ __align__(16) char smem[];
  __shared__ unsigned long long s_agg[kAggSlots];
  const uint32_t k = blockIdx.y;
  const int n = a.n;
  const int npad = a.npad;  // multiple of 4, >= n + 4
  // chunked tour tables, slot s = position s+1: col | t0..t3.  The column
  // table holds rows (u32), or for generated demands row * gamma (u64: the
  // generator's counter offset); identity tours have none
  constexpr bool kGam = !IDENT && SRC != kSrcTiled;
  uint32_t* s_col = reinterpret_cast<uint32_t*>(smem);
  VT* s_tab = reinterpret_cast<VT*>(s_col + (IDENT ? 0 : kGam ? 2 * npad : npad));
  constexpr int ntab = INTV ? 2 : 4;
  // (fp64 tables read through L1 instead of shared memory, for more CTAs:
  // measured slower, C2 float 0.327 -> 0.405 ms)
  const VT* tab = s_tab;
  {
    const uint32_t* gcol = a.ccol + static_cast<uint64_t>(k) * npad;
    if (kGam) {
      for (int x = threadIdx.x; x < npad; x += T)
        reinterpret_cast<uint64_t*>(s_col)[x] = static_cast<uint64_t>(gcol[x]) * kGamma;
    } else if (!IDENT) {
      for (int x = threadIdx.x; x < npad; x += T) s_col[x] = gcol[x];
    }
    if (INTV) {
      const int32_t* g = a.itab + static_cast<uint64_t>(k) * 2 * npad;
      for (int x = threadIdx.x; x < 2 * npad; x += T) reinterpret_cast<int32_t*>(s_tab)[x] = g[x];
    } else {
      const double* g = a.dtab + static_cast<uint64_t>(k) * 4 * npad;
      for (int x = threadIdx.x; x < 4 * npad; x += T) reinterpret_cast<double*>(s_tab)[x] = g[x];
    }
  }
  const int tid = threadIdx.x;
  // this thread's ring: slot 0 of its f plane (planes follow, see K1Ring)
  const uint32_t rbase = smem_addr(s_tab + ntab * npad) + 4 * tid;
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
    using R = K1Ring<VT, RING, T>;
    s.head = rbase + kStep;
    s.tail = rbase + 2 * kStep;
    R::set_f(rbase, k1_neg_inf<VT>());
    R::set_f(s.head, s.front_f);
    R::set_l(s.head, 0u);
    if (FULL) {
      R::set_idx(s.head, 0);
      R::set_rc(s.head, 0);
    }

    // positions 1..n-1 push; full chunks of 4 first, demands one chunk ahead
    const int npush = n - 1;
    const int nfull = npush >> 2;
    // a chunk pushes 4: room for them below the ring's end (compacting the
    // deque when needed), else the scenario takes the generic path
    // (fp64: the common case -- the tail at least 4 slots below the ring's
    // end -- is one compare against a limit kept in a register: C2 float
    // 0.307 -> 0.302 ms; the int32 forms measured slower with it)
    const uint32_t tail_max4 = rbase + kPlaneOf<RING, T> - 4 * kStep;
    auto room4 = [&] {
      if constexpr (!INTV) return s.tail <= tail_max4 || k1_room<VT, FULL, RING, T>(s, rbase, 4);
      else return k1_room<VT, FULL, RING, T>(s, rbase, 4);
    };
    auto chunk = [&](int s0, uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3) {
      // position constants: int32 A/B for the chunk as two 128-bit loads up
      // front (latency hidden behind the first steps); fp64 (dist, ret, c0,
      // dist_next, interleaved) per position just before its step
      VT t0[4], t1[4], t2[4], t3[4];
      if constexpr (INTV) {
        const int4 x0 = *reinterpret_cast<const int4*>(s_tab + s0);
        const int4 x1 = *reinterpret_cast<const int4*>(s_tab + npad + s0);
        t0[0] = x0.x; t0[1] = x0.y; t0[2] = x0.z; t0[3] = x0.w;
        t1[0] = x1.x; t1[1] = x1.y; t1[2] = x1.z; t1[3] = x1.w;
#pragma unroll
        for (int j = 0; j < 4; ++j) t2[j] = t3[j] = VT(0);
      }
      // (fp64 per position: 64 -> 48 registers; measured 0.45 -> 0.37 ms at
      // C2 with a random tour, 0.351 -> 0.328 ms with the identity tour)
      auto step = [&](auto safe, auto noevict, int j, uint32_t d) {
        constexpr bool kSafe = decltype(safe)::value, kNoEvict = decltype(noevict)::value;
        if constexpr (!INTV) {
          const double2 p = ldtab2(tab + 4 * (s0 + j));
          const double2 q = ldtab2(tab + 4 * (s0 + j) + 2);
          k1_step<VT, FULL, true, kSafe, kNoEvict, RING, T>(s, s0 + j + 1, d, Qc, p.x, p.y, q.x, q.y, Vout,
                                                   Cout);
        } else {
          k1_step<VT, FULL, true, kSafe, kNoEvict, RING, T>(s, s0 + j + 1, d, Qc, t0[j], t1[j], t2[j],
                                                   t3[j], Vout, Cout);
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
        // (measured: pays off for every form since the non-circular ring and
        // the 32-bit span -- C2 0.227 -> 0.212 ms, generated 0.415 -> 0.411,
        // generated random tour 0.417 -> 0.406; random tiled tour neutral)
        constexpr bool kSplitEvict = true;
        // the chunk's last window span: (load - front_l) <= Q plus four
        // demands <= Q each, so 32-bit arithmetic is exact while 5Q < 2^32
        // (int32 forms only: C2 0.215 -> 0.212 ms; the fp64 random-tour form
        // measured slower with it)
        bool none;
        if (INTV && Qc < (1u << 29)) {
          none = (s.load - s.front_l) + (d0 + d1 + d2 + d3) <= Qc;
        } else {
          const uint64_t last = static_cast<uint64_t>(s.load) + d0 + d1 + d2 + d3;
          none = last - s.front_l <= Qc;
        }
        if (kSplitEvict && __all_sync(__activemask(), none)) {
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
    // (identity int32 with two chunks in flight measured slower: 0.264 vs
    // 0.238 ms with the 16-slot ring)
    constexpr int PF = (SRC != kSrcTiled || (IDENT && INTV)) ? 1 : kK1Prefetch;
    if constexpr (PF == 1) {
      uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
      if (nfull > 0) k1_demand4<SRC, IDENT>(a, stream, tile_base, s_col, 0, a0, a1, a2, a3);
      int cidx = 0;
      for (; cidx + 1 < nfull; cidx += 2) {
        const int s0 = cidx * 4;
        if constexpr (FULL && IDENT && SRC == kSrcTiled) {
          // rows s0+16 .. s0+23 of this warp's tile into L2 (one bulk
          // prefetch per warp per 8 positions, no registers held).  Full
          // solutions only: C2 full 0.564 -> 0.549 ms; the cost-only form
          // measured slower with it (0.228 -> 0.239 ms)
          if ((tid & 31) == 0 && s0 + 24 <= n)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                             tile_base + static_cast<uint64_t>(s0 + 16) * kTile),
                         "r"(8 * kTile * 4)
                         : "memory");
        }
        if (!room4()) {
          ok = false;
          break;
        }
        k1_demand4<SRC, IDENT>(a, stream, tile_base, s_col, s0 + 4, b0, b1, b2, b3);
        chunk(s0, a0, a1, a2, a3);
        if (!room4()) {
          ok = false;
          break;
        }
        if (cidx + 2 < nfull)
          k1_demand4<SRC, IDENT>(a, stream, tile_base, s_col, s0 + 8, a0, a1, a2, a3);
        chunk(s0 + 4, b0, b1, b2, b3);
      }
      if (ok && cidx < nfull) {
        if (!room4()) ok = false;
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
          if (!room4()) {
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
      if (!k1_room<VT, FULL, RING, T>(s, rbase, 1)) {
        ok = false;
        break;
      }
      const int sl = i - 1;
      uint32_t d;
      if constexpr (kGam) {
        const uint64_t z = stream + reinterpret_cast<const uint64_t*>(s_col)[sl];
        if constexpr (SRC == kSrcGenU32) d = mix_uniform32(a.gen, z);
        else d = draw_value(a.gen, mix64(z));
      } else {
        d = demand_at(a, SRC, stream, tile_base, IDENT ? sl : s_col[sl]);
      }
      VT x0, x1, x2 = VT(0), x3 = VT(0);
      if constexpr (INTV) {
        x0 = s_tab[sl];
        x1 = s_tab[npad + sl];
      } else {
        x0 = tab[4 * sl];
        x1 = tab[4 * sl + 1];
        x2 = tab[4 * sl + 2];
        x3 = tab[4 * sl + 3];
      }
      if (i < n) k1_step<VT, FULL, true, true, false, RING, T>(s, i, d, Qc, x0, x1, x2, x3, Vout, Cout);
      else k1_step<VT, FULL, false, true, false, RING, T>(s, i, d, Qc, x0, x1, x2, x3, Vout, Cout);
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
