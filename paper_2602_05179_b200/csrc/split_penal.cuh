// split_penal.cuh -- K2-int: penalized split in O(n), exact integer path.
// Included by split.cu (shares SplitArgs / demand_at / push_overflow and the
// K1 helpers).  Reference: split_core_quadratic, proj/src/split.cpp:45-75.
//
// The reference scans every predecessor p < i:
//   cand(p) = ((f(p) + dist_i) + ret_i) [+ beta * (L_i - L_p - Q) if > 0]
// and keeps the first strict minimum.  When every tour cost and beta are
// integers and all sums stay below 2^29 (host- and per-scenario-checked),
// each of those fp64 operations is exact, so
//   p in the window A = {L_i - L_p <= Q}:   cand = f(p) + (dist_i + ret_i)
//   p before it     B = {L_i - L_p >  Q}:   cand = g(p) + (dist_i + ret_i)
//                                                 + beta (L_i - Q),
//   g(p) = f(p) - beta L_p.
// A is a suffix [lo, i) of positions and B the complementary prefix [0, lo),
// so
//   min over A = the monotone-deque front of K1 (earliest minimal f), and
//   min over B = PM(lo-1), the prefix minimum of g up to lo-1 (earliest
//                minimal g), recorded for every position when it is pushed;
// on equal candidates B wins because all of its indices precede A's --
// exactly the reference's first strict minimum over p = 0..i-1.  Penalized
// mode never produces +inf (every p is admissible), so no masking is needed.
//
// Per thread: the deque ring (f, position) and a position ring holding
// (-L_p mod 2^16, PM(p)) for p in [lo-1, i]; per position the window start
// advances with one shared load per step and the B candidate is one more
// load.  Ring counters are byte offsets of 2-byte slots, masked on access
// (see kH below); 16-bit loads and positions keep the CTA at 6 per SM
// (host: Q < 2^15, so every tested window difference <= 2Q fits).  The kernel
// assumes d_i <= Q (the window never empties, so the deque is never empty
// after the front evictions); a larger demand, a window longer than the
// position ring, a deque overflow or a load beyond the exact int32 range
// sends the scenario to the generic kernel (its O(n) form of the same
// decomposition, or the fp64 quadratic form when the range is exceeded).
#pragma once

constexpr int kPenThreads = 128;
constexpr int kPosRing = 32;                  // positions per thread
// Ring counters are byte offsets of 2-byte slots (slot * 2T): 2-byte
// elements (loads mod 2^16, deque positions) sit at (c & mask), 4-byte ones
// at (c & mask) << 1 (one LOP3 + LEA either way).  Shared memory per thread:
// deque 16 x (4 + 2) B, positions 32 x (2 + 4) B = 288 B (6 CTAs/SM) -- the
// kernel is latency-bound, so occupancy is worth the narrower slots.
constexpr int kH = kPenThreads * 2;           // bytes per 2-byte slot (all threads)
constexpr int kDqMaskH = kRing * kH - 1;
constexpr int kPosMaskH = kPosRing * kH - 1;
constexpr int32_t kPenInf = 0x7fffffff;

template <typename E>
__device__ __forceinline__ E& at16(E* base, int c, int mask) {  // 2-byte element
  return *reinterpret_cast<E*>(reinterpret_cast<char*>(base) + (c & mask));
}
template <typename E>
__device__ __forceinline__ E& at32(E* base, int c, int mask) {  // 4-byte element
  return *reinterpret_cast<E*>(reinterpret_cast<char*>(base) + ((c & mask) << 1));
}

// Host side: bytes of the K2-int rings per thread (split.cu sizes the CTA).
__host__ __device__ constexpr int penal_ring_bytes(bool full) {
  return kRing * (4 + 2 + (full ? 4 : 0)) + kPosRing * (2 + 4 + (full ? 8 : 0));
}

template <bool FULL, int SRC, bool IDENT>
__global__ void __launch_bounds__(kPenThreads)
split_penal_kernel(SplitArgs a) {
  constexpr int T = kPenThreads;
  extern __shared__ __align__(16) char smem[];
  __shared__ unsigned long long s_agg[kAggSlots];
  const uint32_t k = blockIdx.y;
  const int n = a.n;
  const int npad = a.npad;
  const int tid = threadIdx.x;
  // thread-minor rings, 4-byte arrays first: deque f [| rc], positions PM
  // [| PM index | PM rc]; then the 2-byte arrays: deque positions, loads
  int32_t* dq_f = reinterpret_cast<int32_t*>(smem) + tid;
  int32_t* dq_r = dq_f + kRing * T;                                            // FULL
  int32_t* ps_pm = dq_f + (FULL ? 2 : 1) * kRing * T;
  int32_t* ps_pi = ps_pm + kPosRing * T;                                       // FULL
  int32_t* ps_pr = ps_pi + kPosRing * T;                                       // FULL
  uint16_t* dq_p = reinterpret_cast<uint16_t*>(ps_pm - tid + (FULL ? 3 : 1) * kPosRing * T) + tid;
  uint16_t* ps_l = dq_p + kRing * T;
  uint32_t* s_col = reinterpret_cast<uint32_t*>(smem + T * penal_ring_bytes(FULL));
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

  const uint64_t wl = blockIdx.x * static_cast<uint64_t>(T) + tid;
  const bool active = wl < a.m_wave;
  const uint64_t w = a.w_base + wl;
  uint32_t Qc = static_cast<uint32_t>(a.Q);  // host: Q < 2^15 (16-bit window differences)
  Qc += static_cast<uint32_t>(a.m_total >> 62);  // + 0, keeps Q in a register
  const int32_t beta = static_cast<int32_t>(a.beta);
  const uint32_t lmax = a.pen_lmax;  // loads above this leave the exact range

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
    ps_l[0] = 0;  // -L_0 mod 2^16
    ps_pm[0] = f0;
    if (FULL) {
      ps_pi[0] = 0;
      ps_pr[0] = 0;
    }
    // deque: -inf sentinel in slot 0, entry p = 0 in slot 1 (K1 layout)
    dq_f[0] = INT32_MIN;
    dq_f[T] = f0;
    dq_p[T] = 0;
    if (FULL) dq_r[T] = 0;
    int head = kH, tail = 2 * kH;       // deque slot counters
    int32_t front_f = f0, back_f = f0;
    int front_p = 0;                    // position of the deque front
    int32_t front_rc = 0;
    int lo_c = 0;                       // window start lo, as a position counter (lo * kH)
    int32_t bmin = kPenInf;             // PM(lo - 1); kPenInf while lo == 0
    int32_t bidx = -1, brc = 0;
    int32_t pm = f0, pm_i = 0, pm_rc = 0;  // running prefix minimum of g
    uint32_t load = 0;
    // window test on 16-bit loads: exact, every tested difference is <= 2Q
    // (the ring holds -L mod 2^16, so the test is one add and one mask)
    auto out_of_window = [&](int c) {
      const uint32_t nl16 = at16(ps_l, c, kPosMaskH);  // zero-extended
      return ((load + nl16) & 0xffffu) > Qc;
    };

    // one DP position (i_c = i * kH); ring capacities are checked per chunk
    // by the caller (room for the chunk's pushes)
    auto step = [&](int i, int i_c, uint32_t d, int32_t Ai, int32_t Bi, auto push_tag) {
      constexpr bool PUSH = decltype(push_tag)::value;
      load += d;
      // the window start advances past positions whose route (p, i]
      // overflows; d_i <= Q keeps p = i-1 inside, so no bound test is needed
      if (out_of_window(lo_c)) {
        // three window tests per trip, their shared loads issued together (the
        // loop is latency-bound).  Test k (k = 2, 3) may look up to lo+k: it is
        // only used when lo+k-1 left the window, and then lo+k <= i-1 (entry
        // i-1 never leaves when d_i <= Q), so it reads a written slot.
        for (;;) {
          const bool o1 = out_of_window(lo_c + kH), o2 = out_of_window(lo_c + 2 * kH),
                     o3 = out_of_window(lo_c + 3 * kH);
          lo_c += kH;
          if (!o1) break;
          lo_c += kH;
          if (!o2) break;
          lo_c += kH;
          if (!o3) break;
        }
        const int pc = lo_c - kH;  // lo - 1
        bmin = at32(ps_pm, pc, kPosMaskH);
        if (FULL) {
          bidx = at32(ps_pi, pc, kPosMaskH);
          brc = at32(ps_pr, pc, kPosMaskH);
        }
        // deque entries before lo leave from the front (entry i-1 stays);
        // the vacated slot becomes the -inf sentinel below the head
        const int lo = static_cast<int>(static_cast<unsigned>(lo_c) / kH);
        if (front_p < lo) {
          do {
            at32(dq_f, head, kDqMaskH) = INT32_MIN;
            head += kH;
            front_p = at16(dq_p, head, kDqMaskH);
          } while (front_p < lo);
          front_f = at32(dq_f, head, kDqMaskH);
          if (FULL) front_rc = at32(dq_r, head, kDqMaskH);
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
        at16(ps_l, i_c, kPosMaskH) = static_cast<uint16_t>(0u - load);
        at32(ps_pm, i_c, kPosMaskH) = pm;
        if (FULL) {
          at32(ps_pi, i_c, kPosMaskH) = pm_i;
          at32(ps_pr, i_c, kPosMaskH) = pm_rc;
        }
        // strict pop (sentinel-terminated), then push (K1 deque); the deque
        // is non-empty here, so it can only empty by popping
        if (back_f > fi) {
          do {
            tail -= kH;
            back_f = at32(dq_f, tail - kH, kDqMaskH);
          } while (back_f > fi);
          if (tail == head) {
            front_f = fi;
            front_p = i;
            if (FULL) front_rc = rc;
          }
        }
        at32(dq_f, tail, kDqMaskH) = fi;
        at16(dq_p, tail, kDqMaskH) = static_cast<uint16_t>(i);
        if (FULL) at32(dq_r, tail, kDqMaskH) = rc;
        tail += kH;
        back_f = fi;
      }
    };
    // demands of slots s0..s0+3 (slot s = position s+1), loaded one chunk
    // ahead of their use: the gathers hit L2 (C5 reuses each scenario tile
    // for every tour), and without the prefetch every position waits on one
    auto load4 = [&](int s0, uint32_t (&dd)[4]) {
      // the column table is padded (npad >= n + 4, multiple of 4): one
      // 128-bit load for the chunk's rows
      uint4 cr = make_uint4(s0, s0 + 1, s0 + 2, s0 + 3);
      if (!IDENT) cr = *reinterpret_cast<const uint4*>(s_col + s0);
      const uint32_t rows[4] = {cr.x, cr.y, cr.z, cr.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        dd[j] = s0 + j < n ? demand_at(a, SRC, stream, tile_base, rows[j]) : 0u;
    };
    // tour constants of slots s0..s0+3 (A = dist+ret, B = c0 - dist_next):
    // two 128-bit broadcast loads per chunk
    auto tab4 = [&](int s0, int4& A4, int4& B4) {
      A4 = *reinterpret_cast<const int4*>(s_tab + s0);
      B4 = *reinterpret_cast<const int4*>(s_tab + npad + s0);
    };
    using Push = std::true_type;
    using Last = std::false_type;
    // room for 4 pushes: the position ring must hold [lo-1, i] for every i
    // of the chunk, the deque its live entries + 4 + the sentinel slot
    auto room = [&](int s0) {
      return (s0 + 4) * kH - lo_c <= (kPosRing - 2) * kH &&
             (tail - head) + 4 * kH <= (kRing - 1) * kH;
    };
    // positions 1..n-1 push; full chunks of 4 first, demands one chunk ahead
    const int npush = n - 1;
    uint32_t dc[4], dn[4] = {0u, 0u, 0u, 0u};
    load4(0, dc);
    int s0 = 0;
    for (; s0 + 4 <= npush; s0 += 4) {
      if (s0 + 4 < n) load4(s0 + 4, dn);
      // a demand above Q would empty the window: generic path
      if (max(max(dc[0], dc[1]), max(dc[2], dc[3])) > Qc || !room(s0)) {
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
    // the remaining (< 4) pushing positions and position n (no push); dc
    // holds the demands of slots s0..s0+3
    if (ok) {
      if (max(max(dc[0], dc[1]), max(dc[2], dc[3])) > Qc || !room(s0)) {
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
  __syncthreads();
  agg_cta_flush(s_agg, a.agg + static_cast<uint64_t>(k) * kAggWords);
}
