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
// A is a suffix of positions and B the complementary prefix, so
//   min over A = the monotone-deque front of K1 (earliest minimal f), and
//   min over B = a running prefix minimum of g (earliest minimal g),
// both maintained in O(1) amortized per position; on equal candidates B wins
// because all of its indices precede A's -- exactly the reference's
// first-strict-minimum over p = 0..i-1.  Penalized mode never produces +inf
// (every p is admissible), so no masking is needed.
//
// Per-thread shared state: the deque ring (K1's, f and position index) and a
// position ring of the last kPosRing positions (f, L) that feeds the prefix
// minimum as positions leave the window.  A window longer than the position
// ring or a deque overflow sends the scenario to the generic kernel's O(n)
// form of the same decomposition; a load that would leave the exact int32
// range sends it to the generic fp64 quadratic form.
#pragma once

constexpr int kPenThreads = 128;
constexpr int kPosRing = 32;  // positions per thread (window length < 32)
constexpr int32_t kPenInf = 0x7fffffff;

template <bool FULL, int SRC, bool IDENT>
__global__ void __launch_bounds__(kPenThreads)
split_penal_kernel(SplitArgs a) {
  constexpr int T = kPenThreads;
  extern __shared__ __align__(16) char smem[];
  __shared__ unsigned long long s_agg[kAggSlots];
  const uint32_t k = blockIdx.y;
  const int n = a.n;
  const int npad = a.npad;
  uint32_t* s_col = reinterpret_cast<uint32_t*>(smem);
  int32_t* s_tab = reinterpret_cast<int32_t*>(s_col + (IDENT ? 0 : npad));  // A | B
  {
    const uint32_t* gcol = a.ccol + static_cast<uint64_t>(k) * npad;
    if (!IDENT)
      for (int x = threadIdx.x; x < npad; x += T) s_col[x] = gcol[x];
    const int32_t* g = a.itab + static_cast<uint64_t>(k) * 2 * npad;
    for (int x = threadIdx.x; x < 2 * npad; x += T) s_tab[x] = g[x];
  }
  const int tid = threadIdx.x;
  // rings, thread-minor: deque [kRing][T] (f, idx), positions [kPosRing][T]
  // (f, L[, rc])
  int32_t* dq_f = s_tab + 2 * npad + tid;
  int32_t* dq_i = dq_f + kRing * T;
  int32_t* ps_f = dq_i + kRing * T;
  uint32_t* ps_l = reinterpret_cast<uint32_t*>(ps_f + kPosRing * T);
  int32_t* ps_r = reinterpret_cast<int32_t*>(ps_l + kPosRing * T);  // FULL
  agg_cta_init(s_agg);
  __syncthreads();

  const uint64_t wl = blockIdx.x * static_cast<uint64_t>(T) + tid;
  const bool active = wl < a.m_wave;
  const uint64_t w = a.w_base + wl;
  uint32_t Qc = static_cast<uint32_t>(a.Q);
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
    // position 0: f(0) = (0.0 + c(0, s_1)) - dist[1], L_0 = 0
    const int32_t f0 = a.f0i[k];
    ps_f[0] = f0;
    ps_l[0] = 0u;
    if (FULL) ps_r[0] = 0;
    // deque: -inf sentinel in slot 0, entry p=0 in slot 1 (K1 layout)
    dq_f[0] = INT32_MIN;
    dq_f[T] = f0;
    dq_i[T] = 0;
    int head = 1, tail = 2;  // slot counters (masked by kRing-1)
    int32_t front_f = f0, front_i = 0, back_f = f0;
    int lo = 0;               // first position inside the window
    int32_t bmin = kPenInf;   // prefix minimum of g over [0, lo)
    int32_t bidx = -1, brc = 0;
    uint32_t load = 0;

    // one DP position; returns false when the scenario must take the generic
    // path (window longer than the position ring, deque overflow)
    auto step = [&](int i, uint32_t d) -> bool {
      const int sl = i - 1;
      const int32_t Ai = s_tab[sl], Bi = s_tab[npad + sl];
      load += d;
      // positions leaving the window join the prefix B (in index order)
      while (lo < i && load - ps_l[(lo & (kPosRing - 1)) * T] > Qc) {
        const int ls = (lo & (kPosRing - 1)) * T;
        const int32_t g = ps_f[ls] - beta * static_cast<int32_t>(ps_l[ls]);
        if (g < bmin) {
          bmin = g;
          bidx = lo;
          if (FULL) brc = ps_r[ls];
        }
        ++lo;
      }
      // deque front leaves with the window; the vacated slot becomes the -inf
      // sentinel below the head (ends the pop loop on an empty deque)
      while (head != tail && front_i < lo) {
        dq_f[(head & (kRing - 1)) * T] = INT32_MIN;
        ++head;
        if (head != tail) {
          const int hs = (head & (kRing - 1)) * T;
          front_f = dq_f[hs];
          front_i = dq_i[hs];
        } else {
          back_f = INT32_MIN;
        }
      }
      // candidates: window A (deque front) and prefix B (prefix minimum)
      const bool hasA = head != tail;
      const int32_t candA = hasA ? front_f + Ai : kPenInf;
      const int32_t candB = bidx >= 0 ? bmin + Ai + beta * static_cast<int32_t>(load - Qc) : kPenInf;
      const bool useB = candB <= candA;  // B's indices come first: ties go to B
      v = useB ? candB : candA;
      const int32_t cut = useB ? bidx : front_i;
      if (FULL) {
        const int32_t frc = useB ? brc : (hasA ? ps_r[(front_i & (kPosRing - 1)) * T] : 0);
        rc = frc + 1;
        Vout[static_cast<uint64_t>(i) * kTile] = static_cast<double>(v);
        Cout[static_cast<uint64_t>(i) * kTile] = cut;
      }
      if (i < n) {
        const int32_t fi = v + Bi;
        // the position ring must hold [lo, i]
        if (i - lo >= kPosRing - 1) return false;
        const int ps = (i & (kPosRing - 1)) * T;
        ps_f[ps] = fi;
        ps_l[ps] = load;
        if (FULL) ps_r[ps] = rc;
        // strict pop (sentinel-terminated), then push (K1 deque)
        while (back_f > fi) {
          --tail;
          back_f = dq_f[((tail - 1) & (kRing - 1)) * T];
        }
        if (tail == head) {
          front_f = fi;
          front_i = i;
        }
        if (tail - head >= kRing - 1) return false;
        const int ts = (tail & (kRing - 1)) * T;
        dq_f[ts] = fi;
        dq_i[ts] = i;
        ++tail;
        back_f = fi;
      }
      return true;
    };
    // demands of slots s0..s0+3 (slot s = position s+1), loaded one chunk
    // ahead of their use: the gathers hit L2 (C5 reuses each scenario tile
    // for every tour), and without the prefetch every position waits on one
    auto load4 = [&](int s0, uint32_t (&dd)[4]) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int sl = s0 + j;
        dd[j] = sl < n ? demand_at(a, SRC, stream, tile_base, IDENT ? sl : s_col[sl]) : 0u;
      }
    };
    uint32_t dc[4], dn[4] = {0u, 0u, 0u, 0u};
    load4(0, dc);
    for (int s0 = 0; s0 < n && ok; s0 += 4) {
      if (s0 + 4 < n) load4(s0 + 4, dn);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = s0 + j + 1;
        if (i <= n && ok) ok = step(i, dc[j]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) dc[j] = dn[j];
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
