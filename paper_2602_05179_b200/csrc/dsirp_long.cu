// dsirp_long.cu -- K3 for horizons above 32 (the register-resident sparse
// frontier of dsirp_kernels.cuh holds at most 33 slots): the reference's own
// dense forward pass (forward_pass, oudp.cpp:40-87), pick_terminal (94-106)
// and assemble_schedule (108-132), one thread per (customer, scenario) unit.
//
// Per thread: frontiers a, b over states 0..U (fp64) and, for schedules, the
// backpointers [H][U+1] (pred | deliver << 16 | option << 17, the
// reference's packing), all in global scratch interleaved across the grid
// ([element][thread]: the lanes of a warp sweep the states together, so the
// accesses coalesce).  The grid is sized to the scratch budget and walks the
// units with a grid stride.  Work per unit: H * ((U+1) + R*U) candidates --
// the reference's dense scan; this path exists for completeness (horizons
// the reference accepts), the BASELINE shapes (H = 6) never take it.
#include "common.cuh"
#include "internal.hpp"
#include "dsirp_kernels.cuh"

namespace scendp_dsirp {
namespace {

template <typename T>
struct Plane {
  T* p;
  uint64_t s;  // grid threads
  __device__ __forceinline__ T& operator[](uint64_t i) const { return p[i * s]; }
};

template <bool FULL>
__global__ void __launch_bounds__(128)
dsirp_dense_kernel(DsirpArgs a, char* scratch, uint32_t max_states) {
  const uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t S = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t plane = static_cast<uint64_t>(max_states) * S;
  double* base = reinterpret_cast<double*>(scratch);
  Plane<double> fa{base + g, S}, fb{base + plane + g, S};
  const Plane<uint32_t> bp{reinterpret_cast<uint32_t*>(base + 2 * plane) + g, S};
  const uint64_t items = static_cast<uint64_t>(a.nc) * a.m_wave;
  for (uint64_t item = g; item < items; item += S) {
    const uint32_t c = static_cast<uint32_t>(item / a.m_wave);
    const uint64_t wl = item % a.m_wave, w = a.w_base + wl;
    const CustDev cd = a.cust[c];
    const int U = cd.U, H = cd.H, R = cd.R, states = U + 1;
    const double* fixed = a.pool + cd.off_fixed;
    const double* unit = a.pool + cd.off_unit;
    const double* dtable = a.pool + cd.off_dtable;
    const double* htable = a.pool + cd.off_htable;
    const bool dtab = cd.del_tab != 0, htab = cd.hold_tab != 0;
    auto hold = [&](int j, int s) -> double {  // oudp.hpp:58-62
      if (htab) return __ldg(htable + j);
      return __dadd_rn(__dmul_rn(cd.h, static_cast<double>(j)), __dmul_rn(cd.rh, static_cast<double>(s)));
    };
    const uint64_t row0 = static_cast<uint64_t>(c) * H;
    const uint32_t* tile = a.tiled ? a.tiled + ((wl >> 5) * a.rows + row0) * kTile + (wl & 31) : nullptr;
    const uint64_t stream = a.tiled ? 0 : derive_stream(a.gen.seed, kStreamScenario, a.gen.first_index + wl);
    auto demand = [&](int t) -> int {
      return static_cast<int>(tile ? __ldg(tile + static_cast<uint64_t>(t) * kTile)
                                   : draw_counter(a.gen, stream, row0 + t));
    };
    Plane<double> A = fa, B = fb;
    for (int i = 0; i < states; ++i) A[i] = kInfD;
    A[cd.I0] = 0.0;
    for (int t = 0; t < H; ++t) {
      const int d = demand(t);
      for (int i = 0; i < states; ++i) {
        B[i] = kInfD;
        if (FULL) bp[static_cast<uint64_t>(t) * max_states + i] = 0u;
      }
      // no delivery: F(t, 0, 0) = 0
      for (int i = 0; i < states; ++i) {
        const double vi = A[i];
        if (!(vi < kInfD)) continue;
        const int j = max(0, i - d), s = max(0, d - i);
        const double cand = __dadd_rn(vi, __dadd_rn(0.0, hold(j, s)));
        if (cand < B[j]) {
          B[j] = cand;
          if (FULL) bp[static_cast<uint64_t>(t) * max_states + j] = static_cast<uint32_t>(i);
        }
      }
      // delivery up to U: options ascending, states ascending
      const int j1 = max(0, U - d), s1 = max(0, d - U);
      const double hold1 = hold(j1, s1);
      for (int r = 0; r < R; ++r) {
        const double fx = dtab ? 0.0 : fixed[t * R + r];
        const double un = dtab ? 0.0 : unit[t * R + r];
        for (int i = 0; i < U; ++i) {
          const double vi = A[i];
          if (!(vi < kInfD)) continue;
          const int q = U - i;
          const double F = dtab ? __ldg(dtable + static_cast<uint64_t>(t) * states + q)
                                : __dadd_rn(fx, __dmul_rn(un, static_cast<double>(q)));
          const double cand = __dadd_rn(vi, __dadd_rn(F, hold1));
          if (cand < B[j1]) {
            B[j1] = cand;
            if (FULL)
              bp[static_cast<uint64_t>(t) * max_states + j1] =
                  static_cast<uint32_t>(i) | (1u << 16) | (static_cast<uint32_t>(r) << 17);
          }
        }
      }
      const Plane<double> tmp = A;
      A = B;
      B = tmp;
    }
    // pick_terminal: smallest state with the minimal value (strict <)
    double total = kInfD;
    int ts = -1;
    for (int j = 0; j < states; ++j) {
      const double v = A[j];
      if (v < total) {
        total = v;
        ts = j;
      }
    }
    const bool ok = ts >= 0;  // else the reference's logic_error: evaluated = 0
    if (a.totals) a.totals[static_cast<uint64_t>(c) * a.tot_stride + w] = total;
    if (a.evaluated) a.evaluated[static_cast<uint64_t>(c) * a.ev_stride + w] = ok ? 1 : 0;
    if (FULL) {
      // assemble_schedule: backtrack, then quantities forward (tiled outputs)
      const uint64_t tiles = a.sched_tiles;
      const uint64_t ob = ((static_cast<uint64_t>(c) * tiles + (w >> 5)) * H) * kTile + (w & 31);
      int j = ts;
      for (int t = H - 1; t >= 0; --t) {
        const uint32_t e = ok ? bp[static_cast<uint64_t>(t) * max_states + j] : 0u;
        const bool z = (e >> 16) & 1u;
        a.end_inventory[ob + t * kTile] = ok ? j : 0;
        a.deliver[ob + t * kTile] = z ? 1 : 0;
        a.route_option[ob + t * kTile] = z ? static_cast<int32_t>(e >> 17) : 0;
        j = static_cast<int>(e & 0xffffu);
      }
      int inv = cd.I0;
      for (int t = 0; t < H; ++t) {
        const bool z = a.deliver[ob + t * kTile] != 0;
        a.quantity[ob + t * kTile] = z ? U - inv : 0;
        inv = a.end_inventory[ob + t * kTile];
      }
    }
    agg_item_global(a.agg + static_cast<uint64_t>(c) * kAggWords, total, ok);
  }
}

}  // namespace

void launch_long(scendp_ctx* ctx, const DsirpArgs& a, bool full, int max_u, int H) {
  const uint64_t items = static_cast<uint64_t>(a.nc) * a.m_wave;
  if (items == 0) return;
  const uint32_t max_states = static_cast<uint32_t>(max_u) + 1;
  const uint64_t per_thread = static_cast<uint64_t>(max_states) *
                              (2 * sizeof(double) + (full ? static_cast<uint64_t>(H) * 4 : 0));
  // as many threads as 512 MB of scratch allows, at least one warp, in
  // CTAs of 128 (or of one warp when fewer than 128 fit)
  constexpr uint64_t kBudget = 512ull << 20;
  if (per_thread > (16ull << 30) / 32)
    scendp_host::fail(SCENDP_ERR_UNSUPPORTED,
                      "dsirp: capacity x horizon too large for the dense long-horizon path");
  uint64_t threads = std::max<uint64_t>(32, kBudget / per_thread);
  threads = std::min<uint64_t>(threads, (items + 31) / 32 * 32);
  threads = std::min<uint64_t>(threads, static_cast<uint64_t>(ctx->sm_count) * 2048);
  const unsigned block = threads >= 128 ? 128u : 32u;
  const unsigned blocks = static_cast<unsigned>(std::max<uint64_t>(1, threads / block));
  const uint64_t grid_threads = static_cast<uint64_t>(blocks) * block;
  char* scratch = static_cast<char*>(
      ctx->scratch_get(scendp_host::kScrLongHorizon, grid_threads * per_thread + 16));
  const int tok = ctx->timing_begin(0);
  if (full) dsirp_dense_kernel<true><<<blocks, block, 0, ctx->stream>>>(a, scratch, max_states);
  else dsirp_dense_kernel<false><<<blocks, block, 0, ctx->stream>>>(a, scratch, max_states);
  scendp_host::cuda_check(cudaGetLastError(), "dsirp dense kernel launch");
  ctx->timing_end(tok);
  ctx->count_launch();
}

}  // namespace scendp_dsirp
