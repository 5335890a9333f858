// scengen.cu -- K4 scenario generator + HBM layout conversions.
//
// Reference: generate_scenario_column / generate_scenarios
// (proj/src/scenario.cpp:92-114), DistributionSpec::sample (22-40).
// Column w draws sequentially from SplitMix64(derive_stream(seed,
// kStreamScenario, w)).  For uniform and poisson every value consumes exactly
// one next(), so row r of column w is a pure function of (w, r): the kernel
// is element-parallel and writes the tiled layout with coalesced 128-byte
// rows.  tnormal rejection-samples a variable number of draws per value and
// is generated sequentially per column (one thread per scenario).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

using namespace scendp_dev;
using namespace scendp_host;

namespace {

constexpr int kGenThreads = 256;

// Counter-based kinds: one thread per scenario, loop over rows; a warp writes
// one 128-byte line per row of the tiled layout.
__global__ void __launch_bounds__(kGenThreads)
gen_counter_kernel(GenParams g, uint64_t rows, uint64_t count, uint32_t* out) {
  extern __shared__ double s_cdf[];
  if (g.kind == SCENDP_DIST_POISSON) {
    for (int k = threadIdx.x; k < g.cdf_len; k += blockDim.x) s_cdf[k] = g.cdf[k];
    __syncthreads();
  }
  const uint64_t w = blockIdx.x * uint64_t(kGenThreads) + threadIdx.x;
  if (w >= count) return;
  const uint64_t stream = derive_stream(g.seed, kStreamScenario, g.first_index + w);
  uint32_t* dst = out + (w >> 5) * rows * kTile + (w & 31);
  if (g.kind == SCENDP_DIST_UNIFORM) {
    uint64_t st = stream;
    for (uint64_t r = 0; r < rows; ++r) {
      const uint64_t x = mix64(st);
      st += kGamma;
      dst[r * kTile] = uniform_draw(g, x);
    }
  } else {
    uint64_t st = stream;
    for (uint64_t r = 0; r < rows; ++r) {
      const uint64_t x = mix64(st);
      st += kGamma;
      const double u = static_cast<double>((x >> 11) + 1) * 0x1.0p-53;
      int k = 0;
      while (u > s_cdf[k]) ++k;
      dst[r * kTile] = static_cast<uint32_t>(k);
    }
  }
}

// tnormal (scenario.cpp:30-39): Box-Muller, llround, <= 64 rejections, then
// clamp(llround(mean)).  No FMA contraction (built with -fmad=false).
//
// Exactness by construction.  The reference's value depends on glibc's log
// and cos, which CUDA's libm does not reproduce bit for bit.  Every draw
// therefore also computes an interval certain to contain glibc's
// mean + stddev * z: log and cos are each within 2^-46 relative of the
// device's results (CUDA: <= 1 and 2 ulp; glibc: <= 1 ulp; 2^-46 is 64
// ulp), and the remaining operations (-2 x, sqrt, product, stddev * z,
// mean + ...) are monotone, so directed-rounding bounds carry through.  When
// llround of both ends agree, that integer is the reference's (and the
// rejection decision with it).  A column with any draw whose interval
// straddles a rounding boundary (about 1e-13 per draw) is listed for the
// host, which regenerates that column with the reference's own arithmetic
// (glibc, tnormal_column_host) and writes it over the device's.
__device__ __forceinline__ bool tnormal_draw(double u1, double u2, double mean, double stddev,
                                             long long& r) {
  const double two_pi = 2.0 * 0x1.921fb54442d18p+1;  // 2.0 * std::numbers::pi
  const double L = -2.0 * log(u1);
  const double c = cos(two_pi * u2);
  const double z = sqrt(L) * c;
  r = llround(mean + stddev * z);
  constexpr double e = 0x1p-46;
  const double Slo = __dsqrt_rn(__dmul_rd(L, 1.0 - e)), Shi = __dsqrt_rn(__dmul_ru(L, 1.0 + e));
  const double ce = __dmul_ru(fabs(c), e);
  const double clo = __dsub_rd(c, ce), chi = __dadd_ru(c, ce);
  const double zlo = fmin(fmin(__dmul_rd(Slo, clo), __dmul_rd(Slo, chi)),
                          fmin(__dmul_rd(Shi, clo), __dmul_rd(Shi, chi)));
  const double zhi = fmax(fmax(__dmul_ru(Slo, clo), __dmul_ru(Slo, chi)),
                          fmax(__dmul_ru(Shi, clo), __dmul_ru(Shi, chi)));
  const long long rlo = llround(__dadd_rn(mean, __dmul_rn(stddev, zlo)));
  const long long rhi = llround(__dadd_rn(mean, __dmul_rn(stddev, zhi)));
  return rlo == rhi;
}

__global__ void __launch_bounds__(kGenThreads)
gen_tnormal_kernel(int64_t lo, int64_t hi, double mean, double stddev,
                   uint64_t seed, uint64_t first_index, uint64_t rows,
                   uint64_t count, uint32_t* out, unsigned int* n_amb,
                   unsigned long long* amb, uint32_t amb_cap, uint32_t force_every) {
  const uint64_t w = blockIdx.x * uint64_t(kGenThreads) + threadIdx.x;
  if (w >= count) return;
  uint64_t st = derive_stream(seed, kStreamScenario, first_index + w);
  uint32_t* dst = out + (w >> 5) * rows * kTile + (w & 31);
  // SCENDP_TNORMAL_HOST_EVERY=k (tests): every k-th column takes the host
  // path as if ambiguous
  bool certain = !(force_every && (first_index + w) % force_every == 0);
  for (uint64_t r = 0; r < rows; ++r) {
    uint32_t v = 0;
    bool done = false;
    for (int attempt = 0; attempt < 64 && !done; ++attempt) {
      const uint64_t x1 = mix64(st);
      st += kGamma;
      const uint64_t x2 = mix64(st);
      st += kGamma;
      const double u1 = static_cast<double>((x1 >> 11) + 1) * 0x1.0p-53;
      const double u2 = static_cast<double>((x2 >> 11) + 1) * 0x1.0p-53;
      long long rr;
      certain &= tnormal_draw(u1, u2, mean, stddev, rr);
      if (rr >= lo && rr <= hi) {
        v = static_cast<uint32_t>(rr);
        done = true;
      }
    }
    if (!done) {
      long long rr = llround(mean);
      rr = rr < lo ? lo : (rr > hi ? hi : rr);
      v = static_cast<uint32_t>(rr);
    }
    dst[r * kTile] = v;
  }
  if (!certain) {
    const unsigned int slot = atomicAdd(n_amb, 1u);
    if (slot < amb_cap) amb[slot] = w;
  }
}

// Reference layout [count][rows] -> tiled [count/32][rows][32] (32x32 smem
// transpose, both sides coalesced).  Element type is 4 bytes.
template <typename T, typename S = T>
__global__ void __launch_bounds__(256)
to_tiled_kernel(const S* __restrict__ src, uint64_t rows, uint64_t count,
                T* __restrict__ dst) {
  __shared__ T tile[32][33];
  const uint64_t w0 = blockIdx.x * uint64_t(32);
  const uint64_t r0 = blockIdx.y * uint64_t(32);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int s = ty; s < 32; s += 8) {
    const uint64_t w = w0 + s, r = r0 + tx;
    if (w < count && r < rows) tile[s][tx] = src[w * rows + r];
  }
  __syncthreads();
  for (int rr = ty; rr < 32; rr += 8) {
    const uint64_t r = r0 + rr, w = w0 + tx;
    if (w < count && r < rows) dst[tiled_index(w, r, rows)] = tile[tx][rr];
  }
}

// Tiled [count/32][rows][32] -> reference [count][rows].
template <typename T>
__global__ void __launch_bounds__(256)
from_tiled_kernel(const T* __restrict__ src, uint64_t rows, uint64_t count,
                  T* __restrict__ dst) {
  __shared__ T tile[32][33];
  const uint64_t w0 = blockIdx.x * uint64_t(32);
  const uint64_t r0 = blockIdx.y * uint64_t(32);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int rr = ty; rr < 32; rr += 8) {
    const uint64_t r = r0 + rr, w = w0 + tx;
    if (w < count && r < rows) tile[rr][tx] = src[tiled_index(w, r, rows)];
  }
  __syncthreads();
  for (int s = ty; s < 32; s += 8) {
    const uint64_t w = w0 + s, r = r0 + tx;
    if (w < count && r < rows) dst[w * rows + r] = tile[tx][s];
  }
}

void check_dist(const scendp_dist* d) {
  if (!d) fail(SCENDP_ERR_INVALID_ARGUMENT, "distribution is null");
  if (d->lo > d->hi) fail(SCENDP_ERR_INVALID_ARGUMENT, "distribution bounds: lo > hi");
  if (d->lo < 0)
    fail(SCENDP_ERR_INVALID_ARGUMENT, "demands are nonnegative: lo must be >= 0");
  if (d->hi > 0xffffffffLL)
    fail(SCENDP_ERR_INVALID_ARGUMENT, "demands are u32: hi must be < 2^32");
  if (d->kind == SCENDP_DIST_TNORMAL && !(d->stddev > 0.0))
    fail(SCENDP_ERR_INVALID_ARGUMENT, "truncated normal: std must be > 0");
  if (d->kind == SCENDP_DIST_POISSON) {
    if (!(d->mean > 0.0)) fail(SCENDP_ERR_INVALID_ARGUMENT, "poisson: lambda must be > 0");
    if (d->lo != 0) fail(SCENDP_ERR_INVALID_ARGUMENT, "poisson: lo must be 0");
    if (d->hi > (1 << 20)) fail(SCENDP_ERR_UNSUPPORTED, "poisson: hi must be <= 2^20");
  }
  if (d->kind < 0 || d->kind > 2) fail(SCENDP_ERR_INVALID_ARGUMENT, "unknown distribution kind");
}

}  // namespace

namespace scendp_host {

// Host CDF table, summed in index order; P[hi] = 1.
std::vector<double> poisson_table(double lambda, int64_t hi) {
  std::vector<double> p(static_cast<size_t>(hi) + 1);
  double term = std::exp(-lambda), acc = 0.0;
  for (int64_t k = 0; k <= hi; ++k) {
    if (k > 0) term = term * lambda / static_cast<double>(k);
    acc = acc + term;
    p[k] = acc;
  }
  p[hi] = 1.0;
  return p;
}

GenParams make_gen_params(scendp_ctx* ctx, const scendp_dist* d, uint64_t first_index) {
  check_dist(d);
  GenParams g{};
  g.kind = d->kind;
  g.lo = d->lo;
  g.span = static_cast<uint64_t>(d->hi - d->lo) + 1;
  g.span32 = g.span < (uint64_t{1} << 32) ? static_cast<uint32_t>(g.span) : 0u;
  g.seed = d->seed;
  g.first_index = first_index;
  if (d->kind == SCENDP_DIST_POISSON) {
    // the table stays resident for the next call with the same (mean, hi)
    // unless its scratch slot was reallocated or reused (tnormal's list)
    // table [len] doubles, then the 65-entry guide of draw_value
    const size_t len = static_cast<size_t>(d->hi) + 1;
    const size_t bytes = len * sizeof(double) + 65 * sizeof(int32_t);
    char* dev = static_cast<char*>(ctx->scratch_get(kScrCdf, bytes));
    if (!(ctx->cdf_mean == d->mean && ctx->cdf_hi == d->hi &&
          ctx->cdf_dev == reinterpret_cast<double*>(dev) &&
          ctx->cdf_gen == ctx->scratch_gen[kScrCdf])) {
      std::vector<double> cdf = poisson_table(d->mean, d->hi);
      std::vector<char> blob(bytes);
      std::memcpy(blob.data(), cdf.data(), len * sizeof(double));
      int32_t* guide = reinterpret_cast<int32_t*>(blob.data() + len * sizeof(double));
      int32_t k = 0;
      for (int j = 0; j <= 64; ++j) {
        while (k + 1 < static_cast<int32_t>(len) && cdf[k] < j / 64.0) ++k;
        guide[j] = k;
      }
      ctx->copy(dev, blob.data(), bytes, cudaMemcpyHostToDevice);
      ctx->cdf_mean = d->mean;
      ctx->cdf_hi = d->hi;
      ctx->cdf_dev = reinterpret_cast<double*>(dev);
      ctx->cdf_gen = ctx->scratch_gen[kScrCdf];
    }
    g.cdf_len = static_cast<int32_t>(len);
    g.cdf = reinterpret_cast<const double*>(dev);
    g.guide = reinterpret_cast<const int32_t*>(dev + len * sizeof(double));
  }
  return g;
}

// One tnormal column with the reference's own arithmetic (SplitMix64 over
// derive_stream(seed, kStreamScenario, w), DistributionSpec::sample,
// scenario.cpp:22-40; glibc log / cos / sqrt / llround): the host side of
// the certified generator above.
void tnormal_column_host(const scendp_dist* d, uint64_t w, uint64_t rows, uint32_t* col) {
  uint64_t st = derive_stream(d->seed, kStreamScenario, w);
  auto next_unit = [&st] {
    const uint64_t x = mix64(st);
    st += kGamma;
    return static_cast<double>((x >> 11) + 1) * 0x1.0p-53;
  };
  const double two_pi = 2.0 * 0x1.921fb54442d18p+1;
  for (uint64_t r = 0; r < rows; ++r) {
    bool done = false;
    for (int attempt = 0; attempt < 64 && !done; ++attempt) {
      const double u1 = next_unit();
      const double u2 = next_unit();
      const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2);
      const long long rr = std::llround(d->mean + d->stddev * z);
      if (rr >= d->lo && rr <= d->hi) {
        col[r] = static_cast<uint32_t>(rr);
        done = true;
      }
    }
    if (!done) col[r] = static_cast<uint32_t>(std::clamp<long long>(std::llround(d->mean), d->lo, d->hi));
  }
}

void launch_generate_tiled(scendp_ctx* ctx, const scendp_dist* d, uint64_t rows,
                           uint64_t w0, uint64_t count, uint32_t* out) {
  if (count == 0) return;
  const unsigned blocks = static_cast<unsigned>((count + kGenThreads - 1) / kGenThreads);
  const int tok = ctx->timing_begin(1);
  if (d->kind == SCENDP_DIST_TNORMAL) {
    check_dist(d);
    constexpr uint32_t kAmbCap = 4096;
    auto* amb = static_cast<char*>(ctx->scratch_get(kScrCdf, 16 + kAmbCap * 8ull));
    ctx->cdf_dev = nullptr;  // the slot now holds tnormal's list, not a Poisson table
    CUDA_CHECK(cudaMemsetAsync(amb, 0, 16, ctx->stream));
    static const uint32_t force_every = [] {
      const char* e = std::getenv("SCENDP_TNORMAL_HOST_EVERY");
      return e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : 0u;
    }();
    gen_tnormal_kernel<<<blocks, kGenThreads, 0, ctx->stream>>>(
        d->lo, d->hi, d->mean, d->stddev, d->seed, w0, rows, count, out,
        reinterpret_cast<unsigned int*>(amb), reinterpret_cast<unsigned long long*>(amb + 16),
        kAmbCap, force_every);
    CUDA_CHECK(cudaGetLastError());
    ctx->timing_end(tok);
    ctx->count_launch();
    // columns the device could not certify: regenerate them on the host
    // with the reference's arithmetic (all of them if the list overflowed)
    uint32_t n_amb = 0;
    CUDA_CHECK(cudaMemcpyAsync(&n_amb, amb, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (n_amb == 0) return;
    std::vector<uint64_t> cols;
    if (n_amb <= kAmbCap) {
      cols.resize(n_amb);
      CUDA_CHECK(cudaMemcpy(cols.data(), amb + 16, n_amb * 8ull, cudaMemcpyDeviceToHost));
    } else {
      cols.resize(count);
      for (uint64_t w = 0; w < count; ++w) cols[w] = w;
    }
    std::vector<uint32_t> col(rows);
    for (uint64_t w : cols) {
      tnormal_column_host(d, w0 + w, rows, col.data());
      // column w of the tiled layout: rows values 128 bytes apart
      CUDA_CHECK(cudaMemcpy2DAsync(out + (w >> 5) * rows * kTile + (w & 31), kTile * 4, col.data(),
                                   4, 4, rows, cudaMemcpyHostToDevice, ctx->stream));
      CUDA_CHECK(cudaStreamSynchronize(ctx->stream));  // col is reused
      ctx->tnormal_host_columns += 1;
    }
    return;
  } else {
    GenParams g = make_gen_params(ctx, d, w0);
    const size_t smem = g.kind == SCENDP_DIST_POISSON ? g.cdf_len * sizeof(double) : 0;
    if (smem > 48 * 1024)
      CUDA_CHECK(cudaFuncSetAttribute(gen_counter_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    gen_counter_kernel<<<blocks, kGenThreads, smem, ctx->stream>>>(g, rows, count, out);
  }
  CUDA_CHECK(cudaGetLastError());
  ctx->timing_end(tok);
  ctx->count_launch();
}

template <typename T>
void launch_to_tiled(scendp_ctx* ctx, const T* src, uint64_t rows, uint64_t count, T* dst) {
  if (count == 0 || rows == 0) return;
  dim3 grid(static_cast<unsigned>((count + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  to_tiled_kernel<T><<<grid, 256, 0, ctx->stream>>>(src, rows, count, dst);
  CUDA_CHECK(cudaGetLastError());
  ctx->count_launch();
}

template <typename T>
void launch_from_tiled(scendp_ctx* ctx, const T* src, uint64_t rows, uint64_t count, T* dst) {
  if (count == 0 || rows == 0) return;
  dim3 grid(static_cast<unsigned>((count + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  from_tiled_kernel<T><<<grid, 256, 0, ctx->stream>>>(src, rows, count, dst);
  CUDA_CHECK(cudaGetLastError());
  ctx->count_launch();
}

template void launch_to_tiled<uint32_t>(scendp_ctx*, const uint32_t*, uint64_t, uint64_t, uint32_t*);
template void launch_from_tiled<double>(scendp_ctx*, const double*, uint64_t, uint64_t, double*);
template void launch_from_tiled<int32_t>(scendp_ctx*, const int32_t*, uint64_t, uint64_t, int32_t*);
template void launch_from_tiled<uint8_t>(scendp_ctx*, const uint8_t*, uint64_t, uint64_t, uint8_t*);
template void launch_from_tiled<uint32_t>(scendp_ctx*, const uint32_t*, uint64_t, uint64_t, uint32_t*);

// Narrowed host chunks (u8 per demand) widened while tiling.
void launch_to_tiled_u8(scendp_ctx* ctx, const uint8_t* src, uint64_t rows, uint64_t count,
                        uint32_t* dst) {
  if (count == 0 || rows == 0) return;
  dim3 grid(static_cast<unsigned>((count + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  to_tiled_kernel<uint32_t, uint8_t><<<grid, 256, 0, ctx->stream>>>(src, rows, count, dst);
  CUDA_CHECK(cudaGetLastError());
  ctx->count_launch();
}

// u32 -> u8 of `n` values split over up to `threads` host threads; false if
// any value needs more than 8 bits (the chunk then goes as u32)
static bool parallel_pack_u8(uint8_t* dst, const uint32_t* src, uint64_t n, int threads) {
  const uint64_t per = ((n + threads - 1) / threads + 4095) & ~uint64_t{4095};
  const int parts = static_cast<int>(std::max<uint64_t>(1, (n + per - 1) / per));
  std::vector<uint32_t> wide(parts, 0u);
  parallel_parts(parts, [&](int t) {
    const uint64_t lo = per * t, hi = std::min(n, per * (t + 1));
    uint32_t acc = 0u;
    for (uint64_t i = lo; i < hi; ++i) {
      const uint32_t v = src[i];
      acc |= v;
      dst[i] = static_cast<uint8_t>(v);
    }
    wide[t] = acc >> 8;
  });
  uint32_t any = 0u;
  for (uint32_t w : wide) any |= w;
  return any == 0u;
}

// memcpy of `bytes` split over up to `threads` host threads
static void parallel_copy(char* dst, const char* src, uint64_t bytes, int threads) {
  const uint64_t per = ((bytes + threads - 1) / threads + 4095) & ~uint64_t{4095};
  const int parts = static_cast<int>(std::max<uint64_t>(1, (bytes + per - 1) / per));
  parallel_parts(parts, [&](int t) {
    const uint64_t lo = per * t, hi = std::min(bytes, per * (t + 1));
    std::memcpy(dst + lo, src + lo, hi - lo);
  });
}

// A pageable host scenario set (the reference's ScenarioBatch vector) into
// the tiled layout, in whole-tile chunks: up to 16 host threads stage each
// chunk into one of two page-locked buffers (alternating, event-guarded)
// while the previous chunk's H2D copy and tiling run on the stream (a
// driver-staged copy from pageable memory runs at ~11 GB/s).  Demands below
// 256 are narrowed to one byte while staging (1/4 of the PCIe bytes, widened
// by the tiling kernel); a chunk with a wider value is copied as is.
// Scenarios per staging chunk of a pageable upload (whole tiles, ~64 MB).
uint64_t pageable_chunk(uint64_t rows, uint64_t count) {
  constexpr uint64_t kChunkBytes = 64ull << 20;
  const uint64_t col_bytes = rows * 4;
  const uint64_t chunk = std::max<uint64_t>(32, (kChunkBytes / col_bytes) & ~uint64_t{31});
  return std::min(chunk, (count + 31) & ~uint64_t{31});
}

uint64_t pageable_chunk_bytes(uint64_t rows, uint64_t count) {
  return pageable_chunk(rows, count) * rows * 4;
}

void upload_pageable_tiled(scendp_ctx* ctx, const uint32_t* src, uint64_t rows, uint64_t count,
                           uint32_t* dst) {
  const uint64_t col_bytes = rows * 4;
  const uint64_t chunk = pageable_chunk(rows, count);
  const uint64_t stage_bytes = chunk * col_bytes;
  char* pin[2] = {static_cast<char*>(ctx->pinned_stage(0, stage_bytes)),
                  static_cast<char*>(ctx->pinned_stage(1, stage_bytes))};
  uint32_t* dstage = static_cast<uint32_t*>(ctx->scratch_get(kScrStaging, stage_bytes));
  const int threads = static_cast<int>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
  cudaEvent_t done[2];
  for (auto& e : done) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  bool used[2] = {false, false};
  const char* s = reinterpret_cast<const char*>(src);
  // demands below 256 (the usual case) cross PCIe as one byte each: packed
  // by the host threads while they stage, widened by the tiling kernel; the
  // first chunk with a wider value switches the rest of the call to u32
  bool narrow = true;
  for (uint64_t c0 = 0, j = 0; c0 < count; c0 += chunk, ++j) {
    const uint64_t cn = std::min(chunk, count - c0);
    const int b = static_cast<int>(j & 1);
    if (used[b]) CUDA_CHECK(cudaEventSynchronize(done[b]));
    const uint64_t bytes = cn * col_bytes;
    if (narrow) {
      uint8_t* p8 = reinterpret_cast<uint8_t*>(pin[b]);
      if (parallel_pack_u8(p8, src + c0 * rows, cn * rows, threads)) {
        uint8_t* d8 = reinterpret_cast<uint8_t*>(dstage);
        ctx->copy(d8, p8, cn * rows, cudaMemcpyHostToDevice);
        launch_to_tiled_u8(ctx, d8, rows, cn, dst + (c0 / 32) * rows * 32);
        CUDA_CHECK(cudaEventRecord(done[b], ctx->stream));
        used[b] = true;
        continue;
      }
      narrow = false;
    }
    parallel_copy(pin[b], s + c0 * col_bytes, bytes, threads);
    ctx->copy(dstage, pin[b], bytes, cudaMemcpyHostToDevice);
    launch_to_tiled<uint32_t>(ctx, dstage, rows, cn, dst + (c0 / 32) * rows * 32);
    CUDA_CHECK(cudaEventRecord(done[b], ctx->stream));
    used[b] = true;
  }
  // the staging buffers are reused by the next call: drain before returning
  for (int b = 0; b < 2; ++b)
    if (used[b]) CUDA_CHECK(cudaEventSynchronize(done[b]));
  for (auto& e : done) CUDA_CHECK(cudaEventDestroy(e));
}


void download(scendp_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  constexpr uint64_t kChunk = 64ull << 20;
  if (bytes <= (16ull << 20) || mapped_host_alias(dst)) {
    ctx->copy(dst, src, bytes, cudaMemcpyDeviceToHost);
    return;
  }
  const int threads = static_cast<int>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
  char* pin[2] = {static_cast<char*>(ctx->pinned_stage(0, kChunk)),
                  static_cast<char*>(ctx->pinned_stage(1, kChunk))};
  cudaEvent_t done[2];
  for (auto& e : done) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  char* d = static_cast<char*>(dst);
  const char* sp = static_cast<const char*>(src);
  const uint64_t nchunks = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](uint64_t j) {
    const uint64_t off = j * kChunk, len = std::min(kChunk, bytes - off);
    ctx->copy(pin[j & 1], sp + off, len, cudaMemcpyDeviceToHost);
    CUDA_CHECK(cudaEventRecord(done[j & 1], ctx->stream));
  };
  issue(0);
  for (uint64_t j = 0; j < nchunks; ++j) {
    if (j + 1 < nchunks) issue(j + 1);  // the other buffer is free: drained below
    CUDA_CHECK(cudaEventSynchronize(done[j & 1]));
    const uint64_t off = j * kChunk, len = std::min(kChunk, bytes - off);
    parallel_copy(d + off, pin[j & 1], len, threads);
  }
  for (auto& e : done) CUDA_CHECK(cudaEventDestroy(e));
}

const uint32_t* stage_scenarios(scendp_ctx* ctx, const scendp_scenarios* sc,
                                bool allow_fused, void* gen_params_out, bool* fused) {
  *fused = false;
  const uint64_t rows = sc->rows, count = sc->count;
  const uint64_t tiled_bytes = scendp_tiled_bytes(rows, count);
  switch (sc->mem_kind) {
    case SCENDP_MEM_DEVICE_TILED:
      if (!sc->data && count) fail(SCENDP_ERR_INVALID_ARGUMENT, "scenario data is null");
      return sc->data;
    case SCENDP_MEM_GENERATED: {
      if (!sc->dist) fail(SCENDP_ERR_INVALID_ARGUMENT, "generated scenarios need a dist");
      if (allow_fused && sc->dist->kind != SCENDP_DIST_TNORMAL) {
        *static_cast<GenParams*>(gen_params_out) = make_gen_params(ctx, sc->dist, sc->first_index);
        *fused = true;
        return nullptr;
      }
      uint32_t* dst = static_cast<uint32_t*>(ctx->scratch_get(kScrScenarios, tiled_bytes));
      launch_generate_tiled(ctx, sc->dist, rows, sc->first_index, count, dst);
      return dst;
    }
    case SCENDP_MEM_HOST: {
      if (!sc->data && count) fail(SCENDP_ERR_INVALID_ARGUMENT, "scenario data is null");
      uint32_t* dst = static_cast<uint32_t*>(ctx->scratch_get(kScrScenarios, tiled_bytes));
      if (mapped_host_alias(const_cast<uint32_t*>(sc->data)) || rows * count * 4 <= (16ull << 20)) {
        // page-locked (DMA straight from it: measured faster than narrowing
        // it on the host) or small: one copy
        uint32_t* stg = static_cast<uint32_t*>(ctx->scratch_get(kScrStaging, rows * count * 4));
        ctx->copy(stg, sc->data, rows * count * 4, cudaMemcpyHostToDevice);
        launch_to_tiled<uint32_t>(ctx, stg, rows, count, dst);
      } else {
        upload_pageable_tiled(ctx, sc->data, rows, count, dst);
      }
      return dst;
    }
    case SCENDP_MEM_DEVICE: {
      if (!sc->data && count) fail(SCENDP_ERR_INVALID_ARGUMENT, "scenario data is null");
      uint32_t* dst = static_cast<uint32_t*>(ctx->scratch_get(kScrScenarios, tiled_bytes));
      launch_to_tiled<uint32_t>(ctx, sc->data, rows, count, dst);
      return dst;
    }
    default:
      fail(SCENDP_ERR_INVALID_ARGUMENT, "unknown scenario mem_kind");
  }
}

uint64_t stage_footprint(const scendp_scenarios* sc, uint64_t* fixed) {
  const uint64_t rows = sc->rows;
  *fixed = 0;
  switch (sc->mem_kind) {
    case SCENDP_MEM_GENERATED:
      if (sc->dist && sc->dist->kind == SCENDP_DIST_TNORMAL) return 4 * rows;  // tiled set
      if (sc->dist && sc->dist->kind == SCENDP_DIST_POISSON) *fixed = 64 << 10;  // CDF table
      return 0;  // generated inside the DP kernels
    case SCENDP_MEM_HOST:
      // page-locked or small (<= 16 MB): one staging copy + the tiled set;
      // larger pageable sets: the tiled set + one ~64 MB staging chunk
      if ((sc->data && mapped_host_alias(const_cast<uint32_t*>(sc->data))) ||
          rows * sc->count * 4 <= (16ull << 20))
        return 8 * rows;
      *fixed = pageable_chunk_bytes(rows, sc->count);
      return 4 * rows;
    case SCENDP_MEM_DEVICE:
      return 4 * rows;
    default:
      return 0;
  }
}

void reserve_stage(scendp_ctx* ctx, const scendp_scenarios* sc, uint64_t mw) {
  const uint64_t rows = sc->rows, tiled = scendp_tiled_bytes(rows, mw);
  switch (sc->mem_kind) {
    case SCENDP_MEM_GENERATED:
      if (sc->dist && sc->dist->kind == SCENDP_DIST_TNORMAL) {
        ctx->scratch_get(kScrScenarios, tiled);
        ctx->scratch_get(kScrCdf, 16 + 4096 * 8);  // uncertified-column list
      }
      return;
    case SCENDP_MEM_HOST: {
      ctx->scratch_get(kScrScenarios, tiled);
      const bool direct = (sc->data && mapped_host_alias(const_cast<uint32_t*>(sc->data))) ||
                          rows * mw * 4 <= (16ull << 20);
      ctx->scratch_get(kScrStaging, direct ? rows * mw * 4 : pageable_chunk_bytes(rows, mw));
      return;
    }
    case SCENDP_MEM_DEVICE:
      ctx->scratch_get(kScrScenarios, tiled);
      return;
    default:
      return;
  }
}

void release_wave_scratch(scendp_ctx* ctx) {
  for (int s : {kScrScenarios, kScrStaging, kScrTotals, kScrOut1, kScrOut2, kScrOut3, kScrOut4,
                kScrOut5, kScrOut6, kScrOut7, kScrOut8, kScrOut9, kScrOverflow, kScrHandoff})
    ctx->scratch_free(s);
}

}  // namespace scendp_host

extern "C" {

uint64_t scendp_tiled_bytes(uint64_t rows, uint64_t count) {
  return ((count + 31) / 32) * rows * 32 * sizeof(uint32_t);
}

scendp_status scendp_gen_scenarios(scendp_ctx* ctx, const scendp_dist* dist, uint64_t rows,
                                   uint64_t w0, uint64_t count, uint32_t layout,
                                   uint32_t* out) {
  NvtxRange nvtx("scendp_gen_scenarios");
  return guard([&] {
    if (!ctx || !out) fail(SCENDP_ERR_INVALID_ARGUMENT, "null ctx or output");
    check_dist(dist);
    if (rows == 0) fail(SCENDP_ERR_INVALID_ARGUMENT, "scenario grid must have at least one cell");
    CUDA_CHECK(cudaSetDevice(ctx->device));
    if (layout == SCENDP_MEM_DEVICE_TILED) {
      launch_generate_tiled(ctx, dist, rows, w0, count, out);
    } else if (layout == SCENDP_MEM_DEVICE) {
      uint32_t* tmp = static_cast<uint32_t*>(
          ctx->scratch_get(kScrScenarios, scendp_tiled_bytes(rows, count)));
      launch_generate_tiled(ctx, dist, rows, w0, count, tmp);
      launch_from_tiled<uint32_t>(ctx, tmp, rows, count, out);
    } else {
      fail(SCENDP_ERR_INVALID_ARGUMENT, "layout must be SCENDP_MEM_DEVICE or DEVICE_TILED");
    }
    ctx->sync();
  });
}

scendp_status scendp_scenarios_to_tiled(scendp_ctx* ctx, const uint32_t* src, uint64_t rows,
                                        uint64_t count, uint32_t* dst) {
  return guard([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    launch_to_tiled<uint32_t>(ctx, src, rows, count, dst);
    ctx->sync();
  });
}

}  // extern "C"
