// minplus.cu -- K5: the generic dense (min,+) stage sweep (the paper's
// Alg. 1; reference minplus.cpp:56-102), batched over many
// frontiers that share one stage chain.
//
//   J_{s+1}[b][j] = min_r min_i ( A_s(i, j; r) + J_s[b][i] )
//
// with the reference's scan order (option r ascending, then predecessor i
// ascending, extended_min keeping the incumbent on ties).  The values are
// order-independent except for the sign of a zero tie; the kernel runs the
// reference's own compare-and-select (extended_min, exact for signed zeros
// and NaN alike), which on sm_100 is also cheaper than fmin.
//
// Execution model: a min-plus "GEMM" (no tensor-core form exists for the
// (min,+) semiring).  A CTA owns a tile of kTB frontiers x kTJ columns; the
// predecessor axis is walked in chunks of kTI rows, the frontier chunk
// J[b][i..] and the matrix chunk A[r][i..][j..] are staged in shared memory,
// and every thread accumulates a 4 x 4 micro-tile in registers (32 FP64 ops
// per 8 shared loads).  Padding rows/columns hold +inf, which never wins.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

using namespace scendp_host;

namespace {

constexpr int kTB = 64;   // frontiers per CTA
constexpr int kTJ = 64;   // columns per CTA
constexpr int kTI = 16;   // predecessors per smem chunk
constexpr int kMB = 4;    // micro-tile rows (frontiers) per thread
constexpr int kMJ = 4;    // micro-tile columns per thread
constexpr int kThreads = (kTB / kMB) * (kTJ / kMJ);  // 256
constexpr double kInf = __builtin_huge_val();

template <bool EXACT_TIES>
__device__ __forceinline__ double mp_min(double best, double cand) {
  if constexpr (EXACT_TIES) return cand < best ? cand : best;  // extended_min
  else return fmin(best, cand);
}

// in: [B][in_stride] (first `rows` entries), a: [depth][rows][cols],
// out: [B][out_stride] (first `cols` entries)
template <bool EXACT_TIES>
__global__ void __launch_bounds__(kThreads)
minplus_stage_kernel(const double* __restrict__ in, uint64_t in_stride,
                     const double* __restrict__ a, uint64_t rows, uint64_t cols, uint64_t depth,
                     double* __restrict__ out, uint64_t out_stride, uint64_t batch) {
  __shared__ __align__(16) double sJ[kTI][kTB + 2];  // [i][b]  (+2: bank spread)
  __shared__ __align__(16) double sA[kTI][kTJ];      // [i][j]
  const int tx = threadIdx.x % (kTJ / kMJ);  // column group
  const int ty = threadIdx.x / (kTJ / kMJ);  // frontier group
  const uint64_t b0 = static_cast<uint64_t>(blockIdx.y) * kTB;
  const uint64_t j0 = static_cast<uint64_t>(blockIdx.x) * kTJ;
  double acc[kMB][kMJ];
#pragma unroll
  for (int x = 0; x < kMB; ++x)
#pragma unroll
    for (int y = 0; y < kMJ; ++y) acc[x][y] = kInf;

  for (uint64_t r = 0; r < depth; ++r) {
    const double* ar = a + r * rows * cols;
    for (uint64_t i0 = 0; i0 < rows; i0 += kTI) {
      // stage J[b0.., i0..] transposed to [i][b] and A[r][i0..][j0..]
      for (int e = threadIdx.x; e < kTI * kTB; e += kThreads) {
        const int ii = e % kTI, bb = e / kTI;  // consecutive threads: consecutive i
        const uint64_t b = b0 + bb, i = i0 + ii;
        sJ[ii][bb] = (b < batch && i < rows) ? in[b * in_stride + i] : kInf;
      }
      for (int e = threadIdx.x; e < kTI * kTJ; e += kThreads) {
        const int jj = e % kTJ, ii = e / kTJ;
        const uint64_t j = j0 + jj, i = i0 + ii;
        sA[ii][jj] = (j < cols && i < rows) ? ar[i * cols + j] : kInf;
      }
      __syncthreads();
#pragma unroll 4
      for (int ii = 0; ii < kTI; ++ii) {
        double jv[kMB], av[kMJ];
#pragma unroll
        for (int x = 0; x < kMB; ++x) jv[x] = sJ[ii][ty * kMB + x];
#pragma unroll
        for (int y = 0; y < kMJ; ++y) av[y] = sA[ii][tx * kMJ + y];
#pragma unroll
        for (int x = 0; x < kMB; ++x)
#pragma unroll
          for (int y = 0; y < kMJ; ++y) acc[x][y] = mp_min<EXACT_TIES>(acc[x][y], __dadd_rn(av[y], jv[x]));
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int x = 0; x < kMB; ++x) {
    const uint64_t b = b0 + ty * kMB + x;
    if (b >= batch) continue;
#pragma unroll
    for (int y = 0; y < kMJ; ++y) {
      const uint64_t j = j0 + tx * kMJ + y;
      if (j < cols) out[b * out_stride + j] = acc[x][y];
    }
  }
}

}  // namespace

extern "C" scendp_status scendp_minplus_sweep(scendp_ctx* ctx, const scendp_minplus_stage* stages,
                                              uint32_t n_stages, const double* init,
                                              uint64_t init_size, uint64_t batch,
                                              uint32_t mem_kind, uint32_t flags, double* out) {
  NvtxRange nvtx("scendp_minplus_sweep");
  return guard([&] {
    if (!ctx) fail(SCENDP_ERR_INVALID_ARGUMENT, "ctx is null");
    if (mem_kind != SCENDP_MEM_HOST && mem_kind != SCENDP_MEM_DEVICE)
      fail(SCENDP_ERR_INVALID_ARGUMENT, "mem_kind must be SCENDP_MEM_HOST or SCENDP_MEM_DEVICE");
    if (n_stages && !stages) fail(SCENDP_ERR_INVALID_ARGUMENT, "stages is null");
    // dimension checks in the reference's wording (minplus.cpp:24-30, 58-63)
    uint64_t width = init_size, total = init_size, blob = 0;
    for (uint32_t s = 0; s < n_stages; ++s) {
      const scendp_minplus_stage& st = stages[s];
      if (st.rows == 0 || st.cols == 0 || st.depth == 0)
        fail(SCENDP_ERR_INVALID_ARGUMENT, "transition matrix dimensions must be positive");
      if (st.rows != width)
        fail(SCENDP_ERR_INVALID_ARGUMENT, "min-plus apply: matrix has " + std::to_string(st.rows) +
                                              " rows but frontier has " + std::to_string(width) +
                                              " entries");
      if (!st.entries) fail(SCENDP_ERR_INVALID_ARGUMENT, "stage entries are null");
      width = st.cols;
      total += st.cols;
      blob += st.depth * st.rows * st.cols;
    }
    const bool all = (flags & SCENDP_MINPLUS_ALL_STAGES) != 0;
    const uint64_t out_width = all ? total : width;
    if (batch == 0) return;
    if (!init || !out) fail(SCENDP_ERR_INVALID_ARGUMENT, "init/out is null");
    CUDA_CHECK(cudaSetDevice(ctx->device));
    const bool host = mem_kind == SCENDP_MEM_HOST;
    // The compare-select form is extended_min itself (cost.hpp:39-41: NaN and
    // signed-zero semantics included) and it is also the cheaper one on
    // sm_100 (DSETP + 2 selects; fmin lowers to DSETP.MIN + selects + NaN
    // quieting), so it always runs; the flag is kept for ABI compatibility.
    const bool exact = true;
    // device staging: stage matrices (host kind), input frontiers, outputs
    std::vector<const double*> dA(n_stages);
    if (host) {
      double* d_blob = static_cast<double*>(ctx->scratch_get(kScrOut1, std::max<uint64_t>(1, blob) * 8));
      uint64_t off = 0;
      for (uint32_t s = 0; s < n_stages; ++s) {
        const uint64_t e = stages[s].depth * stages[s].rows * stages[s].cols;
        ctx->copy(d_blob + off, stages[s].entries, e * 8, cudaMemcpyHostToDevice);
        dA[s] = d_blob + off;
        off += e;
      }
    } else {
      for (uint32_t s = 0; s < n_stages; ++s) dA[s] = stages[s].entries;
    }
    const double* d_init = init;
    if (host) {
      double* p = static_cast<double*>(ctx->scratch_get(kScrOut2, batch * init_size * 8));
      ctx->copy(p, init, batch * init_size * 8, cudaMemcpyHostToDevice);
      d_init = p;
    }
    double* d_out = host ? static_cast<double*>(ctx->scratch_get(kScrOut3, batch * out_width * 8)) : out;
    // all stages: frontiers are written straight into their slots of the
    // [B][total] output; final-only: ping-pong through scratch
    double* ping = nullptr;
    double* pong = nullptr;
    uint64_t max_w = init_size;
    for (uint32_t s = 0; s < n_stages; ++s) max_w = std::max<uint64_t>(max_w, stages[s].cols);
    if (!all && n_stages > 1) {
      ping = static_cast<double*>(ctx->scratch_get(kScrOut4, batch * max_w * 8));
      pong = static_cast<double*>(ctx->scratch_get(kScrOut5, batch * max_w * 8));
    }
    if (all) {
      // initial frontier copied into slot 0 of every item row
      CUDA_CHECK(cudaMemcpy2DAsync(d_out, out_width * 8, d_init, init_size * 8, init_size * 8,
                                   batch, cudaMemcpyDeviceToDevice, ctx->stream));
    } else if (n_stages == 0) {
      CUDA_CHECK(cudaMemcpyAsync(d_out, d_init, batch * init_size * 8, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
    }
    const double* cur = all ? d_out : d_init;
    uint64_t cur_stride = all ? out_width : init_size;
    uint64_t slot = init_size;
    for (uint32_t s = 0; s < n_stages; ++s) {
      const scendp_minplus_stage& st = stages[s];
      double* dst;
      uint64_t dst_stride;
      if (all) {
        dst = d_out + slot;
        dst_stride = out_width;
      } else if (s + 1 == n_stages) {
        dst = d_out;
        dst_stride = st.cols;
      } else {
        dst = (s & 1) ? pong : ping;
        dst_stride = st.cols;
      }
      dim3 grid(static_cast<unsigned>((st.cols + kTJ - 1) / kTJ),
                static_cast<unsigned>((batch + kTB - 1) / kTB));
      const int tok = ctx->timing_begin(0);
      if (exact)
        minplus_stage_kernel<true><<<grid, kThreads, 0, ctx->stream>>>(
            cur, cur_stride, dA[s], st.rows, st.cols, st.depth, dst, dst_stride, batch);
      else
        minplus_stage_kernel<false><<<grid, kThreads, 0, ctx->stream>>>(
            cur, cur_stride, dA[s], st.rows, st.cols, st.depth, dst, dst_stride, batch);
      CUDA_CHECK(cudaGetLastError());
      ctx->timing_end(tok);
      ctx->count_launch();
      cur = all ? d_out + slot : dst;
      cur_stride = dst_stride;
      slot += st.cols;
    }
    if (host) ctx->copy(out, d_out, batch * out_width * 8, cudaMemcpyDeviceToHost);
    ctx->sync();
  });
}
