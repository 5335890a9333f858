/*
 * scendp_cuda.h -- the C-ABI of the B200-native scenario-batched DP engine.
 *
 * Plain C: opaque context, plain pointers and sizes, status codes, no
 * exceptions and no C++/torch types across the boundary.  The C++ drop-in
 * facade (include/scendp/ headers) and the Python/ctypes host mirror
 * (paper_2602_05179_b200/) both sit on top of this header.
 *
 * Each evaluator replaces one reference entry point (paths relative to
 * /root/reference/proj):
 *
 *   scendp_split_eval    <- batched_split_costs            split.hpp:108-111
 *                           batched_expected_split         split.hpp:102-104
 *                           batched_split_costs_generated  split.hpp:116-119
 *                           K-tour candidate scoring        saa.cpp:127-131
 *   scendp_dsirp_eval    <- batched_expected_cost          oudp.hpp:135-138
 *                           (one call covers many customers: rows c*H+t)
 *   scendp_gen_scenarios <- generate_scenarios             scenario.hpp:103-105
 *                           generate_scenario_column       scenario.hpp:97-98
 *   scendp_agg           <- BatchResultSet::{mean_cost, finite_count,
 *                           infeasible_count}              engine.hpp:76-87
 *
 * Semantics kept bit-for-bit: +inf masking and strict-< first-minimum ties
 * (cost.hpp:33-41), the reference's fp64 association (no FMA contraction),
 * customer-id demand indexing (split.cpp:33), hard mode -> linear deque cuts
 * (split.cpp:316-318), penalized -> quadratic (split.cpp:45-75), DSIRP tie
 * order no-delivery < route option < state (oudp.cpp:36-39).
 *
 * Errors: every call validates synchronously before any device work, like the
 * reference's std::invalid_argument checks (split.cpp:128-178, oudp.cpp:136-
 * 207, 402-407), and returns a status; scendp_last_error() (thread-local)
 * holds the message.  There is no CPU fallback: a context cannot be created
 * without a CUDA device (SCENDP_ERR_NO_DEVICE).
 */
#ifndef SCENDP_CUDA_H
#define SCENDP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCENDP_ABI_VERSION 1

typedef enum {
  SCENDP_OK = 0,
  SCENDP_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  SCENDP_ERR_CUDA = 2,
  SCENDP_ERR_NCCL = 3,
  SCENDP_ERR_OUT_OF_MEMORY = 4,
  SCENDP_ERR_NO_DEVICE = 5,
  SCENDP_ERR_LOGIC = 6,            /* std::logic_error */
  SCENDP_ERR_RUNTIME = 7,          /* std::runtime_error */
  SCENDP_ERR_UNSUPPORTED = 8       /* valid input outside this build's limits */
} scendp_status;

typedef struct scendp_ctx scendp_ctx;

/* ---- context ------------------------------------------------------------
 * One context = one CUDA device + one stream + cached scratch.  The
 * reference's BackendConfig (engine.hpp:24-51) maps onto it: memory_budget
 * -> scratch_limit (device bytes a single call's scratch may use; 0 = the
 * free device memory), batch_size -> max_batch (scenarios per launch wave;
 * 0 = whole call).  A call runs in waves sized by its device footprint
 * model (scendp_split_footprint / scendp_dsirp_footprint) under that budget;
 * an allocation failure halves the wave and retries (never below one
 * 32-scenario tile), so results never depend on the budget. */
typedef struct {
  int32_t device;          /* CUDA ordinal; -1 = current device */
  uint64_t scratch_limit;  /* device scratch budget of a call (bytes): caps
                              the wave size; 0 = free device memory */
  uint64_t max_batch;      /* scenarios per launch wave; 0 = unlimited */
  uint32_t flags;          /* SCENDP_CTX_* */
} scendp_opts;

#define SCENDP_CTX_KERNEL_TIMING 0x1u /* CUDA events around hot kernels */

scendp_status scendp_ctx_create(const scendp_opts* opts, scendp_ctx** out);
void scendp_ctx_destroy(scendp_ctx* ctx);
const char* scendp_last_error(void);
int32_t scendp_abi_version(void);
/* device ordinal, SM count and the stream all work is enqueued on */
scendp_status scendp_ctx_info(scendp_ctx* ctx, int32_t* device,
                              int32_t* sm_count, void** cuda_stream);
scendp_status scendp_ctx_sync(scendp_ctx* ctx);
/* per-call wave size (BackendConfig::batch_size after adjust_batch_size) */
scendp_status scendp_ctx_set_max_batch(scendp_ctx* ctx, uint64_t max_batch);

/* device / pinned-host memory helpers (tests, bench, SCNB staging) */
scendp_status scendp_device_alloc(scendp_ctx* ctx, uint64_t bytes, void** ptr);
scendp_status scendp_device_free(scendp_ctx* ctx, void* ptr);
scendp_status scendp_host_alloc_pinned(uint64_t bytes, void** ptr);
scendp_status scendp_host_free_pinned(void* ptr);
/* kind: 0 = host->device, 1 = device->host, 2 = device->device (stream
 * ordered, synchronous unless SCENDP_ASYNC) */
scendp_status scendp_memcpy(scendp_ctx* ctx, void* dst, const void* src,
                            uint64_t bytes, int32_t kind, uint32_t flags);
scendp_status scendp_memset(scendp_ctx* ctx, void* dst, int32_t value,
                            uint64_t bytes);

/* ---- scenario distributions (scenario.hpp:60-76) ---------------------- */
typedef enum {
  SCENDP_DIST_UNIFORM = 0,  /* lo + next_below(hi-lo+1): scenario.cpp:23-26 */
  SCENDP_DIST_TNORMAL = 1,  /* Box-Muller + llround + rejection: 30-39 */
  SCENDP_DIST_POISSON = 2   /* new kind: inverse CDF over P[0..hi], one
                               next_unit per draw; mean = lambda, lo = 0 */
} scendp_dist_kind;

typedef struct {
  int32_t kind;
  int64_t lo, hi;
  double mean, stddev;
  uint64_t seed;  /* DistributionSpec::seed; column w uses
                     derive_stream(seed, kStreamScenario, w) */
} scendp_dist;

/* Scenario-set memory kinds. */
typedef enum {
  SCENDP_MEM_HOST = 0,         /* reference layout on the host: column w is
                                  data[w*rows .. (w+1)*rows) (scenario.hpp:78-92) */
  SCENDP_MEM_DEVICE = 1,       /* reference layout, device pointer */
  SCENDP_MEM_DEVICE_TILED = 2, /* native HBM layout, device pointer:
                                  [w/32][row][w%32] (32-scenario tiles, one
                                  128-byte line per (tile,row)); a prefix of
                                  whole tiles is a prefix of the buffer */
  SCENDP_MEM_GENERATED = 3     /* generated in-kernel from `dist` (fused
                                  generate+DP, split.cpp:373-388) */
} scendp_mem_kind;

typedef struct {
  uint32_t mem_kind;
  const uint32_t* data;     /* HOST / DEVICE / DEVICE_TILED */
  uint64_t rows;            /* n (split) or n_customers*H (dsirp) */
  uint64_t count;           /* scenarios in this call (this shard) */
  uint64_t first_index;     /* global index of scenario 0 of this call: the
                               generator stream index for GENERATED (other
                               kinds: informational).  A DEVICE_TILED `data`
                               holds this call's scenario 0 in lane 0 of its
                               first tile (a tile-aligned shard of a larger
                               tiled set is a byte range of it) */
  const scendp_dist* dist;  /* GENERATED only */
} scendp_scenarios;

/* Bytes of a DEVICE_TILED buffer holding `count` scenarios of `rows` rows. */
uint64_t scendp_tiled_bytes(uint64_t rows, uint64_t count);

/* K4: generate scenarios [w0, w0+count) into `out` (device pointer) in the
 * given layout (SCENDP_MEM_DEVICE = reference layout, or DEVICE_TILED).
 * Bit-identical to generate_scenarios for uniform and poisson; tnormal uses
 * CUDA libm (log/cos may differ from glibc by <= 1 ulp before rounding). */
scendp_status scendp_gen_scenarios(scendp_ctx* ctx, const scendp_dist* dist,
                                   uint64_t rows, uint64_t w0, uint64_t count,
                                   uint32_t layout, uint32_t* out);

/* Reference layout (device) -> tiled layout (device). */
scendp_status scendp_scenarios_to_tiled(scendp_ctx* ctx, const uint32_t* src,
                                        uint64_t rows, uint64_t count,
                                        uint32_t* dst_tiled);

/* ---- SCNB scenario files (io.hpp:44-49, io.cpp:276-344) -----------------
 * Little-endian "SCNB" | u16 version=1 | u32 rows | u32 cols | u16 dtype=1
 * (u32), then rows*cols u32 values, scenario-major.  The 16-byte header keeps
 * the payload 16-byte aligned, and scenarios [a, b) are one contiguous file
 * range, so a shard is read without touching the rest of the file.  Errors
 * use the reference's messages (SCENDP_ERR_RUNTIME = its runtime_error). */
typedef struct {
  uint64_t rows;   /* ScenarioBatch::rows */
  uint64_t count;  /* ScenarioBatch::count (the header's "cols") */
} scendp_scnb_header;

scendp_status scendp_scnb_header_read(const char* path, scendp_scnb_header* hdr);

/* Streams scenarios [first, first+count) of an SCNB file into device memory
 * `out` in `layout` (SCENDP_MEM_DEVICE: reference layout, count*rows u32;
 * SCENDP_MEM_DEVICE_TILED: native layout, scendp_tiled_bytes(rows, count),
 * scenario `first` in tile 0).  Whole-tile chunks are read with pread() into
 * two page-locked staging buffers, alternating, while the previous chunk's
 * H2D copy (and tiling) runs on the context stream.  Synchronous. */
scendp_status scendp_scnb_load(scendp_ctx* ctx, const char* path, uint64_t first,
                               uint64_t count, uint32_t layout, uint32_t* out);

/* write_scenario_binary (io.cpp:300-307) for a host scenario set in the
 * reference layout. */
scendp_status scendp_scnb_write(const char* path, const uint32_t* data,
                                uint64_t rows, uint64_t count);

/* ---- aggregates ----------------------------------------------------------
 * Per candidate (tour or customer): the finite-cost sum, exact.  Every
 * finite cost is added into a fixed-point integer accumulator (32-bit digits
 * held in 64-bit words, weights 2^-192 .. 2^192), so the sum is independent
 * of scenario order, block shape and GPU count (integer addition is
 * associative) and is the correctly rounded double of the true sum.  The
 * reference's sequential double sum (engine.hpp:195-211) differs from it by
 * at most its own rounding (<= m*eps relative); both are bit-identical when
 * all costs are integers and the sum is below 2^53. */
#define SCENDP_AGG_DIGITS 12
typedef struct {
  uint64_t digits[SCENDP_AGG_DIGITS]; /* raw device accumulator (NCCL sums these) */
  uint64_t finite_count;
  uint64_t infeasible_count;          /* evaluated, cost == +inf */
  uint64_t error_count;               /* evaluated == 0 (engine.hpp:159-165) */
  uint64_t range_errors;              /* finite costs >= 2^192 (not summed) */
} scendp_agg_raw;

typedef struct {
  double sum;               /* correctly rounded exact sum of finite costs */
  double mean;              /* sum / finite_count; NaN when finite_count==0 */
  uint64_t finite_count;
  uint64_t infeasible_count;
  uint64_t error_count;
  uint64_t range_errors;
} scendp_agg;

/* Combine raw accumulators (e.g. shards evaluated on different devices) and
 * finalize; `n` raw records per candidate, `k` candidates, raw is [n][k]. */
scendp_status scendp_agg_finalize(const scendp_agg_raw* raw, uint32_t n,
                                  uint32_t k, scendp_agg* out);

/* ---- CVRPSD split (split.hpp / split.cpp) ------------------------------ */
typedef struct {
  int32_t n;              /* customers; nodes 0 (out depot) .. n+1 (in depot) */
  int64_t capacity;       /* Q > 0 */
  int32_t hard;           /* 1: +inf mask (linear deque); 0: beta*excess */
  double penalty_beta;
  const double* costs;    /* (n+2)*(n+2) row-major, host memory */
} scendp_routing;

#define SCENDP_SPLIT_COST_ONLY 0u /* totals + aggregates */
#define SCENDP_SPLIT_FULL 1u      /* + V, cuts, route_count (k_tours == 1) */
#define SCENDP_ASYNC 0x100u       /* do not synchronise the stream on return */
#define SCENDP_QUADRATIC 0x200u   /* force the O(n^2) form in hard mode */

typedef struct {
  uint32_t mem_kind;     /* SCENDP_MEM_HOST, SCENDP_MEM_DEVICE (reference
                            layout) or SCENDP_MEM_DEVICE_TILED */
  double* totals;        /* [k][m] per-scenario totals, or NULL */
  double* values;        /* FULL: V, [m][n+1] (tiled: [m/32][n+1][32]) */
  int32_t* cuts;         /* FULL: argmin predecessors, -1 unreachable */
  int32_t* route_count;  /* FULL: [m] */
  uint8_t* feasible;     /* FULL: [m] */
  scendp_agg* agg;       /* [k] host memory, or NULL */
  scendp_agg_raw* agg_raw; /* [k] host memory, or NULL (un-finalized) */
} scendp_split_out;

/* Evaluates k_tours giant tours (k_tours x n customer ids, host memory,
 * each a permutation of 1..n) on every scenario of `sc`.  One launch covers
 * all (tour, scenario) pairs (SAA candidate batching).  With a communicator
 * attached (scendp_comm_*), the aggregates are all-reduced over all ranks
 * before they are returned. */
scendp_status scendp_split_eval(scendp_ctx* ctx, const scendp_routing* inst,
                                const int32_t* tours, uint32_t k_tours,
                                const scendp_scenarios* sc, uint32_t flags,
                                const scendp_split_out* out);

/* Argmin over finalized aggregates: smallest index with the minimal mean
 * (strict <, saa.cpp:134); -1 if no candidate has a finite mean. */
int64_t scendp_best_candidate(const scendp_agg* agg, uint32_t k);

/* ---- DSIRP order-up-to DP (oudp.hpp / oudp.cpp) ------------------------ */
typedef struct {
  int32_t capacity;            /* U in [0, 65535] */
  int32_t initial_inventory;   /* I0 in [0, U] */
  int32_t horizon;             /* H >= 1 (all customers of a call share H) */
  double holding;              /* h >= 0 */
  double stockout_multiplier;  /* rho > 1 */
  int32_t options;             /* R in [1, 256] */
  const double* fixed;         /* [H][R] (standard delivery model) */
  const double* unit;          /* [H][R] */
  int32_t delivery_tabular;    /* F_t(q) = table[t][q], table[t][0] == 0 */
  const double* delivery_table;/* [H][U+1] */
  int32_t holding_tabular;     /* hold = table[J] */
  const double* holding_table; /* [U+1] */
} scendp_customer;

#define SCENDP_DSIRP_COST_ONLY 0u
#define SCENDP_DSIRP_FULL 1u   /* + schedules (ScheduleResult, oudp.hpp:69-75) */
#define SCENDP_DSIRP_FP64 0x400u /* force the fp64 kernel (no exact-integer path) */

typedef struct {
  uint32_t mem_kind;       /* HOST / DEVICE (reference-like layout below) or
                              DEVICE_TILED ([c][m/32][H][32]) */
  double* totals;          /* [c][m]; error slots hold +inf */
  uint8_t* evaluated;      /* [c][m]; 0 = error slot */
  uint8_t* deliver;        /* FULL: [c][m][H] */
  int32_t* quantity;       /* FULL: [c][m][H] */
  int32_t* end_inventory;  /* FULL: [c][m][H] */
  int32_t* route_option;   /* FULL: [c][m][H] */
  scendp_agg* agg;         /* [n_customers] host memory, or NULL */
  scendp_agg_raw* agg_raw; /* [n_customers] or NULL */
} scendp_dsirp_out;

/* Customer c reads rows [c*H, (c+1)*H) of each scenario column. */
scendp_status scendp_dsirp_eval(scendp_ctx* ctx,
                                const scendp_customer* customers,
                                uint32_t n_customers,
                                const scendp_scenarios* sc, uint32_t flags,
                                const scendp_dsirp_out* out);

/* ---- device footprint model ----------------------------------------------
 * The device analogue of the reference's per-scenario footprint and batch
 * sizing (split_per_scenario_bytes, split.cpp:287-301; oudp.cpp:383-396;
 * adjust_batch_size / memory_footprint, engine.cpp:7-30): the scratch bytes a
 * call with these arguments allocates, split into a part independent of the
 * wave (tour / customer tables, aggregates, hand-off list floor, fallback
 * scratch, a pageable upload's staging chunk) and a part per scenario of a
 * wave (staged tiled input and its staging copy, outputs bound for pageable
 * host memory or the reference layout, hand-off bitmap), and the wave the
 * context's budget allows.  Caller-provided device outputs are not scratch
 * and are not counted. */
typedef struct {
  uint64_t fixed_bytes;
  uint64_t per_scenario_bytes;
  uint64_t wave;     /* scenarios per wave the call would use */
  uint64_t budget;   /* scratch_limit, else held scratch + free memory - 1/16 */
} scendp_footprint;

scendp_status scendp_split_footprint(scendp_ctx* ctx, const scendp_routing* inst,
                                     uint32_t k_tours, const scendp_scenarios* sc,
                                     uint32_t flags, const scendp_split_out* out,
                                     scendp_footprint* fp);
scendp_status scendp_dsirp_footprint(scendp_ctx* ctx, const scendp_customer* customers,
                                     uint32_t n_customers, const scendp_scenarios* sc,
                                     uint32_t flags, const scendp_dsirp_out* out,
                                     scendp_footprint* fp);

typedef struct {
  uint64_t scratch_bytes;  /* device bytes the context holds in scratch */
  uint64_t scratch_peak;   /* high-water mark of scratch_bytes */
  uint64_t device_free;    /* cudaMemGetInfo */
  uint64_t device_total;
  uint64_t oom_retries;    /* waves halved after an allocation failure */
  uint64_t last_wave;      /* wave size of the last split / DSIRP call */
  uint64_t tnormal_host_columns; /* tnormal columns the device could not
                              certify, regenerated with the host's libm */
} scendp_memory_info;

scendp_status scendp_ctx_memory(scendp_ctx* ctx, scendp_memory_info* info);

/* ---- K5: generic dense (min,+) stage sweep (minplus.hpp / minplus.cpp) ---
 * forward_sweep (minplus.cpp:94-102) of `batch` initial frontiers through one
 * shared chain of stage matrices: J_{s+1}[j] = min over options r, then
 * predecessors i, of A_s(i,j;r) + J_s[i] (the reference's scan order and
 * +inf semantics; minplus_apply_options, minplus.cpp:76-92).  Stage s is
 * [depth][rows][cols] row-major (MaskedTransition's slice-major entries);
 * rows of stage 0 == init_size and rows of stage s+1 == cols of stage s. */
typedef struct {
  uint64_t rows, cols, depth;
  const double* entries;  /* host or device, per mem_kind */
} scendp_minplus_stage;

#define SCENDP_MINPLUS_ALL_STAGES 0x1u /* out = every frontier: [B][init_size +
                                          sum cols], else the last: [B][cols] */
#define SCENDP_MINPLUS_EXACT_TIES 0x2u /* force the compare-select min (sign of
                                          zero ties as the reference); chosen
                                          automatically when a host input
                                          holds -0.0 */

/* init: [batch][init_size]; mem_kind SCENDP_MEM_HOST or SCENDP_MEM_DEVICE
 * applies to the stage entries, init and out alike.  Synchronous. */
scendp_status scendp_minplus_sweep(scendp_ctx* ctx,
                                   const scendp_minplus_stage* stages,
                                   uint32_t n_stages, const double* init,
                                   uint64_t init_size, uint64_t batch,
                                   uint32_t mem_kind, uint32_t flags,
                                   double* out);

/* ---- multi-GPU: one tiny NCCL all-reduce of the aggregates --------------
 * Scenario shards never exchange data; only the per-candidate raw
 * aggregates (16 x u64 each) are summed across ranks.  NCCL is loaded at
 * run time (dlopen libnccl.so.2). */
#define SCENDP_NCCL_UNIQUE_ID_BYTES 128
scendp_status scendp_nccl_unique_id(uint8_t out[SCENDP_NCCL_UNIQUE_ID_BYTES]);
/* multi-process: one context per process/GPU */
scendp_status scendp_comm_init_rank(scendp_ctx* ctx,
                                    const uint8_t id[SCENDP_NCCL_UNIQUE_ID_BYTES],
                                    int32_t nranks, int32_t rank);
/* single process driving several devices (ncclCommInitAll).  The contexts
 * of such a group must be driven concurrently, each from its own host
 * thread: a call on one context blocks until every rank joins its
 * all-reduce, so one thread calling scendp_split_eval on context 0, then 1,
 * ... deadlocks on context 0.  scendp_split_eval_multi / _dsirp_eval_multi
 * do the threading: one host thread per context, each evaluating its shard
 * (sc[i], out[i]); they return after every shard, with every context's
 * aggregates all-reduced (identical on all of them). */
scendp_status scendp_comm_init_all(scendp_ctx** ctxs, int32_t n);
scendp_status scendp_comm_destroy(scendp_ctx* ctx);
scendp_status scendp_split_eval_multi(scendp_ctx** ctxs, int32_t n, const scendp_routing* inst,
                                      const int32_t* tours, uint32_t k_tours,
                                      const scendp_scenarios* sc, uint32_t flags,
                                      const scendp_split_out* out);
scendp_status scendp_dsirp_eval_multi(scendp_ctx** ctxs, int32_t n,
                                      const scendp_customer* customers, uint32_t n_customers,
                                      const scendp_scenarios* sc, uint32_t flags,
                                      const scendp_dsirp_out* out);

/* ---- timing (bench) -----------------------------------------------------
 * CUDA events on the context stream. */
scendp_status scendp_timer_start(scendp_ctx* ctx);
scendp_status scendp_timer_stop(scendp_ctx* ctx, double* ms);
/* Hot-kernel statistics since the last reset, when SCENDP_CTX_KERNEL_TIMING
 * is set: launches of our kernels and event-timed milliseconds of the
 * dominant DP kernel. */
typedef struct {
  uint64_t launches;        /* all kernels this library launched */
  uint64_t dp_launches;     /* DP kernels (split / dsirp) */
  double dp_ms;             /* summed event time of the DP kernels */
  uint64_t gen_launches;
  double gen_ms;
  uint64_t h2d_bytes;       /* bytes this library copied host->device */
  uint64_t d2h_bytes;       /* bytes this library copied device->host */
} scendp_kernel_stats;
scendp_status scendp_kernel_stats_get(scendp_ctx* ctx, scendp_kernel_stats* s,
                                      int32_t reset);
/* Writes 2 x 126 MB over a scratch buffer to flush L2 between timed steps. */
scendp_status scendp_flush_l2(scendp_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SCENDP_CUDA_H */
