/*
 * scendp_oracle.h -- CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 engine:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The product (paper_2602_05179_b200/) never links or calls it.
 *
 * Every function restates one reference function and cites it
 * (paths relative to /root/reference/proj).  The restatement is pinned
 * against (a) the paper's golden examples App. A.3 / A.4 and (b) the real
 * reference library built from its own sources into oracle/_ref/ (see
 * oracle/Makefile and tests/test_oracle.py).
 */
#ifndef SCENDP_ORACLE_H
#define SCENDP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- random streams: include/scendp/scenario.hpp:12-57 ---------------- */
uint64_t or_mix64(uint64_t z);
uint64_t or_derive_stream(uint64_t seed, uint64_t tag, uint64_t index);
uint64_t or_next(uint64_t* state);
uint64_t or_next_below(uint64_t* state, uint64_t bound);
double or_next_unit(uint64_t* state);

enum { OR_UNIFORM = 0, OR_TNORMAL = 1, OR_POISSON = 2 };

/* DistributionSpec (scenario.hpp:60-76).  Poisson is the builder's new kind
 * (SURVEY Appendix A): inverse-CDF over a host table, one next_unit per draw.
 * For Poisson, `mean` holds lambda and lo must be 0. */
typedef struct {
  int32_t kind;
  int64_t lo, hi;
  double mean, stddev;
  uint64_t seed;
} or_dist;

/* Poisson CDF table P[0..hi], P[hi] forced to 1.0.  Returns hi+1. */
int64_t or_poisson_table(double lambda, int64_t hi, double* out);

/* DistributionSpec::sample (scenario.cpp:22-40) + poisson. */
uint32_t or_sample(const or_dist* d, const double* cdf, uint64_t* state);
/* generate_scenario_column (scenario.cpp:92-96). */
void or_generate_column(const or_dist* d, const double* cdf, uint64_t w,
                        uint32_t* out, uint64_t rows);
/* generate_scenarios (scenario.cpp:98-114) for columns [w0, w0+count),
 * reference (column-contiguous) layout. */
void or_generate_scenarios(const or_dist* d, const double* cdf, uint64_t rows,
                           uint64_t w0, uint64_t count, uint32_t* out);

/* make_random_instance (split.cpp:390-409): costs (n+2)^2 row-major. */
void or_make_random_instance(int32_t n, uint64_t seed, double* costs);

/* ---- split: split.cpp:24-126 ------------------------------------------ */
/* split_core_linear over fill_prefixes; V/cuts may be NULL.  *max_deque
 * (optional) receives the largest deque occupancy seen. */
double or_split_linear(int32_t n, int64_t Q, const double* costs,
                       const int32_t* tour, const uint32_t* demand, double* V,
                       int32_t* cuts, int32_t* max_deque);
/* split_core_quadratic over fill_prefixes; V/cuts may be NULL. */
double or_split_quadratic(int32_t n, int64_t Q, int32_t hard, double beta,
                          const double* costs, const int32_t* tour,
                          const uint32_t* demand, double* V, int32_t* cuts);
/* finalize_solution (split.cpp:120-126). */
int32_t or_route_count(int32_t n, const int32_t* cuts, double total);
/* brute_force_split (split.cpp:247-285). */
double or_brute_force_split(int32_t n, int64_t Q, int32_t hard, double beta,
                            const double* costs, const int32_t* tour,
                            const uint32_t* demand);

/* batched split over a reference-layout batch (m columns of n rows):
 * hard -> linear, penalized -> quadratic (split.cpp:303-371).  V/cuts/
 * route_count may be NULL. */
void or_split_batch(int32_t n, int64_t Q, int32_t hard, double beta,
                    const double* costs, const int32_t* tour,
                    const uint32_t* demand, uint64_t m, double* totals,
                    double* V, int32_t* cuts, int32_t* route_count);

/* ---- DSIRP OU DP: oudp.hpp / oudp.cpp --------------------------------- */
typedef struct {
  int32_t capacity;          /* U */
  int32_t initial_inventory; /* I0 */
  int32_t horizon;           /* H */
  double holding;            /* h */
  double stockout_multiplier;/* rho */
  int32_t options;           /* R */
  const double* fixed;       /* [H][R] */
  const double* unit;        /* [H][R] */
  int32_t delivery_tabular;
  const double* delivery_table; /* [H][U+1] */
  int32_t holding_tabular;
  const double* holding_table;  /* [U+1] */
} or_customer;

/* forward_pass + pick_terminal + assemble_schedule (oudp.cpp:40-132).
 * Returns 0 on success, -1 for an all-infinite frontier (logic_error). */
int32_t or_dsirp_scenario(const or_customer* c, const uint32_t* demands,
                          double* total, uint8_t* deliver, int32_t* quantity,
                          int32_t* end_inventory, int32_t* route_option);
/* simulate_schedule (oudp.cpp:325-345). */
double or_dsirp_simulate(const or_customer* c, const uint32_t* demands,
                         const uint8_t* deliver, const int32_t* route_option);
/* brute_force_schedule (oudp.cpp:347-381). */
double or_dsirp_brute_force(const or_customer* c, const uint32_t* demands);

/* run_batched's fixed-order aggregate (engine.hpp:195-211). */
void or_mean(const double* totals, const uint8_t* evaluated, uint64_t m,
             double* mean, int32_t* has_mean, uint64_t* finite,
             uint64_t* infeasible);

#ifdef __cplusplus
}
#endif
#endif
