/*
 * scendp_oracle.c -- CPU restatement of the reference hot path (TEST ONLY).
 *
 * Header comment in scendp_oracle.h.  Built with -ffp-contract=off and no
 * -march so every double operation is a single IEEE-rounded op, exactly as
 * the reference's own Release build on baseline x86-64 (no FMA available).
 */
#include "scendp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9e3779b97f4a7c15ULL
#define OR_PI 0x1.921fb54442d18p+1 /* std::numbers::pi */
#define TAG_SCENARIO 0x5343454eULL /* scenario.hpp:49 */
#define TAG_INSTANCE 0x494e5354ULL /* scenario.hpp:51 */

static const double kInf = INFINITY;

/* scenario.hpp:12-17 */
uint64_t or_mix64(uint64_t z) {
  z += GAMMA;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* scenario.hpp:54-57 */
uint64_t or_derive_stream(uint64_t seed, uint64_t tag, uint64_t index) {
  return or_mix64(or_mix64(or_mix64(seed) ^ tag) ^ index);
}

/* SplitMix64::next (scenario.hpp:28-34): advancing the state by gamma and
 * finalising is mix64 of the pre-advance state. */
uint64_t or_next(uint64_t* state) {
  uint64_t out = or_mix64(*state);
  *state += GAMMA;
  return out;
}

/* scenario.hpp:37-40: 128-bit multiply-high. */
uint64_t or_next_below(uint64_t* state, uint64_t bound) {
  unsigned __int128 p = (unsigned __int128)or_next(state) * bound;
  return (uint64_t)(p >> 64);
}

/* scenario.hpp:43-45: (0,1]. */
double or_next_unit(uint64_t* state) {
  return (double)((or_next(state) >> 11) + 1) * 0x1.0p-53;
}

/* P[k] = sum_{j<=k} e^-l l^j / j!, summed in index
 * order, P[hi] forced to 1. */
int64_t or_poisson_table(double lambda, int64_t hi, double* out) {
  double term = exp(-lambda);
  double acc = 0.0;
  for (int64_t k = 0; k <= hi; ++k) {
    if (k > 0) term = term * lambda / (double)k;
    acc = acc + term;
    out[k] = acc;
  }
  out[hi] = 1.0;
  return hi + 1;
}

/* DistributionSpec::sample (scenario.cpp:22-40) */
uint32_t or_sample(const or_dist* d, const double* cdf, uint64_t* state) {
  if (d->kind == OR_UNIFORM) {
    uint64_t span = (uint64_t)(d->hi - d->lo) + 1;
    return (uint32_t)(d->lo + (int64_t)or_next_below(state, span));
  }
  if (d->kind == OR_POISSON) {
    double u = or_next_unit(state);
    int64_t k = 0;
    while (u > cdf[k]) ++k; /* cdf[hi] == 1 >= u terminates */
    return (uint32_t)k;
  }
  for (int attempt = 0; attempt < 64; ++attempt) {
    double u1 = or_next_unit(state);
    double u2 = or_next_unit(state);
    double z = sqrt(-2.0 * log(u1)) * cos(2.0 * OR_PI * u2);
    long long r = llround(d->mean + d->stddev * z);
    if (r >= d->lo && r <= d->hi) return (uint32_t)r;
  }
  long long r = llround(d->mean);
  if (r < d->lo) r = d->lo;
  if (r > d->hi) r = d->hi;
  return (uint32_t)r;
}

/* scenario.cpp:92-96 */
void or_generate_column(const or_dist* d, const double* cdf, uint64_t w,
                        uint32_t* out, uint64_t rows) {
  uint64_t st = or_derive_stream(d->seed, TAG_SCENARIO, w);
  for (uint64_t r = 0; r < rows; ++r) out[r] = or_sample(d, cdf, &st);
}

/* scenario.cpp:98-114 */
void or_generate_scenarios(const or_dist* d, const double* cdf, uint64_t rows,
                           uint64_t w0, uint64_t count, uint32_t* out) {
  for (uint64_t k = 0; k < count; ++k)
    or_generate_column(d, cdf, w0 + k, out + k * rows, rows);
}

/* split.cpp:390-409 */
void or_make_random_instance(int32_t n, uint64_t seed, double* costs) {
  int side = n + 2;
  memset(costs, 0, sizeof(double) * (size_t)side * side);
  uint64_t st = or_derive_stream(seed, TAG_INSTANCE, 0);
  for (int a = 0; a < side; ++a)
    for (int b = a + 1; b < side; ++b) {
      double c = (double)(1 + or_next_below(&st, 20));
      costs[a * side + b] = c;
      costs[b * side + a] = c;
    }
}

/* fill_prefixes (split.cpp:24-39): load by customer id, dist sequential. */
static void prefixes(int32_t n, const double* costs, const int32_t* tour,
                     const uint32_t* demand, double* dist, int64_t* load) {
  int side = n + 2;
  dist[0] = 0.0;
  load[0] = 0;
  if (n >= 1) dist[1] = 0.0;
  for (int i = 1; i <= n; ++i) {
    load[i] = load[i - 1] + demand[tour[i - 1] - 1];
    if (i >= 2) dist[i] = dist[i - 1] + costs[tour[i - 2] * side + tour[i - 1]];
  }
}

/* split_core_linear (split.cpp:77-118) */
double or_split_linear(int32_t n, int64_t Q, const double* costs,
                       const int32_t* tour, const uint32_t* demand, double* V,
                       int32_t* cuts, int32_t* max_deque) {
  int side = n + 2;
  double* dist = malloc(sizeof(double) * (n + 2));
  int64_t* load = malloc(sizeof(int64_t) * (n + 2));
  double* f = malloc(sizeof(double) * (n + 1));
  int* dq = malloc(sizeof(int) * (n + 2));
  prefixes(n, costs, tour, demand, dist, load);
  int head = 0, tail = 0, peak = 1;
  double vi = 0.0;
  if (V) V[0] = 0.0;
  if (cuts) cuts[0] = 0;
  f[0] = (0.0 + costs[0 * side + tour[0]]) - dist[1];
  dq[tail++] = 0;
  for (int i = 1; i <= n; ++i) {
    while (head < tail && load[i] - load[dq[head]] > Q) ++head;
    int32_t cut;
    if (head >= tail) {
      vi = kInf;
      cut = -1;
    } else {
      int p = dq[head];
      vi = (f[p] + dist[i]) + costs[tour[i - 1] * side + (n + 1)];
      cut = vi < kInf ? p : -1;
    }
    if (V) V[i] = vi;
    if (cuts) cuts[i] = cut;
    if (i < n) {
      double fi = (vi + costs[0 * side + tour[i]]) - dist[i + 1];
      while (tail > head && f[dq[tail - 1]] > fi) --tail;
      dq[tail++] = i;
      f[i] = fi;
      if (tail - head > peak) peak = tail - head;
    }
  }
  if (max_deque) *max_deque = peak;
  free(dist); free(load); free(f); free(dq);
  return vi;
}

/* split_core_quadratic (split.cpp:45-75) */
double or_split_quadratic(int32_t n, int64_t Q, int32_t hard, double beta,
                          const double* costs, const int32_t* tour,
                          const uint32_t* demand, double* V, int32_t* cuts) {
  int side = n + 2;
  double* dist = malloc(sizeof(double) * (n + 2));
  int64_t* load = malloc(sizeof(int64_t) * (n + 2));
  double* v = malloc(sizeof(double) * (n + 1));
  prefixes(n, costs, tour, demand, dist, load);
  v[0] = 0.0;
  if (cuts) cuts[0] = 0;
  for (int i = 1; i <= n; ++i) {
    double di = dist[i];
    double ret = costs[tour[i - 1] * side + (n + 1)];
    double best = kInf;
    int32_t bestp = -1;
    for (int p = 0; p < i; ++p) {
      if (!(v[p] < kInf)) continue;
      int64_t excess = load[i] - load[p] - Q;
      double fp = (v[p] + costs[0 * side + tour[p]]) - dist[p + 1];
      double cand = (fp + di) + ret;
      if (excess > 0) {
        if (hard) continue;
        cand += beta * (double)excess;
      }
      if (cand < best) {
        best = cand;
        bestp = p;
      }
    }
    v[i] = best;
    if (cuts) cuts[i] = bestp;
  }
  double total = v[n];
  if (V) memcpy(V, v, sizeof(double) * (n + 1));
  free(dist); free(load); free(v);
  return total;
}

/* finalize_solution (split.cpp:120-126) */
int32_t or_route_count(int32_t n, const int32_t* cuts, double total) {
  if (!(total < kInf)) return 0;
  int32_t rc = 0;
  for (int i = n; i > 0; i = cuts[i]) ++rc;
  return rc;
}

/* brute_force_split (split.cpp:247-285) */
double or_brute_force_split(int32_t n, int64_t Q, int32_t hard, double beta,
                            const double* costs, const int32_t* tour,
                            const uint32_t* demand) {
  int side = n + 2;
  double best = kInf;
  uint64_t patterns = 1ULL << (n - 1);
  for (uint64_t mask = 0; mask < patterns; ++mask) {
    double total = 0.0;
    int ok = 1, start = 1;
    for (int i = 1; i <= n && ok; ++i) {
      int ends = (i == n) || ((mask >> (i - 1)) & 1);
      if (!ends) continue;
      double c = costs[0 * side + tour[start - 1]];
      int64_t load = 0;
      for (int k = start; k <= i; ++k) {
        load += demand[tour[k - 1] - 1];
        if (k > start) c += costs[tour[k - 2] * side + tour[k - 1]];
      }
      c += costs[tour[i - 1] * side + (n + 1)];
      if (load > Q) {
        if (hard) { ok = 0; break; }
        c += beta * (double)(load - Q);
      }
      total += c;
      start = i + 1;
    }
    if (ok && total < best) best = total;
  }
  return best;
}

void or_split_batch(int32_t n, int64_t Q, int32_t hard, double beta,
                    const double* costs, const int32_t* tour,
                    const uint32_t* demand, uint64_t m, double* totals,
                    double* V, int32_t* cuts, int32_t* route_count) {
  int32_t* tmp_cuts = malloc(sizeof(int32_t) * (n + 1));
  for (uint64_t w = 0; w < m; ++w) {
    const uint32_t* col = demand + w * (uint64_t)n;
    double* vw = V ? V + w * (uint64_t)(n + 1) : NULL;
    int32_t* cw = cuts ? cuts + w * (uint64_t)(n + 1) : tmp_cuts;
    double t = hard ? or_split_linear(n, Q, costs, tour, col, vw, cw, NULL)
                    : or_split_quadratic(n, Q, 0, beta, costs, tour, col, vw, cw);
    if (totals) totals[w] = t;
    if (route_count) route_count[w] = or_route_count(n, cw, t);
  }
  free(tmp_cuts);
}

/* ---- DSIRP ------------------------------------------------------------ */

/* DeliveryCostModel::cost (oudp.hpp:41-46) */
static double delivery_cost(const or_customer* c, int day, int r, int q) {
  if (q == 0) return 0.0;
  if (c->delivery_tabular)
    return c->delivery_table[(day - 1) * (c->capacity + 1) + q];
  return c->fixed[(day - 1) * c->options + r] +
         c->unit[(day - 1) * c->options + r] * (double)q;
}

/* HoldingPenaltyModel::cost (oudp.hpp:58-62) */
static double holding_cost(const or_customer* c, int j, int s) {
  if (c->holding_tabular) return c->holding_table[j];
  return c->holding * (double)j + c->stockout_multiplier * c->holding * (double)s;
}

static int imax(int a, int b) { return a > b ? a : b; }

/* forward_pass (oudp.cpp:40-87), pick_terminal (94-106),
 * assemble_schedule (108-132); backpointers packed as in oudp.cpp:17-24. */
int32_t or_dsirp_scenario(const or_customer* c, const uint32_t* demands,
                          double* total, uint8_t* deliver, int32_t* quantity,
                          int32_t* end_inventory, int32_t* route_option) {
  int S = c->capacity + 1, H = c->horizon, U = c->capacity;
  double* a = malloc(sizeof(double) * S);
  double* b = malloc(sizeof(double) * S);
  uint32_t* bp = calloc((size_t)H * S, sizeof(uint32_t));
  for (int s = 0; s < S; ++s) a[s] = kInf;
  a[c->initial_inventory] = 0.0;
  for (int t = 1; t <= H; ++t) {
    int d = (int)demands[t - 1];
    uint32_t* bpt = bp + (size_t)(t - 1) * S;
    for (int s = 0; s < S; ++s) b[s] = kInf;
    for (int i = 0; i < S; ++i) {
      if (!(a[i] < kInf)) continue;
      int j = imax(0, i - d), sh = imax(0, d - i);
      double cand = a[i] + (delivery_cost(c, t, 0, 0) + holding_cost(c, j, sh));
      if (cand < b[j]) { b[j] = cand; bpt[j] = (uint32_t)i; }
    }
    int j1 = imax(0, U - d), s1 = imax(0, d - U);
    for (int r = 0; r < c->options; ++r)
      for (int i = 0; i < U; ++i) {
        if (!(a[i] < kInf)) continue;
        double cand = a[i] + (delivery_cost(c, t, r, U - i) + holding_cost(c, j1, s1));
        if (cand < b[j1]) {
          b[j1] = cand;
          bpt[j1] = (uint32_t)i | (1u << 16) | ((uint32_t)r << 17);
        }
      }
    double* sw = a; a = b; b = sw;
  }
  int js = -1;
  double best = kInf;
  for (int j = 0; j < S; ++j)
    if (a[j] < best) { best = a[j]; js = j; }
  int32_t rc = 0;
  if (js < 0) {
    rc = -1;
  } else {
    *total = best;
    int j = js;
    for (int t = H; t >= 1; --t) {
      uint32_t e = bp[(size_t)(t - 1) * S + j];
      int dl = (int)((e >> 16) & 1);
      if (end_inventory) end_inventory[t - 1] = j;
      if (deliver) deliver[t - 1] = (uint8_t)dl;
      if (route_option) route_option[t - 1] = dl ? (int32_t)(e >> 17) : 0;
      j = (int)(e & 0xffff);
    }
    if (quantity && deliver && end_inventory) {
      int inv = c->initial_inventory;
      for (int t = 1; t <= H; ++t) {
        quantity[t - 1] = deliver[t - 1] ? U - inv : 0;
        inv = end_inventory[t - 1];
      }
    }
  }
  free(a); free(b); free(bp);
  return rc;
}

/* simulate_schedule (oudp.cpp:325-345) */
double or_dsirp_simulate(const or_customer* c, const uint32_t* demands,
                         const uint8_t* deliver, const int32_t* route_option) {
  double total = 0.0;
  int inv = c->initial_inventory;
  for (int t = 1; t <= c->horizon; ++t) {
    int d = (int)demands[t - 1];
    int q = deliver[t - 1] ? c->capacity - inv : 0;
    int r = deliver[t - 1] ? route_option[t - 1] : 0;
    int j = imax(0, inv + q - d), s = imax(0, d - inv - q);
    total += delivery_cost(c, t, r, q) + holding_cost(c, j, s);
    inv = j;
  }
  return total;
}

/* brute_force_schedule (oudp.cpp:347-381) */
double or_dsirp_brute_force(const or_customer* c, const uint32_t* demands) {
  double best = kInf;
  uint32_t patterns = 1u << c->horizon;
  for (uint32_t mask = 0; mask < patterns; ++mask) {
    double total = 0.0;
    int inv = c->initial_inventory;
    for (int t = 1; t <= c->horizon; ++t) {
      int d = (int)demands[t - 1];
      int z = (mask >> (t - 1)) & 1;
      int q = z ? c->capacity - inv : 0;
      double f = delivery_cost(c, t, 0, q);
      for (int r = 1; r < c->options && q > 0; ++r) {
        double g = delivery_cost(c, t, r, q);
        if (g < f) f = g;
      }
      int j = imax(0, inv + q - d), s = imax(0, d - inv - q);
      total += f + holding_cost(c, j, s);
      inv = j;
    }
    if (total < best) best = total;
  }
  return best;
}

/* engine.hpp:195-211 */
void or_mean(const double* totals, const uint8_t* evaluated, uint64_t m,
             double* mean, int32_t* has_mean, uint64_t* finite,
             uint64_t* infeasible) {
  double sum = 0.0;
  uint64_t fc = 0, ic = 0;
  for (uint64_t w = 0; w < m; ++w) {
    if (evaluated && !evaluated[w]) continue;
    if (totals[w] < kInf) { sum += totals[w]; ++fc; } else { ++ic; }
  }
  *finite = fc;
  *infeasible = ic;
  *has_mean = fc > 0;
  *mean = fc > 0 ? sum / (double)fc : 0.0;
}
