"""GPU parity at the BASELINE shapes, against the real
reference (oracle/_ref) on the same box.

* C2 (split n=200, 10^6 scenarios, uniform:1:10): the reference's own
  generate_scenarios + batched_split_costs over all 10^6 columns; every total
  bit-exact, for the materialized (tiled) and the in-kernel-generated paths;
  the aggregate equals the exact mean of the totals.
* C3 (DSIRP 50 customers x 10^5, H=6): all 50 customers x all 10^5
  scenarios against the reference's per-customer batched_expected_cost,
  totals bit-exact and means within 1e-9, on the exact-integer and the fp64
  launch.
* C4 (200 customers x 10^6): all 200 customers on the first 20,000
  scenarios (prefix of the full launch; means of a 20,000-scenario call),
  three customers over all 10^6 (totals and means).
* C5 (1000 tours x 10^5, n=50, penalized beta=10): sampled tours' totals
  bit-exact over 10^5 and the first-minimum argmin consistent with the
  per-tour means; all 1000 tours on a 10,000-scenario prefix against the
  reference (totals, means, argmin).
* C2 float-cost twin over 10^6 (one launch and 300,000-scenario waves), C2
  full solutions and penalized totals on 200,000 scenarios, C3 full
  schedules, and K5 at the bench shape against forward_sweep.
"""
import os

import numpy as np
import pytest

from oracle import TAG_SCENARIO, UNIFORM
from oracle import Customer as RefCustomer
from paper_2602_05179_b200 import Customer, Distribution, RoutingInstance
from paper_2602_05179_b200 import _capi as A

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1


def test_c2_full_size_bit_exact(ctx, reference):
    n, m, Q = 200, 1_000_000, 100
    seed = reference.derive_stream(1, TAG_SCENARIO, 0)
    costs = reference.make_random_instance(n, 1)
    inst = RoutingInstance(n, Q, True, 0.0, costs)
    tour = np.arange(1, n + 1, dtype=np.int32)
    dem = reference.generate(UNIFORM, 1, 10, seed, n, 1, m)  # the reference's own batch
    ref_tot, (ref_mean, fc, ic) = reference.split_costs(n, Q, 1, 0.0, costs, tour, dem, THREADS)
    dist = Distribution("uniform", 1, 10, seed=seed)
    got_g = ctx.split_eval(inst, tour, dist, count=m)
    np.testing.assert_array_equal(got_g["totals"][0], ref_tot)
    got_h = ctx.split_eval(inst, tour, dem)
    np.testing.assert_array_equal(got_h["totals"][0], ref_tot)
    for got in (got_g, got_h):
        a = got["agg"][0]
        assert (a["finite_count"], a["infeasible_count"]) == (fc, ic)
        assert a["mean"] == ref_mean  # integral costs: every partial sum exact
    # the device-generated set is the reference's batch, byte for byte
    scen = ctx.gen_scenarios(dist, n, m, tiled=False)
    np.testing.assert_array_equal(scen.download(np.uint32, n * m).reshape(m, n), dem)
    scen.free()


def _c3_customers(nc, H, dyadic_only=False):
    """C3 pins (U=100, I0=50, h=1, rho=2, R=3, fixed 40+5r, unit 0.5+0.25r),
    perturbed per customer by dyadic offsets; unless dyadic_only, customer 1
    gets non-dyadic costs, which moves the whole launch onto the K3 fp64
    path (the exact-integer path needs every customer of a launch)."""
    ours, refs = [], []
    for c in range(nc):
        fixed = np.tile(40 + 5 * np.arange(3.0), (H, 1)) + (c % 7)
        unit = np.tile(0.5 + 0.25 * np.arange(3.0), (H, 1)) + 0.25 * (c % 3)
        h = 1.0
        if c == 1 and not dyadic_only:
            fixed = fixed + 0.1
            h = 0.7
        kw = dict(U=100, I0=50, H=H, h=h, rho=2.0, fixed=fixed, unit=unit)
        ours.append(Customer(**kw))
        refs.append(RefCustomer(**kw))
    return ours, refs


def _check_customer(got, c, ref_out, mean_check=True):
    tot, _, _, _, _, ev, (mean, fc, ic) = ref_out
    assert ev.all()
    np.testing.assert_array_equal(got["totals"][c], tot)
    if mean_check:
        a = got["agg"][c]
        assert a["finite_count"] == fc and a["infeasible_count"] == ic
        assert abs(a["mean"] - mean) <= 1e-9 * abs(mean)


@pytest.mark.parametrize("dyadic_only", [True, False])
def test_dsirp_c3_all_customers_bit_exact(ctx, reference, dyadic_only):
    """C3 in full: all 50 customers x all 10^5 scenarios against the
    reference's per-customer batched_expected_cost (oudp.cpp:398-438, the
    composition oracle of SURVEY 8c): every total bit-exact, every mean within
    1e-9; the exact-integer launch (dyadic pins) and the fp64 launch."""
    nc, m, H = 50, 100_000, 6
    ours, refs = _c3_customers(nc, H, dyadic_only)
    dist = Distribution("uniform", 0, 33, seed=7)
    scen = ctx.gen_scenarios(dist, nc * H, m)
    got = ctx.dsirp_eval(ours, (scen, A.MEM_DEVICE_TILED), count=m)
    scen.free()
    assert got["evaluated"].all()
    dem = reference.generate(UNIFORM, 0, 33, 7, nc, H, m)  # rows c*H + t
    for c in range(nc):
        _check_customer(got, c, reference.expected_cost(
            refs[c], np.ascontiguousarray(dem[:, c * H:(c + 1) * H]), THREADS))


@pytest.mark.parametrize("dyadic_only", [True, False])
def test_dsirp_c4_all_customers(ctx, reference, dyadic_only):
    """C4 (200 customers x 10^6 scenarios, one GPU): all 200 customers on the
    first 20,000 scenarios -- the prefix of the full 10^6 launch, and a
    20,000-scenario call whose per-customer means must match the reference's
    within 1e-9 -- plus three customers over all 10^6 scenarios (totals and
    means)."""
    nc, m, H, pre = 200, 1_000_000, 6, 20_000
    ours, refs = _c3_customers(nc, H, dyadic_only)
    dist = Distribution("uniform", 0, 33, seed=7)
    scen = ctx.gen_scenarios(dist, nc * H, m)
    full = ctx.dsirp_eval(ours, (scen, A.MEM_DEVICE_TILED), count=m)
    part = ctx.dsirp_eval(ours, (scen, A.MEM_DEVICE_TILED), count=pre)
    scen.free()
    assert full["evaluated"].all()
    dem = reference.generate(UNIFORM, 0, 33, 7, nc, H, pre)
    for c in range(nc):
        r = reference.expected_cost(refs[c], np.ascontiguousarray(dem[:, c * H:(c + 1) * H]),
                                    THREADS)
        np.testing.assert_array_equal(full["totals"][c][:pre], r[0])
        _check_customer(part, c, r)
    big = reference.generate(UNIFORM, 0, 33, 7, nc, H, m)
    for c in (0, 1, nc - 1):
        _check_customer(full, c, reference.expected_cost(
            refs[c], np.ascontiguousarray(big[:, c * H:(c + 1) * H]), THREADS))


def test_c5_saa_sweep_bit_exact(ctx, reference):
    n, m, K, Q, beta = 50, 100_000, 1000, 100, 10.0
    costs = reference.make_random_instance(n, 5)
    inst = RoutingInstance(n, Q, False, beta, costs)
    rng = np.random.default_rng(5)
    tours = np.stack([rng.permutation(n) + 1 for _ in range(K)]).astype(np.int32)
    seed = reference.derive_stream(5, TAG_SCENARIO, 0)
    dist = Distribution("uniform", 1, 10, seed=seed)
    scen = ctx.gen_scenarios(dist, n, m)
    got = ctx.split_eval(inst, tours, (scen, A.MEM_DEVICE_TILED), count=m)
    scen.free()
    means = np.array([a["mean"] for a in got["agg"]])
    best = got["best"]
    assert best == int(np.argmin(means))  # first minimum, saa.cpp:134
    dem = reference.generate(UNIFORM, 1, 10, seed, n, 1, m)
    for t in sorted({0, 1, 500, K - 1, best}):
        tot, (mean, fc, ic) = reference.split_costs(n, Q, 0, beta, costs, tours[t], dem, THREADS)
        np.testing.assert_array_equal(got["totals"][t], tot)
        assert got["agg"][t]["mean"] == mean


def test_c5_all_tours_prefix_bit_exact(ctx, reference):
    """C5's 1000 candidate tours, every one of them, on the first 10,000
    scenarios: totals bit-exact, means equal, and the selected candidate is
    the first minimum of the reference's per-tour means (SAA scorer,
    saa.cpp:127-134)."""
    n, m, K, Q, beta = 50, 10_000, 1000, 100, 10.0
    costs = reference.make_random_instance(n, 5)
    inst = RoutingInstance(n, Q, False, beta, costs)
    rng = np.random.default_rng(5)
    tours = np.stack([rng.permutation(n) + 1 for _ in range(K)]).astype(np.int32)
    seed = reference.derive_stream(5, TAG_SCENARIO, 0)
    got = ctx.split_eval(inst, tours, Distribution("uniform", 1, 10, seed=seed), count=m)
    dem = reference.generate(UNIFORM, 1, 10, seed, n, 1, m)
    ref_means = np.empty(K)
    for t in range(K):
        tot, (mean, fc, ic) = reference.split_costs(n, Q, 0, beta, costs, tours[t], dem, THREADS)
        np.testing.assert_array_equal(got["totals"][t], tot)
        assert got["agg"][t]["mean"] == mean and got["agg"][t]["finite_count"] == fc
        ref_means[t] = mean
    assert got["best"] == int(np.argmin(ref_means))


def _float_costs(n, seed):
    rng = np.random.default_rng(seed)
    c = rng.random((n + 2, n + 2)) * 20.0
    c = np.triu(c, 1)
    return c + c.T


def test_c2_float_costs_and_waves_bit_exact(ctx, reference):
    """C2 with non-integral costs (K1 fp64: the reference's association
    verbatim) over all 10^6 scenarios, in one launch and in waves of 300,000
    (BackendConfig::batch_size; not a multiple of the 32-scenario tile)."""
    n, m, Q = 200, 1_000_000, 100
    costs = _float_costs(n, 200)
    inst = RoutingInstance(n, Q, True, 0.0, costs)
    tour = (np.random.default_rng(4).permutation(n) + 1).astype(np.int32)
    seed = reference.derive_stream(3, TAG_SCENARIO, 0)
    dem = reference.generate(UNIFORM, 1, 10, seed, n, 1, m)
    ref_tot, (ref_mean, fc, ic) = reference.split_costs(n, Q, 1, 0.0, costs, tour, dem, THREADS)
    dist = Distribution("uniform", 1, 10, seed=seed)
    got = ctx.split_eval(inst, tour, dist, count=m)
    np.testing.assert_array_equal(got["totals"][0], ref_tot)
    a = got["agg"][0]
    assert (a["finite_count"], a["infeasible_count"]) == (fc, ic)
    assert abs(a["mean"] - ref_mean) <= 1e-9 * abs(ref_mean)
    ctx.set_max_batch(300_000)
    try:
        waves = ctx.split_eval(inst, tour, dist, count=m)
    finally:
        ctx.set_max_batch(0)
    np.testing.assert_array_equal(waves["totals"], got["totals"])
    assert waves["agg"] == got["agg"]


def test_c2_full_solutions_and_penalized_bit_exact(ctx, reference):
    """Full solutions (V, cuts, route counts) on 200,000 C2 scenarios, and the
    penalized (beta = 10) C2 totals -- K2-int -- on the same set."""
    n, m, Q = 200, 200_000, 100
    costs = reference.make_random_instance(n, 1)
    tour = np.arange(1, n + 1, dtype=np.int32)
    seed = reference.derive_stream(1, TAG_SCENARIO, 0)
    dem = reference.generate(UNIFORM, 1, 10, seed, n, 1, m)
    inst = RoutingInstance(n, Q, True, 0.0, costs)
    got = ctx.split_eval(inst, tour, dem, full=True)
    tot, V, cuts, rc, feas, _ = reference.expected_split(n, Q, 1, 0.0, costs, tour, dem, THREADS)
    np.testing.assert_array_equal(got["totals"][0], tot)
    np.testing.assert_array_equal(got["V"], V)
    np.testing.assert_array_equal(got["cuts"], cuts)
    np.testing.assert_array_equal(got["route_count"], rc)
    np.testing.assert_array_equal(got["feasible"], feas)
    pinst = RoutingInstance(n, Q, False, 10.0, costs)
    gp = ctx.split_eval(pinst, tour, dem)
    ptot, (pmean, _, _) = reference.split_costs(n, Q, 0, 10.0, costs, tour, dem, THREADS)
    np.testing.assert_array_equal(gp["totals"][0], ptot)
    assert gp["agg"][0]["mean"] == pmean


def test_c3_full_schedules_bit_exact(ctx, reference):
    """DSIRP schedules (deliver, quantity, end inventory, route option) for
    every scenario of two C3 customers, one of them on the fp64 path."""
    H, nc, m = 6, 50, 100_000
    ours, refs = _c3_customers(nc, H)
    dist = Distribution("uniform", 0, 33, seed=7)
    scen = ctx.gen_scenarios(dist, nc * H, m)
    got = ctx.dsirp_eval(ours, (scen, A.MEM_DEVICE_TILED), count=m, full=True)
    scen.free()
    dem = reference.generate(UNIFORM, 0, 33, 7, nc, H, m)
    for c in (0, 1):
        tot, dl, q, ei, ro, ev, _ = reference.expected_cost(refs[c], dem[:, c * H:(c + 1) * H],
                                                            THREADS)
        np.testing.assert_array_equal(got["totals"][c], tot)
        np.testing.assert_array_equal(got["deliver"][c], dl)
        np.testing.assert_array_equal(got["quantity"][c], q)
        np.testing.assert_array_equal(got["end_inventory"][c], ei)
        np.testing.assert_array_equal(got["route_option"][c], ro)


def test_k5_bench_shape_matches_forward_sweep(ctx, reference):
    """K5 at the bench shape (6 stages x 3 options x 101 x 101, 10^5
    frontiers): every final frontier entry against the reference's
    forward_sweep on 200 sampled frontiers (the frontiers are independent)."""
    rng = np.random.default_rng(11)
    stages = []
    for _ in range(6):
        st = np.floor(rng.random((3, 101, 101)) * 100.0)
        st[rng.random(st.shape) < 0.5] = np.inf
        stages.append(st)
    B = 100_000
    init = np.full((B, 101), np.inf)
    init[np.arange(B), rng.integers(0, 101, B)] = 0.0
    out = ctx.minplus_sweep(stages, init)
    for b in rng.choice(B, 200, replace=False):
        ref = reference.forward_sweep(stages, init[b])
        np.testing.assert_array_equal(out[b], ref[-101:])
