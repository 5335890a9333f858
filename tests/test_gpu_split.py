"""GPU parity: split evaluators (K1 linear, K2 quadratic, K6 multi-tour)
against the real reference (oracle/_ref) and the C restatement (oracle/).

Bar (BASELINE.json): per-scenario totals, V and cuts, route counts
bit-exact; aggregate mean within 1e-9 relative (bit-exact for integer costs).
"""
import numpy as np
import pytest

from oracle import POISSON, TAG_SCENARIO, UNIFORM
from paper_2602_05179_b200 import Distribution, RoutingInstance

pytestmark = pytest.mark.gpu

MEAN_RTOL = 1e-9


def float_instance(n, Q, seed, hard=True, beta=0.0):
    """random_float_instance (oracle.cpp:41-57 style): non-integral costs pin
    the fp64 operation order."""
    rng = np.random.default_rng(seed)
    c = rng.random((n + 2, n + 2)) * 20.0
    c = np.triu(c, 1)
    c = c + c.T
    return RoutingInstance(n, Q, hard, beta, c)


def rand_tour(n, seed):
    return (np.random.default_rng(seed).permutation(n) + 1).astype(np.int32)


def check_mean(agg, ref_mean):
    assert agg["mean"] is not None
    assert abs(agg["mean"] - ref_mean) <= MEAN_RTOL * abs(ref_mean)


@pytest.mark.parametrize("n,m", [(50, 1024), (200, 4096), (7, 333)])
@pytest.mark.parametrize("costs", ["int", "float"])
def test_split_costs_hard_matches_reference(ctx, oracle, reference, n, m, costs):
    seed = oracle.derive_stream(1, TAG_SCENARIO, 0)
    dem = oracle.generate(UNIFORM, 1, 10, seed, n, m)
    if costs == "int":
        inst = RoutingInstance(n, 100, True, 0.0, oracle.make_random_instance(n, 1))
    else:
        inst = float_instance(n, 100, n)
    for tour in (np.arange(1, n + 1, dtype=np.int32), rand_tour(n, 3)):
        got = ctx.split_eval(inst, tour, dem)
        ref_tot, (ref_mean, fc, ic) = reference.split_costs(n, 100, 1, 0.0, inst.costs, tour, dem)
        np.testing.assert_array_equal(got["totals"][0], ref_tot)
        a = got["agg"][0]
        assert a["finite_count"] == fc and a["infeasible_count"] == ic
        check_mean(a, ref_mean)
        if costs == "int":
            assert a["mean"] == ref_mean


def test_split_costs_tiled_and_fused_match(ctx, oracle):
    n, m = 200, 10_000
    inst = RoutingInstance(n, 100, True, 0.0, oracle.make_random_instance(n, 1))
    tour = np.arange(1, n + 1, dtype=np.int32)
    dist = Distribution("uniform", 1, 10, seed=oracle.derive_stream(1, TAG_SCENARIO, 0))
    host = oracle.generate(UNIFORM, 1, 10, dist.seed, n, m)
    want = oracle.split_batch(n, 100, 1, 0.0, inst.costs, tour, host)
    tiled = ctx.gen_scenarios(dist, n, m)
    got_t = ctx.split_eval(inst, tour, (tiled, 2), count=m)
    got_g = ctx.split_eval(inst, tour, dist, count=m)
    np.testing.assert_array_equal(got_t["totals"][0], want)
    np.testing.assert_array_equal(got_g["totals"][0], want)
    assert got_t["agg"][0] == got_g["agg"][0]
    tiled.free()


def test_split_full_matches_reference(ctx, oracle, reference):
    n, m = 50, 1024
    for costs in ("int", "float"):
        inst = (RoutingInstance(n, 100, True, 0.0, oracle.make_random_instance(n, 1))
                if costs == "int" else float_instance(n, 100, 5))
        seed = oracle.derive_stream(2, TAG_SCENARIO, 0)
        dem = oracle.generate(POISSON, 0, 47, seed, n, m, mean=5.0)
        tour = rand_tour(n, 9)
        got = ctx.split_eval(inst, tour, dem, full=True)
        tot, V, cuts, rc, feas, (mean, fc, ic) = reference.expected_split(
            n, 100, 1, 0.0, inst.costs, tour, dem)
        np.testing.assert_array_equal(got["totals"][0], tot)
        np.testing.assert_array_equal(got["V"], V)
        np.testing.assert_array_equal(got["cuts"], cuts)
        np.testing.assert_array_equal(got["route_count"], rc)
        np.testing.assert_array_equal(got["feasible"], feas)
        check_mean(got["agg"][0], mean)


@pytest.mark.parametrize("n", [10, 50, 120])
def test_split_penalized_matches_reference(ctx, oracle, reference, n):
    m = 2048
    seed = oracle.derive_stream(3, TAG_SCENARIO, 0)
    dem = oracle.generate(UNIFORM, 1, 10, seed, n, m)
    for inst in (RoutingInstance(n, 40, False, 10.0, oracle.make_random_instance(n, 4)),
                 float_instance(n, 40, 11, hard=False, beta=2.75)):
        tour = rand_tour(n, n)
        got = ctx.split_eval(inst, tour, dem, full=True)
        tot, V, cuts, rc, feas, (mean, fc, ic) = reference.expected_split(
            n, 40, 0, inst.penalty_beta, inst.costs, tour, dem)
        np.testing.assert_array_equal(got["totals"][0], tot)
        np.testing.assert_array_equal(got["V"], V)
        np.testing.assert_array_equal(got["cuts"], cuts)
        np.testing.assert_array_equal(got["route_count"], rc)
        check_mean(got["agg"][0], mean)


def test_multi_tour_candidates_match_per_tour_calls(ctx, oracle, reference):
    """K6: K tours in one launch == K reference calls; argmin = first min."""
    n, m, K = 50, 1000, 33
    inst = RoutingInstance(n, 100, False, 10.0, oracle.make_random_instance(n, 7))
    seed = oracle.derive_stream(7, TAG_SCENARIO, 0)
    dem = oracle.generate(UNIFORM, 1, 10, seed, n, m)
    tours = np.stack([rand_tour(n, 100 + q) for q in range(K)])
    tours[5] = tours[3]  # duplicate: ties resolve to the first index
    got = ctx.split_eval(inst, tours, dem)
    means = []
    for q in range(K):
        tot, (mean, fc, ic) = reference.split_costs(n, 100, 0, 10.0, inst.costs, tours[q], dem)
        np.testing.assert_array_equal(got["totals"][q], tot)
        assert got["agg"][q]["mean"] == mean  # integer costs -> exact
        means.append(mean)
    assert got["best"] == int(np.argmin(means))


def test_edge_cases(ctx, oracle, reference):
    # infeasible scenarios (demand > Q), zero demands (deque growth), n = 1
    n = 30
    inst = RoutingInstance(n, 10, True, 0.0, oracle.make_random_instance(n, 2))
    tour = rand_tour(n, 1)
    rng = np.random.default_rng(0)
    dem = rng.integers(0, 4, size=(512, n)).astype(np.uint32)
    dem[::7, 3] = 11  # > Q: infeasible
    dem[1::5] = 0     # all-zero demand: one long window, deque overflow path
    got = ctx.split_eval(inst, tour, dem, full=True)
    tot, V, cuts, rc, feas, (mean, fc, ic) = reference.expected_split(
        n, 10, 1, 0.0, inst.costs, tour, dem)
    np.testing.assert_array_equal(got["totals"][0], tot)
    np.testing.assert_array_equal(got["V"], V)
    np.testing.assert_array_equal(got["cuts"], cuts)
    assert got["agg"][0]["infeasible_count"] == ic > 0
    assert got["agg"][0]["finite_count"] == fc
    # n = 1
    inst1 = RoutingInstance(1, 5, True, 0.0, oracle.make_random_instance(1, 3))
    d1 = np.array([[3], [6], [0]], np.uint32)
    g1 = ctx.split_eval(inst1, [1], d1, full=True)
    t1, V1, c1, *_ = reference.expected_split(1, 5, 1, 0.0, inst1.costs, np.array([1], np.int32), d1)
    np.testing.assert_array_equal(g1["totals"][0], t1)
    np.testing.assert_array_equal(g1["cuts"], c1)


def test_paper_golden_a3(ctx):
    """PAPER.md App. A.3: V = (0,4,4,8), routes [s1 s2], [s3]."""
    c4 = np.array([[0, 1, 2, 3], [1, 0, 1, 2], [2, 1, 0, 1], [3, 2, 1, 0]], np.float64)
    c = np.zeros((5, 5))
    c[:4, :4] = c4
    c[:4, 4] = [0, 3, 2, 1]
    c[4, :4] = [0, 3, 2, 1]
    inst = RoutingInstance(3, 5, True, 0.0, c)
    got = ctx.split_eval(inst, [1, 2, 3], np.array([[2, 3, 4]], np.uint32), full=True)
    np.testing.assert_array_equal(got["V"][0], [0, 4, 4, 8])
    np.testing.assert_array_equal(got["cuts"][0], [0, 0, 0, 2])
    assert got["route_count"][0] == 2


def test_waves_do_not_change_results(oracle):
    from paper_2602_05179_b200 import Context
    n, m = 60, 3000
    inst = RoutingInstance(n, 50, False, 3.0, oracle.make_random_instance(n, 9))
    dem = oracle.generate(UNIFORM, 0, 12, 77, n, m)
    tour = rand_tour(n, 4)
    with Context(0) as a, Context(0, max_batch=96) as b:
        ra = a.split_eval(inst, tour, dem)
        rb = b.split_eval(inst, tour, dem)
    np.testing.assert_array_equal(ra["totals"], rb["totals"])
    assert ra["agg"] == rb["agg"]


def test_penalized_exact_path_edges(ctx, oracle, reference):
    """K2-int (O(n) penalized form) fall-backs: windows longer than the
    position ring (zero demands), loads beyond the exact int32 range, beta=0,
    and ties between the window and the penalized prefix."""
    n = 60
    rng = np.random.default_rng(12)
    tour = rand_tour(n, 2)
    dem = rng.integers(0, 12, size=(700, n)).astype(np.uint32)
    dem[::5] = 0                       # every route fits: window = whole prefix
    dem[1::9, 7] = 3_000_000_000       # beta * load leaves the int32 range
    dem[2::9] = 1                      # long windows
    for beta in (0.0, 1.0, 10.0, 37.0):
        inst = RoutingInstance(n, 20, False, beta, oracle.make_random_instance(n, 3))
        got = ctx.split_eval(inst, tour, dem, full=True)
        tot, V, cuts, rc, feas, (mean, fc, ic) = reference.expected_split(
            n, 20, 0, beta, inst.costs, tour, dem)
        np.testing.assert_array_equal(got["totals"][0], tot)
        np.testing.assert_array_equal(got["V"], V)
        np.testing.assert_array_equal(got["cuts"], cuts)
        np.testing.assert_array_equal(got["route_count"], rc)
        check_mean(got["agg"][0], mean)
    # ties: all-equal costs make many candidates coincide
    c = np.ones((n + 2, n + 2)) * 4.0
    np.fill_diagonal(c, 0.0)
    inst = RoutingInstance(n, 15, False, 2.0, c)
    d2 = rng.integers(1, 6, size=(300, n)).astype(np.uint32)
    got = ctx.split_eval(inst, tour, d2, full=True)
    tot, V, cuts, rc, feas, agg = reference.expected_split(n, 15, 0, 2.0, c, tour, d2)
    np.testing.assert_array_equal(got["cuts"], cuts)
    np.testing.assert_array_equal(got["totals"][0], tot)


@pytest.mark.parametrize("full", [False, True])
def test_penalized_long_windows_cost_only_and_c2_shape(ctx, oracle, reference, full):
    """Windows longer than K2-int's position ring take the generic kernel's
    O(n) penalized form (not the quadratic one); C2-shaped penalized batch."""
    n = 200
    inst = RoutingInstance(n, 100, False, 10.0, oracle.make_random_instance(n, 1))
    seed = oracle.derive_stream(1, TAG_SCENARIO, 0)
    dem = oracle.generate(UNIFORM, 1, 10, seed, n, 3000)
    dem[::7] = oracle.generate(UNIFORM, 0, 2, seed + 1, n, dem[::7].shape[0])  # windows ~100
    tour = rand_tour(n, 9)
    got = ctx.split_eval(inst, tour, dem, full=full)
    if full:
        tot, V, cuts, rc, feas, (mean, fc, ic) = reference.expected_split(
            n, 100, 0, 10.0, inst.costs, tour, dem)
        np.testing.assert_array_equal(got["V"], V)
        np.testing.assert_array_equal(got["cuts"], cuts)
        np.testing.assert_array_equal(got["route_count"], rc)
    else:
        tot, (mean, fc, ic) = reference.split_costs(n, 100, 0, 10.0, inst.costs, tour, dem)
    np.testing.assert_array_equal(got["totals"][0], tot)
    assert got["agg"][0]["mean"] == mean


def test_pinned_host_totals_are_written_in_place(ctx, oracle):
    """Host totals in page-locked memory are stored by the kernels directly
    (no D2H copy); results equal the pageable-buffer path."""
    from paper_2602_05179_b200 import Customer, pinned_empty
    n, m, k = 50, 5000, 3
    inst = RoutingInstance(n, 100, True, 0.0, oracle.make_random_instance(n, 1))
    tours = np.stack([rand_tour(n, s) for s in range(k)])
    dem = oracle.generate(UNIFORM, 1, 10, 5, n, m)
    want = ctx.split_eval(inst, tours, dem)
    pin = pinned_empty(k * m, np.float64)
    pin[:] = -1.0
    ctx.kernel_stats(reset=True)
    got = ctx.split_eval(inst, tours, dem, host_totals=pin)
    st = ctx.kernel_stats(reset=True)
    np.testing.assert_array_equal(pin.reshape(k, m), want["totals"])
    assert got["agg"] == want["agg"]
    assert st["d2h_bytes"] >= k * m * 8
    H = 6
    custs = [Customer(U=60, I0=30, H=H, fixed=np.full((H, 2), 20.0), unit=np.full((H, 2), 0.5))
             for _ in range(2)]
    dd = oracle.generate(UNIFORM, 0, 25, 3, 2 * H, 999)
    want = ctx.dsirp_eval(custs, dd)
    pin2 = pinned_empty(2 * 999, np.float64)
    ctx.dsirp_eval(custs, dd, host_totals=pin2)
    np.testing.assert_array_equal(pin2.reshape(2, 999), want["totals"])


@pytest.mark.parametrize("mode", ["hard", "penalized"])
def test_c1_poisson_generated_in_kernel(ctx, oracle, reference, mode):
    """BASELINE C1: n=50, Q=100, 1,024 seeded Poisson(5) scenarios generated
    inside the DP kernel (GENERATED source) == the reference evaluating the
    same scenarios (the restated sampler over the same streams)."""
    from paper_2602_05179_b200 import poisson_hi
    n, m, lam = 50, 1024, 5.0
    hi = poisson_hi(lam)
    seed = oracle.derive_stream(1, TAG_SCENARIO, 0)
    hard = mode == "hard"
    costs = oracle.make_random_instance(n, 1)
    inst = RoutingInstance(n, 100, hard, 0.0 if hard else 10.0, costs)
    tours = [np.arange(1, n + 1, dtype=np.int32), rand_tour(n, 3)]
    dist = Distribution("poisson", 0, hi, mean=lam, seed=seed)
    dem = oracle.generate(POISSON, 0, hi, seed, n, m, mean=lam)
    for tour in tours:
        got = ctx.split_eval(inst, tour, dist, count=m)
        tot, (mean, fc, ic) = reference.split_costs(n, 100, 1 if hard else 0, inst.penalty_beta,
                                                    costs, tour, dem)
        np.testing.assert_array_equal(got["totals"][0], tot)
        assert got["agg"][0]["mean"] == mean


@pytest.mark.parametrize("hard", [False, True])
def test_overflow_beyond_list_capacity(ctx, oracle, reference, hard):
    """Every scenario leaves the fast kernels (demands 1..2 with Q = 100: the
    penalized capacity window outgrows the 32-position ring; hard: the
    window-start test on a 50-customer tour with tiny demands never evicts
    and the deque outgrows its ring on increasing f) -- 2 x 60,000 items, far
    beyond the 65,536-entry overflow list, so most take the bitmap path."""
    n, m, Q = 50, 60_000, 100
    costs = oracle.make_random_instance(n, 9)
    if hard:
        # f(p) increasing along the tour: every predecessor stays in the deque
        c = np.zeros((n + 2, n + 2))
        for i in range(n + 2):
            for j in range(n + 2):
                c[i, j] = abs(i - j) if i != j else 0.0
        costs = c
    inst = RoutingInstance(n, Q, hard, 0.0 if hard else 10.0, costs)
    # a DSIRP call with reference-layout schedules first: its staging
    # buffers must not share memory with the hand-off bitmap (regression)
    from paper_2602_05179_b200 import Customer
    H = 6
    cust = Customer(U=100, I0=50, H=H, fixed=np.tile(40 + 5 * np.arange(3.0), (H, 1)),
                    unit=np.tile(0.5 + 0.25 * np.arange(3.0), (H, 1)))
    ctx.dsirp_eval([cust], oracle.generate(UNIFORM, 0, 33, 5, H, 20_000), full=True)
    tours = np.stack([np.arange(1, n + 1), np.random.default_rng(2).permutation(n) + 1])
    tours = tours.astype(np.int32)
    dem = oracle.generate(UNIFORM, 1, 2, 99, n, m)
    got = ctx.split_eval(inst, tours, dem)
    for t in range(2):
        tot, (mean, fc, ic) = reference.split_costs(n, Q, int(hard), inst.penalty_beta, costs, tours[t],
                                                    dem, 16)
        np.testing.assert_array_equal(got["totals"][t], tot)
        a = got["agg"][t]
        assert (a["finite_count"], a["infeasible_count"]) == (fc, ic)
        check_mean(a, mean)
    # a second call reuses the (cleared) bitmap
    again = ctx.split_eval(inst, tours, dem)
    np.testing.assert_array_equal(again["totals"], got["totals"])
    assert again["agg"] == got["agg"]


def test_scratch_limit_caps_waves(oracle):
    """scendp_opts.scratch_limit (the memory_budget analogue) bounds the
    per-wave staged scenario copy: results are unchanged, split and DSIRP."""
    from paper_2602_05179_b200 import Context, Customer
    n, m = 70, 5000
    inst = RoutingInstance(n, 60, True, 0.0, oracle.make_random_instance(n, 4))
    dem = oracle.generate(UNIFORM, 1, 9, 21, n, m)
    tour = rand_tour(n, 6)
    H = 6
    cust = Customer(U=50, I0=20, H=H, fixed=np.full((H, 2), 9.0), unit=np.full((H, 2), 0.75))
    dd = oracle.generate(UNIFORM, 0, 30, 8, 2 * H, m)
    with Context(0) as a, Context(0, scratch_limit=4 * n * 100) as b:
        ra, rb = a.split_eval(inst, tour, dem), b.split_eval(inst, tour, dem)
        da, db = a.dsirp_eval([cust, cust], dd, full=True), b.dsirp_eval([cust, cust], dd, full=True)
    np.testing.assert_array_equal(ra["totals"], rb["totals"])
    assert ra["agg"] == rb["agg"]
    for key in ("totals", "deliver", "quantity", "end_inventory", "route_option"):
        np.testing.assert_array_equal(da[key], db[key])
    assert da["agg"] == db["agg"]


def test_pageable_upload_narrow_and_wide_chunks(ctx, oracle):
    """Pageable host sets above 16 MB are staged in 64 MB chunks; demands
    below 256 cross PCIe as bytes.  A wide value in a later chunk switches
    the rest of the call to u32; a wide value in the first chunk keeps it
    u32 throughout.  Totals equal the oracle's either way."""
    n, m, Q = 100, 300_000, 1000
    inst = RoutingInstance(n, Q, True, 0.0, oracle.make_random_instance(n, 12))
    tour = rand_tour(n, 13)
    base = oracle.generate(UNIFORM, 1, 10, 33, n, m)
    for where in (None, m // 2, 3):
        dem = base.copy()
        if where is not None:
            dem[where, 7] = 300   # needs 9 bits
        got = ctx.split_eval(inst, tour, dem)
        want = oracle.split_batch(n, Q, 1, 0.0, inst.costs, tour, dem)
        np.testing.assert_array_equal(got["totals"][0], want)


@pytest.mark.parametrize("Q", [100, 1 << 30, (1 << 31) - 1])
@pytest.mark.parametrize("costs", ["int", "float"])
def test_hard_demands_near_u32_max(ctx, oracle, reference, Q, costs):
    """Demands up to 2^32-1 are legal (u32 batches, DistributionSpec lo >= 0).
    A demand d_i >= 2^32 - Q must empty the window even though the u32 load
    difference wraps (the reference's loads are int64, split.cpp:93), and
    loads that wrap u32 with d_i <= Q keep exact window differences."""
    n, m = 40, 640
    rng = np.random.default_rng(Q % 1000 + (costs == "int"))
    dem = rng.integers(0, min(Q, 12) + 1, size=(m, n)).astype(np.uint32)
    big = rng.random((m, n)) < 0.05
    dem[big] = np.uint32(0xFFFFFFF0)
    dem[::9, 5] = np.uint32(0xFFFFFFFF)
    if Q >= (1 << 30):
        dem[1::3] = rng.integers(Q // 2, Q + 1, size=(len(dem[1::3]), n)).astype(np.uint32)
    inst = (RoutingInstance(n, Q, True, 0.0, oracle.make_random_instance(n, 4)) if costs == "int"
            else float_instance(n, Q, 9))
    for tour in (np.arange(1, n + 1, dtype=np.int32), rand_tour(n, 5)):
        got = ctx.split_eval(inst, tour, dem, full=True)
        tot, V, cuts, rc, feas, (mean, fc, ic) = reference.expected_split(
            n, Q, 1, 0.0, inst.costs, tour, dem)
        np.testing.assert_array_equal(got["totals"][0], tot)
        np.testing.assert_array_equal(got["V"], V)
        np.testing.assert_array_equal(got["cuts"], cuts)
        co = ctx.split_eval(inst, tour, dem)
        np.testing.assert_array_equal(co["totals"][0], tot)
        assert co["agg"][0]["finite_count"] == fc and co["agg"][0]["infeasible_count"] == ic


@pytest.mark.parametrize("costs", ["int", "float"])
def test_hard_deque_compaction(ctx, oracle, reference, costs):
    """K1's deque ring is not circular: the front advances by evictions and
    the live entries move back to the ring's bottom when a chunk's pushes
    would run past its end.  A line metric (f increasing along the tour:
    nothing pops) with a window of ~3 positions (Q = 12, demands 3..5)
    evicts at almost every position, so the entries are compacted every few
    chunks; cost-only and full solutions, identity (12-slot ring) and random
    (16-slot ring) tours."""
    n, m, Q = 203, 4133, 12
    idx = np.arange(n + 2, dtype=np.float64)
    c = np.abs(idx[:, None] - idx[None, :])
    if costs == "float":
        c = c * 1.37 + np.triu(np.random.default_rng(4).random((n + 2, n + 2)), 1) * 0.01
        c = np.triu(c, 1)
        c = c + c.T
    inst = RoutingInstance(n, Q, True, 0.0, c)
    dem = oracle.generate(UNIFORM, 3, 5, 77, n, m)
    for tour in (np.arange(1, n + 1, dtype=np.int32), rand_tour(n, 8)):
        got = ctx.split_eval(inst, tour, dem)
        ref_tot, (ref_mean, fc, ic) = reference.split_costs(n, Q, 1, 0.0, c, tour, dem, 16)
        np.testing.assert_array_equal(got["totals"][0], ref_tot)
        a = got["agg"][0]
        assert (a["finite_count"], a["infeasible_count"]) == (fc, ic)
        check_mean(a, ref_mean)
        sub = dem[:512]
        full = ctx.split_eval(inst, tour, sub, full=True)
        tot, V, cuts, rc, feas, _ = reference.expected_split(n, Q, 1, 0.0, c, tour, sub)
        np.testing.assert_array_equal(full["totals"][0], tot)
        np.testing.assert_array_equal(full["V"], V)
        np.testing.assert_array_equal(full["cuts"], cuts)
        np.testing.assert_array_equal(full["route_count"], rc)


@pytest.mark.parametrize("costs", ["int", "float"])
def test_handoff_full_solutions(ctx, oracle, reference, costs):
    """Full solutions (V, cuts, route counts) of scenarios that all take the
    hand-off pass: line metric with zero-heavy demands keeps up to ~60
    entries in every deque (K1's ring holds 12/16); the generic kernel's
    deque carries each entry's f, load, index and route count.  Identity and
    random tours, 70,000 scenarios: beyond the 65,536-entry hand-off list,
    so the bitmap path (one item per lane) runs too."""
    n, m, Q = 60, 70_000, 100
    idx = np.arange(n + 2, dtype=np.float64)
    c = np.abs(idx[:, None] - idx[None, :])
    if costs == "float":
        c = c * 1.37
    inst = RoutingInstance(n, Q, True, 0.0, c)
    dem = oracle.generate(UNIFORM, 0, 2, 31, n, m)
    for tour in (np.arange(1, n + 1, dtype=np.int32), rand_tour(n, 5)):
        got = ctx.split_eval(inst, tour, dem, full=True)
        tot, V, cuts, rc, feas, (mean, fc, ic) = reference.expected_split(n, Q, 1, 0.0, c, tour, dem)
        np.testing.assert_array_equal(got["totals"][0], tot)
        np.testing.assert_array_equal(got["V"], V)
        np.testing.assert_array_equal(got["cuts"], cuts)
        np.testing.assert_array_equal(got["route_count"], rc)
        np.testing.assert_array_equal(got["feasible"], feas)
        check_mean(got["agg"][0], mean)


@pytest.mark.parametrize("lo,hi,Q", [(0, 1, 3), (1, 10, 100), (0, 999_999, 3_000_000),
                                     (5, (1 << 31) + 6, (1 << 31) - 1),
                                     (0, (1 << 32) - 2, (1 << 31) - 1)])
def test_fused_uniform_draws_all_spans(ctx, oracle, lo, hi, Q):
    """K1's fused generator computes mix64's low word only when the draw's
    carry term can matter (probability ~span / 2^32); identity and random
    tours over spans 2 .. 2^32-1 give the reference's demands, hence its
    totals (checked against the materialized host batch)."""
    n, m = 60, 40_000
    inst = RoutingInstance(n, Q, True, 0.0, oracle.make_random_instance(n, 2))
    dist = Distribution("uniform", lo, hi, seed=oracle.derive_stream(7, TAG_SCENARIO, hi))
    host = oracle.generate(UNIFORM, lo, hi, dist.seed, n, m)
    for tour in (np.arange(1, n + 1, dtype=np.int32), rand_tour(n, 4)):
        want = oracle.split_batch(n, Q, 1, 0.0, inst.costs, tour, host)
        got = ctx.split_eval(inst, tour, dist, count=m)
        np.testing.assert_array_equal(got["totals"][0], want)


@pytest.mark.parametrize("full", [False, True])
def test_penalized_window_bitmap_kernel(ctx, oracle, reference, full):
    """K2-bits: penalized split with the window start counted from a 128-bit
    register bitmap, taken when Q <= 127 and every demand of the wave lies in
    [1, min(31, Q)] -- decided from the distribution (generated demands) or
    from a pass over the materialized wave.  Both kernels are exact, so a
    wave with one zero demand (old kernel) and one without (bitmap kernel)
    must both match the reference; Q = 127 puts the entry bit at the top of
    the bitmap, demands up to 31 shift it by a full word less one."""
    n, m = 57, 3000
    for Q, lo, hi in ((127, 1, 31), (100, 1, 10), (40, 3, 31)):
        inst = RoutingInstance(n, Q, False, 7.0, oracle.make_random_instance(n, Q))
        tour = rand_tour(n, Q)
        dem = oracle.generate(UNIFORM, lo, hi, 17 + Q, n, m)
        variants = [dem]
        z = dem.copy()
        z[m - 1, n // 2] = 0  # the last scenario: a zero demand -> the ring kernel
        variants.append(z)
        for d in variants:
            got = ctx.split_eval(inst, tour, d, full=full)
            if full:
                tot, V, cuts, rc, feas, (mean, fc, ic) = reference.expected_split(
                    n, Q, 0, 7.0, inst.costs, tour, d)
                np.testing.assert_array_equal(got["V"], V)
                np.testing.assert_array_equal(got["cuts"], cuts)
                np.testing.assert_array_equal(got["route_count"], rc)
            else:
                tot, (mean, fc, ic) = reference.split_costs(n, Q, 0, 7.0, inst.costs, tour, d)
            np.testing.assert_array_equal(got["totals"][0], tot)
            check_mean(got["agg"][0], mean)
        # generated demands: the decision comes from the distribution
        dist = Distribution("uniform", lo, hi, seed=oracle.derive_stream(3, TAG_SCENARIO, Q))
        host = oracle.generate(UNIFORM, lo, hi, dist.seed, n, m)
        want = oracle.split_batch(n, Q, 0, 7.0, inst.costs, tour, host)
        np.testing.assert_array_equal(ctx.split_eval(inst, tour, dist, count=m)["totals"][0], want)
    # deque compaction: a line metric (f grows along the identity tour, the
    # front leaves by window exits) with a ~3-position window moves the
    # deque's head at almost every position, so its entries are moved back
    # to the ring's bottom every few chunks
    n2, Q2 = 203, 12
    idx = np.arange(n2 + 2, dtype=np.float64)
    line = RoutingInstance(n2, Q2, False, 3.0, np.abs(idx[:, None] - idx[None, :]))
    d2 = oracle.generate(UNIFORM, 3, 5, 29, n2, 2000)
    t2 = np.arange(1, n2 + 1, dtype=np.int32)
    got = ctx.split_eval(line, t2, d2, full=full)
    tot, (mean, fc, ic) = reference.split_costs(n2, Q2, 0, 3.0, line.costs, t2, d2)
    np.testing.assert_array_equal(got["totals"][0], tot)
    if full:
        _, V, cuts, rc, _, _ = reference.expected_split(n2, Q2, 0, 3.0, line.costs, t2, d2)
        np.testing.assert_array_equal(got["V"], V)
        np.testing.assert_array_equal(got["cuts"], cuts)
        np.testing.assert_array_equal(got["route_count"], rc)
