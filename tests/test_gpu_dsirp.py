"""GPU parity: DSIRP order-up-to DP (K3) against the real reference's
batched_expected_cost (oracle/_ref) and the C restatement.

Per-scenario totals and schedules (deliver, quantity, end inventory, route
option) bit-exact; means within 1e-9 relative.  Multi-customer calls are
checked against the composition oracle: batched_expected_cost per row slice
[c*H, (c+1)*H).
"""
import numpy as np
import pytest

from oracle import Customer as OCustomer
from oracle import UNIFORM
from paper_2602_05179_b200 import Customer

pytestmark = pytest.mark.gpu


def random_customer(rng, U=None, H=None, R=None, integer=False, tab_hold=None, tab_del=None):
    U = int(rng.integers(0, 120)) if U is None else U
    H = int(rng.integers(1, 11)) if H is None else H
    R = int(rng.integers(1, 5)) if R is None else R
    I0 = int(rng.integers(0, U + 1))
    if integer:
        h, rho = float(rng.integers(1, 5)), float(rng.integers(2, 4))
        fixed = rng.integers(0, 11, size=(H, R)).astype(float)
        unit = rng.integers(0, 6, size=(H, R)).astype(float)
    else:
        h, rho = rng.random() * 2, 1.0 + rng.random() * 3
        fixed, unit = rng.random((H, R)) * 50, rng.random((H, R)) * 2
    tab_hold = rng.random() < 0.3 if tab_hold is None else tab_hold
    tab_del = rng.random() < 0.2 if tab_del is None else tab_del
    htab = rng.random(U + 1) * 10 if tab_hold else None
    dtab = None
    if tab_del:
        dtab = rng.random((H, U + 1)) * 30
        dtab[:, 0] = 0.0
    kw = dict(U=U, I0=I0, H=H, h=h, rho=rho)
    if dtab is not None:
        g = Customer(**kw, delivery_table=dtab, holding_table=htab, R=R)
        o = OCustomer(U, I0, H, h, rho, delivery_table=dtab, holding_table=htab, R=R)
    else:
        g = Customer(**kw, fixed=fixed, unit=unit, holding_table=htab)
        o = OCustomer(U, I0, H, h, rho, fixed=fixed, unit=unit, holding_table=htab)
    return g, o


def compare_one(ctx, reference, g, o, dem):
    got = ctx.dsirp_eval([g], dem, full=True)
    tot, dl, q, ei, ro, ev, (mean, fc, ic) = reference.expected_cost(o, dem)
    np.testing.assert_array_equal(got["evaluated"][0], ev)
    np.testing.assert_array_equal(got["totals"][0], tot)
    np.testing.assert_array_equal(got["deliver"][0], dl)
    np.testing.assert_array_equal(got["quantity"][0], q)
    np.testing.assert_array_equal(got["end_inventory"][0], ei)
    np.testing.assert_array_equal(got["route_option"][0], ro)
    a = got["agg"][0]
    assert a["finite_count"] == fc
    if mean is not None:
        assert abs(a["mean"] - mean) <= 1e-9 * abs(mean) + 1e-300
    # cost-only call (the fast form's fp64 table path for non-dyadic models)
    co = ctx.dsirp_eval([g], dem)
    np.testing.assert_array_equal(co["totals"][0], tot)
    np.testing.assert_array_equal(co["evaluated"][0], ev)
    assert co["agg"] == got["agg"]
    return got


def test_dsirp_random_instances_match_reference(ctx, reference):
    rng = np.random.default_rng(2024)
    for trial in range(60):
        g, o = random_customer(rng, integer=(trial % 3 == 0))
        m = int(rng.integers(1, 700))
        dem = rng.integers(0, max(2, 2 * g.U // 3 + 3), size=(m, g.H)).astype(np.uint32)
        compare_one(ctx, reference, g, o, dem)


@pytest.mark.parametrize("H", [1, 4, 6, 8, 9, 16, 17, 32])
def test_dsirp_horizons(ctx, reference, H):
    rng = np.random.default_rng(H)
    g, o = random_customer(rng, U=100, H=H, R=3)
    dem = rng.integers(0, 40, size=(300, H)).astype(np.uint32)
    compare_one(ctx, reference, g, o, dem)


def test_dsirp_edge_states(ctx, reference):
    rng = np.random.default_rng(5)
    # U = 0 (no delivery possible), huge demands (all collapse to 0), zero demands
    for U, lo, hi in ((0, 0, 3), (10, 20, 40), (50, 0, 1), (1, 0, 2)):
        g, o = random_customer(rng, U=U, H=6, R=2, tab_hold=False, tab_del=False)
        dem = rng.integers(lo, hi, size=(257, 6)).astype(np.uint32)
        compare_one(ctx, reference, g, o, dem)


def test_paper_golden_a4(ctx):
    """PAPER.md App. A.4: U=2, I0=1, d=(1,1), F(q)=q, hold {0:5,1:1,2:0} -> 4."""
    H, U = 2, 2
    dtab = np.array([[0, 1, 2], [0, 1, 2]], np.float64)
    g = Customer(U=U, I0=1, H=H, delivery_table=dtab, holding_table=np.array([5.0, 1.0, 0.0]))
    got = ctx.dsirp_eval([g], np.array([[1, 1]], np.uint32), full=True)
    assert got["totals"][0, 0] == 4.0
    np.testing.assert_array_equal(got["deliver"][0, 0], [1, 1])
    np.testing.assert_array_equal(got["quantity"][0, 0], [1, 1])


def test_dsirp_multi_customer_composition(ctx, oracle, reference):
    """rows c*H+t of one scenario column == per-customer reference calls."""
    rng = np.random.default_rng(11)
    nc, H, m = 12, 6, 2000
    pairs = [random_customer(rng, U=int(rng.integers(20, 120)), H=H, R=3) for _ in range(nc)]
    dem = oracle.generate(UNIFORM, 0, 33, 99, nc * H, m)
    got = ctx.dsirp_eval([p[0] for p in pairs], dem, full=True)
    for c, (g, o) in enumerate(pairs):
        sl = np.ascontiguousarray(dem[:, c * H:(c + 1) * H])
        tot, dl, q, ei, ro, ev, (mean, fc, ic) = reference.expected_cost(o, sl)
        np.testing.assert_array_equal(got["totals"][c], tot)
        np.testing.assert_array_equal(got["deliver"][c], dl)
        np.testing.assert_array_equal(got["route_option"][c], ro)
        np.testing.assert_array_equal(got["end_inventory"][c], ei)
        assert abs(got["agg"][c]["mean"] - mean) <= 1e-9 * abs(mean)


def test_dsirp_generated_matches_materialized(ctx):
    from paper_2602_05179_b200 import Distribution
    rng = np.random.default_rng(3)
    nc, H, m = 5, 6, 5000
    custs = [random_customer(rng, U=100, H=H, R=3, tab_hold=False, tab_del=False)[0]
             for _ in range(nc)]
    dist = Distribution("uniform", 0, 33, seed=1234)
    buf = ctx.gen_scenarios(dist, nc * H, m)
    a = ctx.dsirp_eval(custs, (buf, 2), count=m)
    b = ctx.dsirp_eval(custs, dist, count=m)
    np.testing.assert_array_equal(a["totals"], b["totals"])
    assert a["agg"] == b["agg"]
    buf.free()


@pytest.mark.parametrize("H,U,full", [(33, 40, True), (48, 100, False), (60, 25, True), (120, 7, True)])
def test_long_horizons_dense_fallback(ctx, oracle, reference, H, U, full):
    """Horizons above the sparse kernels' 32 run the reference's dense forward
    pass on the GPU (dsirp_long.cu): totals and schedules bit-exact, tabular
    and linear models, two customers with different capacities."""
    from oracle import Customer as RefCustomer
    rng = np.random.default_rng(H)
    kws = [dict(U=U, I0=U // 2, H=H, h=0.7, rho=2.5,
                fixed=rng.random((H, 3)) * 40, unit=rng.random((H, 3)) * 2),
           dict(U=U + 3, I0=1, H=H, h=1.0, rho=2.0, R=1,
                delivery_table=np.c_[np.zeros(H), rng.random((H, U + 3)) * 50],
                holding_table=rng.random(U + 4) * 3)]
    m = 700
    dem = oracle.generate(UNIFORM, 0, U, 17 + H, 2 * H, m)
    got = ctx.dsirp_eval([Customer(**kw) for kw in kws], dem, full=full)
    for c, kw in enumerate(kws):
        tot, dl, q, ei, ro, ev, (mean, fc, ic) = reference.expected_cost(
            RefCustomer(**kw), dem[:, c * H:(c + 1) * H], 8)
        np.testing.assert_array_equal(got["totals"][c], tot)
        np.testing.assert_array_equal(got["evaluated"][c], ev)
        if full:
            np.testing.assert_array_equal(got["deliver"][c], dl)
            np.testing.assert_array_equal(got["quantity"][c], q)
            np.testing.assert_array_equal(got["end_inventory"][c], ei)
            np.testing.assert_array_equal(got["route_option"][c], ro)
        a = got["agg"][c]
        assert (a["finite_count"], a["infeasible_count"]) == (fc, ic)
        assert abs(a["mean"] - mean) <= 1e-9 * abs(mean)


@pytest.mark.parametrize("U,hi", [(300, 260), (100, 140), (200, 129), (20, 200)])
def test_fp64_std_hold_large_demands(ctx, reference, U, hi):
    """fp64 fast form with standard holding and demands on both sides of U
    and of 128 (d = 128 and 129 exactly): shortage hold terms (rho h)*(-x)
    for large -x, bit for bit against the reference."""
    rng = np.random.default_rng(U + hi)
    g, o = random_customer(rng, U=U, H=6, R=3, tab_hold=False, tab_del=False)
    m = 900
    dem = rng.integers(0, min(hi, 129), size=(m, 6)).astype(np.uint32)
    big = rng.random(m) < 0.3
    dem[big, rng.integers(0, 6, size=int(big.sum()))] = rng.integers(
        100, hi + 1, size=int(big.sum())).astype(np.uint32)
    dem[0, :] = 128
    dem[1, 2] = 129
    compare_one(ctx, reference, g, o, dem)


def test_fp64_std_hold_multi_customer(ctx, reference):
    """several fp64 standard-hold customers of different U (incl. 0) in one
    cost-only launch, large demands."""
    rng = np.random.default_rng(77)
    H, m = 5, 1500
    pairs = [random_customer(rng, U=int(u), H=H, R=2, tab_hold=False, tab_del=False)
             for u in (3, 250, 64, 129, 0, 180)]
    dem = rng.integers(0, 160, size=(m, len(pairs) * H)).astype(np.uint32)
    got = ctx.dsirp_eval([p[0] for p in pairs], dem)
    for c, (g, o) in enumerate(pairs):
        sl = np.ascontiguousarray(dem[:, c * H:(c + 1) * H])
        tot, dl, q, ei, ro, ev, (mean, fc, ic) = reference.expected_cost(o, sl)
        np.testing.assert_array_equal(got["totals"][c], tot)
        np.testing.assert_array_equal(got["evaluated"][c], ev)


@pytest.mark.parametrize("h", [0.0, -0.0, 5e-324, 1e40])
def test_fp64_hold_extremes(ctx, reference, h):
    """fp64 fast form hold term fma(h, j, (rho h)*(j - x)) against the
    reference's product at signed-zero, subnormal and huge holding costs
    (non-dyadic delivery costs keep the call on the fp64 path)."""
    rng = np.random.default_rng(31)
    H, U = 6, 80
    fixed, unit = rng.random((H, 3)) * 50, rng.random((H, 3)) * 2
    g = Customer(U=U, I0=40, H=H, h=h, rho=1.7, fixed=fixed, unit=unit)
    o = OCustomer(U, 40, H, h, 1.7, fixed=fixed, unit=unit)
    dem = rng.integers(0, 70, size=(700, H)).astype(np.uint32)
    compare_one(ctx, reference, g, o, dem)


def test_fp64_hold_beyond_aggregate_range(ctx, reference):
    """costs >= 2^192 (h = 1e300): per-scenario totals still bit-exact on the
    fp64 fast form; the exact aggregate reports them as range_errors, not in
    finite_count (include/scendp_cuda.h, scendp_agg_raw)."""
    rng = np.random.default_rng(32)
    H, U = 6, 80
    fixed, unit = rng.random((H, 3)) * 50, rng.random((H, 3)) * 2
    g = Customer(U=U, I0=40, H=H, h=1e300, rho=1.7, fixed=fixed, unit=unit)
    o = OCustomer(U, 40, H, 1e300, 1.7, fixed=fixed, unit=unit)
    dem = rng.integers(0, 70, size=(700, H)).astype(np.uint32)
    tot, dl, q, ei, ro, ev, (mean, fc, ic) = reference.expected_cost(o, dem)
    for full in (True, False):
        got = ctx.dsirp_eval([g], dem, full=full)
        np.testing.assert_array_equal(got["totals"][0], tot)
        np.testing.assert_array_equal(got["evaluated"][0], ev)
        a = got["agg"][0]
        big = int(np.sum(np.isfinite(tot) & (tot >= 2.0 ** 192)))
        assert big > 0
        assert a["range_errors"] == big and a["finite_count"] + big == fc
