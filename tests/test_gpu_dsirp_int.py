"""GPU parity of the exact scaled-integer DSIRP kernel (dsirp_int_kernel):
dyadic cost models (the BASELINE pins are multiples of 1/4) must give the
reference's results bit for bit, identical to the forced fp64 kernel, and
demands beyond the exact range must take the per-unit fp64 fallback."""
import numpy as np
import pytest

from oracle import Customer as OCustomer
from paper_2602_05179_b200 import Customer

pytestmark = pytest.mark.gpu


def dyadic_customer(rng, U, H, R, shift, tab_hold=False, tab_del=False):
    s = float(2 ** shift)
    I0 = int(rng.integers(0, U + 1))
    h = rng.integers(0, 8) / s
    rho = 1.0 + rng.integers(1, 12) / s
    fixed = rng.integers(0, 400, size=(H, R)) / s
    unit = rng.integers(0, 12, size=(H, R)) / s
    kw = dict(U=U, I0=I0, H=H, h=h, rho=rho)
    htab = rng.integers(0, 60, size=U + 1) / s if tab_hold else None
    if tab_del:
        dtab = rng.integers(0, 200, size=(H, U + 1)) / s
        dtab[:, 0] = 0.0
        return (Customer(**kw, delivery_table=dtab, holding_table=htab, R=R),
                OCustomer(U, I0, H, h, rho, delivery_table=dtab, holding_table=htab, R=R))
    return (Customer(**kw, fixed=fixed, unit=unit, holding_table=htab),
            OCustomer(U, I0, H, h, rho, fixed=fixed, unit=unit, holding_table=htab))


def check(ctx, reference, custs, dem, H):
    got = ctx.dsirp_eval([c[0] for c in custs], dem, full=True)
    f64 = ctx.dsirp_eval([c[0] for c in custs], dem, full=True, fp64=True)
    for k in ("totals", "deliver", "quantity", "end_inventory", "route_option"):
        np.testing.assert_array_equal(got[k], f64[k])
    # cost-only: exact-integer and fp64-table fast forms
    for fp64 in (False, True):
        co = ctx.dsirp_eval([c[0] for c in custs], dem, fp64=fp64)
        np.testing.assert_array_equal(co["totals"], got["totals"])
        assert co["agg"] == got["agg"]
    for ci, (g, o) in enumerate(custs):
        sl = np.ascontiguousarray(dem[:, ci * H:(ci + 1) * H])
        tot, dl, q, ei, ro, ev, (mean, fc, ic) = reference.expected_cost(o, sl)
        np.testing.assert_array_equal(got["totals"][ci], tot)
        np.testing.assert_array_equal(got["deliver"][ci], dl)
        np.testing.assert_array_equal(got["quantity"][ci], q)
        np.testing.assert_array_equal(got["end_inventory"][ci], ei)
        np.testing.assert_array_equal(got["route_option"][ci], ro)
        assert got["agg"][ci]["mean"] == mean or abs(got["agg"][ci]["mean"] - mean) <= 1e-9 * mean


@pytest.mark.parametrize("H", [1, 3, 6, 8, 12, 20])
def test_dyadic_customers_int_path(ctx, reference, H):
    rng = np.random.default_rng(100 + H)
    custs = [dyadic_customer(rng, int(rng.integers(0, 120)), H, int(rng.integers(1, 5)),
                             int(rng.integers(0, 4)), tab_hold=(i % 3 == 1), tab_del=(i % 4 == 2))
             for i in range(8)]
    dem = rng.integers(0, 45, size=(1500, 8 * H)).astype(np.uint32)
    check(ctx, reference, custs, dem, H)


def test_baseline_pins_and_fallback(ctx, reference):
    """SURVEY 8d pins (U=100, I0=50, h=1, rho=2, fixed=40+5r, unit=0.5+0.25r)
    with demands far beyond the exact range in a few units."""
    H, R = 6, 3
    fixed = np.tile(40 + 5 * np.arange(R, dtype=float), (H, 1))
    unit = np.tile(0.5 + 0.25 * np.arange(R, dtype=float), (H, 1))
    custs = [(Customer(U=100, I0=50, H=H, h=1.0, rho=2.0, fixed=fixed, unit=unit),
              OCustomer(100, 50, H, 1.0, 2.0, fixed=fixed, unit=unit)) for _ in range(3)]
    rng = np.random.default_rng(4)
    dem = rng.integers(0, 34, size=(2048, 3 * H)).astype(np.uint32)
    dem[5, 2] = 50_000_000       # beyond dlim: fp64 fallback for that unit
    dem[77, 9] = 2_000_000_000
    check(ctx, reference, custs, dem, H)


def test_ties_between_options(ctx, reference):
    """Equal route options (duplicate columns) and equal-cost states."""
    H, R = 5, 4
    fixed = np.full((H, R), 10.0)
    unit = np.full((H, R), 0.5)
    fixed[:, 3] = 9.5
    custs = [(Customer(U=20, I0=10, H=H, h=0.25, rho=3.0, fixed=fixed, unit=unit),
              OCustomer(20, 10, H, 0.25, 3.0, fixed=fixed, unit=unit))]
    dem = np.random.default_rng(1).integers(0, 12, size=(999, H)).astype(np.uint32)
    check(ctx, reference, custs, dem, H)


def test_customer_table_cache_and_dedupe(ctx, reference):
    """Identical customers share one table set, and a call with the same
    customer set as the previous call reuses the device tables; alternating
    sets, the FP64 flag and in-place edits of the caller's arrays must all
    invalidate correctly."""
    from oracle import UNIFORM
    from oracle import Customer as RCustomer
    from paper_2602_05179_b200 import Customer
    H = 5
    fa = np.tile(30.0 + 4.0 * np.arange(2.0), (H, 1))
    ua = np.tile(0.5 + 0.25 * np.arange(2.0), (H, 1))
    fb = fa + 1.5
    set_a = [Customer(U=40, I0=20, H=H, fixed=fa, unit=ua) for _ in range(3)]
    set_b = [Customer(U=40, I0=20, H=H, fixed=fa, unit=ua),
             Customer(U=40, I0=20, H=H, fixed=fb, unit=ua),
             Customer(U=40, I0=20, H=H, fixed=fa, unit=ua)]
    dd = reference.generate(UNIFORM, 0, 25, 9, 3, H, 500)

    def want(custs):
        out = []
        for c, cu in enumerate(custs):
            rc = RCustomer(40, 20, H, 1.0, 2.0, fixed=cu.fixed, unit=cu.unit)
            out.append(reference.expected_cost(rc, dd[:, c * H:(c + 1) * H])[0])
        return np.stack(out)

    wa, wb = want(set_a), want(set_b)
    for custs, w in ((set_a, wa), (set_a, wa), (set_b, wb), (set_a, wa), (set_b, wb)):
        np.testing.assert_array_equal(ctx.dsirp_eval(custs, dd)["totals"], w)
        np.testing.assert_array_equal(ctx.dsirp_eval(custs, dd, fp64=True)["totals"], w)
    # editing the caller's array in place between calls is seen
    fixed = fa.copy()
    c1 = [Customer(U=40, I0=20, H=H, fixed=fixed, unit=ua) for _ in range(3)]
    np.testing.assert_array_equal(ctx.dsirp_eval(c1, dd)["totals"], wa)
    fixed += 1.5
    np.testing.assert_array_equal(ctx.dsirp_eval(c1, dd)["totals"], want(c1))
