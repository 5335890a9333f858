"""Validation parity: invalid inputs are rejected before any device work with
the reference's exception class (std::invalid_argument -> InvalidArgument)
and the reference's message, checked against the real reference library
(split.cpp:128-178, oudp.cpp:136-207, 402-407)."""
import numpy as np
import pytest

from oracle import Customer as RCustomer
from paper_2602_05179_b200 import Customer, RoutingInstance
from paper_2602_05179_b200 import _capi as A

pytestmark = pytest.mark.gpu


def _ref_message(fn):
    with pytest.raises(RuntimeError) as e:
        fn()
    return str(e.value)


def _split_cases(oracle):
    n = 6
    good = oracle.make_random_instance(n, 1)
    neg = good.copy()
    neg[1, 2] = -1.0
    nan = good.copy()
    nan[3, 1] = np.nan
    inf = good.copy()
    inf[0, 4] = np.inf
    diag = good.copy()
    diag[2, 2] = 1.0
    tour = np.arange(1, n + 1, dtype=np.int32)
    dup = tour.copy()
    dup[3] = dup[2]
    dem = np.full((5, n), 3, np.uint32)
    return [
        ("capacity", (n, 0, 1, 0.0, good, tour, dem)),
        ("negative", (n, 10, 1, 0.0, neg, tour, dem)),
        ("nan", (n, 10, 1, 0.0, nan, tour, dem)),
        ("inf", (n, 10, 1, 0.0, inf, tour, dem)),
        ("diagonal", (n, 10, 1, 0.0, diag, tour, dem)),
        ("beta", (n, 10, 0, -1.0, good, tour, dem)),
        ("tour_dup", (n, 10, 1, 0.0, good, dup, dem)),
        ("tour_range", (n, 10, 1, 0.0, good, np.array([0, 2, 3, 4, 5, 6], np.int32), dem)),
    ]


@pytest.mark.parametrize("case", range(8))
def test_split_validation_messages(ctx, oracle, reference, case):
    name, (n, Q, hard, beta, costs, tour, dem) = _split_cases(oracle)[case]
    want = _ref_message(lambda: reference.split_costs(n, Q, hard, beta, costs, tour, dem))
    inst = RoutingInstance(n, Q, bool(hard), beta, costs)
    with pytest.raises(A.InvalidArgument) as e:
        ctx.split_eval(inst, tour, dem)
    assert e.value.msg == want, name


def test_split_rows_mismatch_message(ctx, oracle):
    # (the reference shim always builds n-row batches; the wording is
    # check_inputs', split.cpp:128-138)
    n = 6
    inst = RoutingInstance(n, 10, True, 0.0, oracle.make_random_instance(n, 1))
    with pytest.raises(A.InvalidArgument) as e:
        ctx.split_eval(inst, np.arange(1, n + 1, dtype=np.int32),
                       np.full((5, n - 1), 3, np.uint32), count=5)
    assert e.value.msg == "demand column has 5 entries, instance has 6 customers"


def _dsirp_cases():
    H = 3
    f = np.full((H, 2), 5.0)
    u = np.full((H, 2), 0.5)
    return [
        ("U", dict(U=70000, I0=0, H=H, fixed=f, unit=u)),
        ("I0", dict(U=10, I0=11, H=H, fixed=f, unit=u)),
        ("I0neg", dict(U=10, I0=-1, H=H, fixed=f, unit=u)),
        ("h", dict(U=10, I0=2, H=H, h=-1.0, fixed=f, unit=u)),
        ("rho", dict(U=10, I0=2, H=H, rho=1.0, fixed=f, unit=u)),
        ("fixed", dict(U=10, I0=2, H=H, fixed=-f, unit=u)),
        ("unit_nan", dict(U=10, I0=2, H=H, fixed=f, unit=u * np.nan)),
        ("htab_neg", dict(U=3, I0=2, H=H, fixed=f, unit=u, holding_table=np.array([0, 1, -2, 3.0]))),
        ("dtab0", dict(U=3, I0=2, H=H, delivery_table=np.ones((H, 4)))),
    ]


@pytest.mark.parametrize("case", range(9))
def test_dsirp_validation_messages(ctx, reference, case):
    name, kw = _dsirp_cases()[case]
    H = kw["H"]
    dd = np.full((4, H), 2, np.uint32)
    rk = dict(kw)
    rc = RCustomer(rk.pop("U"), rk.pop("I0"), rk.pop("H"), rk.pop("h", 1.0), rk.pop("rho", 2.0),
                   fixed=rk.pop("fixed", None), unit=rk.pop("unit", None),
                   delivery_table=rk.pop("delivery_table", None),
                   holding_table=rk.pop("holding_table", None))
    want = _ref_message(lambda: reference.expected_cost(rc, dd))
    with pytest.raises(A.InvalidArgument) as e:
        ctx.dsirp_eval([Customer(**kw)], dd)
    assert e.value.msg == want, name


def test_dsirp_shape_errors(ctx):
    # rows != customers x H (oudp.cpp:402-407) and a holding table that is not
    # U+1 long (the reference shim cannot express either)
    H = 3
    c = dict(U=10, I0=2, H=H, fixed=np.full((H, 1), 5.0), unit=np.full((H, 1), 0.5))
    with pytest.raises(A.InvalidArgument):
        ctx.dsirp_eval([Customer(**c)], np.full((4, H + 1), 2, np.uint32))
