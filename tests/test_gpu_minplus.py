"""K5 (generic dense (min,+) sweep, minplus.cu) and the dense DSIRP path
against the real reference (minplus.cpp, oudp.cpp:226-266), plus the
reference's own randomized oracle trials run against this library."""
import numpy as np
import pytest

from oracle import Customer
from paper_2602_05179_b200 import _capi as A

from test_gpu_facade import run

pytestmark = pytest.mark.gpu
INF = np.inf


def rand_stage(rng, depth, rows, cols, p_inf=0.3, integral=False):
    a = rng.random((depth, rows, cols)) * 50.0
    if integral:
        a = np.floor(a)
    a[rng.random(a.shape) < p_inf] = INF
    return a


def rand_frontier(rng, width, p_inf=0.4):
    j = rng.random(width) * 10.0
    j[rng.random(width) < p_inf] = INF
    j[rng.integers(width)] = 0.0
    return j


@pytest.mark.parametrize("shapes", [
    [(1, 1, 1)],
    [(3, 37, 70), (1, 70, 5), (2, 5, 130)],
    [(1, 101, 101)] * 6,
    [(4, 64, 64), (1, 64, 65), (2, 65, 63)],
])
def test_forward_sweep_matches_reference(ctx, reference, shapes):
    rng = np.random.default_rng(len(shapes) * 7 + shapes[0][1])
    stages = [rand_stage(rng, *s) for s in shapes]
    init = rand_frontier(rng, shapes[0][1])
    got = ctx.minplus_sweep(stages, init, all_stages=True)[0]
    want = reference.forward_sweep(stages, init)
    np.testing.assert_array_equal(got, want)
    # batched: many frontiers through the same chain, last frontier each
    B = 257
    inits = np.stack([rand_frontier(rng, shapes[0][1]) for _ in range(B)])
    last = ctx.minplus_sweep(stages, inits)
    w = shapes[-1][2]
    for b in range(0, B, 16):
        np.testing.assert_array_equal(last[b], reference.forward_sweep(stages, inits[b])[-w:])


def test_golden_a2_and_signed_zero_ties(ctx, reference):
    """PAPER.md:517-558 golden, and -0.0 inputs (sign of zero ties kept as
    the reference's extended_min, via the exact compare-select path)."""
    a = np.array([[[2, 5], [1, INF], [3, 0]]], np.float64)
    got = ctx.minplus_sweep([a], np.array([0, 1, 3.0]))
    np.testing.assert_array_equal(got[0], [2.0, 3.0])
    z = np.array([[[-0.0, 0.0], [0.0, -0.0]]])
    for init in (np.array([-0.0, 0.0]), np.array([0.0, -0.0]), np.array([-0.0, -0.0])):
        got = ctx.minplus_sweep([z, z], init, all_stages=True)[0]
        want = reference.forward_sweep([z, z], init)
        assert got.view(np.uint64).tolist() == want.view(np.uint64).tolist()


def test_dimension_errors(ctx):
    a = np.zeros((1, 3, 2))
    with pytest.raises(A.InvalidArgument) as e:
        ctx.minplus_sweep([a], np.zeros(4))
    assert "min-plus apply: matrix has 3 rows but frontier has 4 entries" in e.value.msg


def test_dense_dsirp_sweep_matches_reference(reference):
    U, I0, H, R, seed, m = 30, 10, 5, 3, 33, 20
    got = run("dense", U, I0, H, R, seed, m)
    fixed = np.array([[40.0 + 5.0 * r + 0.125 * t for r in range(R)] for t in range(H)])
    unit = np.array([[0.5 + 0.25 * r for r in range(R)] for t in range(H)])
    cust = Customer(U, I0, H, 1.25, 2.5, fixed=fixed, unit=unit)
    dem = reference.generate(0, 0, 33, seed, 1, H, m)
    fr = got["frontiers"].reshape(m, H + 1, U + 1)
    for w in range(m):
        np.testing.assert_array_equal(fr[w], reference.sweep_customer(cust, dem[w]))
    # forward_sweep_batch from every start state == per-start sweeps (I0 = s)
    last = got["batch_last"].reshape(U + 1, U + 1)
    for s in (0, 7, U):
        c2 = Customer(U, s, H, 1.25, 2.5, fixed=fixed, unit=unit)
        np.testing.assert_array_equal(last[s], reference.sweep_customer(c2, dem[0])[-1])


@pytest.mark.parametrize("which,trials,seed", [(0, 400, 1), (0, 400, 12345), (1, 300, 7),
                                               (2, 400, 1), (2, 400, 7)])
def test_reference_oracle_trials_pass_on_this_library(reference, which, trials, seed):
    """run_split_oracle_trials / run_split_agreement_trials /
    run_dsirp_oracle_trials (oracle.cpp:61-172), same instances as the
    reference draws them, evaluated by the GPU DPs."""
    got = run("trials", which, trials, seed, 60)
    assert got["trials"] == trials
    assert got["mismatches"] == 0, got
    mism, _ = reference.oracle_trials(which, trials, seed, 60)
    assert mism == 0
