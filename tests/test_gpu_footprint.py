"""Device footprint model and memory-driven waves (the
device analogue of split_per_scenario_bytes / adjust_batch_size,
split.cpp:287-301, oudp.cpp:383-396, engine.cpp:7-30).

* The model's bytes match what a call allocates: scratch high-water mark of
  a fresh context within [model, 2 x model] (SPEC acceptance 12) for split
  and DSIRP at 10^4 and 10^5 scenarios.
* A deliberately small budget (scratch_limit) runs the call in many waves
  with results identical to the unlimited call.
* An allocation failure halves the wave and retries: with most of the
  device taken and an oversized budget, a call whose first wave cannot be
  allocated still succeeds, in waves, bit-identical.
"""
import numpy as np
import pytest

from oracle import UNIFORM
from paper_2602_05179_b200 import Context, Customer, Distribution, RoutingInstance

pytestmark = pytest.mark.gpu


def _split_case(oracle, n, m, seed=3):
    inst = RoutingInstance(n, 100, True, 0.0, oracle.make_random_instance(n, seed))
    dem = oracle.generate(UNIFORM, 1, 10, seed, n, m)
    tour = (np.random.default_rng(seed).permutation(n) + 1).astype(np.int32)
    return inst, tour, dem


def _customers(nc, H):
    return [Customer(U=100, I0=50, H=H, h=1.0, rho=2.0,
                     fixed=np.tile(40 + 5 * np.arange(3.0), (H, 1)) + c % 5,
                     unit=np.tile(0.5 + 0.25 * np.arange(3.0), (H, 1))) for c in range(nc)]


@pytest.mark.parametrize("m", [10_000, 100_000])
@pytest.mark.parametrize("kind", ["split_cost", "split_full", "dsirp_full"])
def test_model_matches_measured_peak(oracle, m, kind):
    with Context(0) as ctx:
        if kind.startswith("split"):
            inst, tour, dem = _split_case(oracle, 200, m)
            full = kind == "split_full"
            fp = ctx.split_eval(inst, tour, dem, full=full, footprint=True)
            got = ctx.split_eval(inst, tour, dem, full=full)
            assert got["agg"][0]["finite_count"] == m
        else:
            custs = _customers(20, 6)
            dd = oracle.generate(UNIFORM, 0, 33, 9, 20 * 6, m)
            fp = ctx.dsirp_eval(custs, dd, full=True, footprint=True)
            ctx.dsirp_eval(custs, dd, full=True)
        mem = ctx.memory_info()
    model = fp["fixed"] + fp["per_scenario"] * min(fp["wave"], m)
    assert fp["wave"] >= m  # 180 GB: one wave
    assert model <= mem["scratch_peak"] <= 2 * model, (model, mem)


def test_small_budget_runs_in_waves_identically(oracle):
    n, m = 60, 20_000
    inst, tour, dem = _split_case(oracle, n, m, seed=5)
    tours = np.stack([tour, tour[::-1].copy()])
    custs = _customers(3, 6)
    dd = oracle.generate(UNIFORM, 0, 33, 4, 3 * 6, m)
    with Context(0) as a:
        ra = a.split_eval(inst, tours, dem)
        fa = a.split_eval(inst, tour, dem, full=True)
        da = a.dsirp_eval(custs, dd, full=True)
    # the fixed part under a small budget (the fallback scratch is sized to
    # 1/8 of the budget, at least 2 CTAs per SM) plus ~1/8 of the call
    with Context(0, scratch_limit=64 << 20) as p:
        fp0 = p.split_eval(inst, tour, dem, full=True, footprint=True)
    # (the allocator keeps 1/8 headroom per block, which the wave sizing
    # charges against the budget)
    budget = fp0["fixed"] * 9 // 8 + (64 << 10) + fp0["per_scenario"] * 9 // 8 * (m // 8)
    with Context(0, scratch_limit=budget) as b:
        fp = b.split_eval(inst, tour, dem, full=True, footprint=True)
        assert fp["wave"] < m and fp["budget"] == budget
        rb = b.split_eval(inst, tours, dem)
        fb = b.split_eval(inst, tour, dem, full=True)
        assert b.memory_info()["last_wave"] < m
        db = b.dsirp_eval(custs, dd, full=True)
    np.testing.assert_array_equal(ra["totals"], rb["totals"])
    assert ra["agg"] == rb["agg"]
    for key in ("totals", "V", "cuts", "route_count", "feasible"):
        np.testing.assert_array_equal(fa[key], fb[key])
    for key in ("totals", "evaluated", "deliver", "quantity", "end_inventory", "route_option"):
        np.testing.assert_array_equal(da[key], db[key])
    assert da["agg"] == db["agg"]


def test_allocation_failure_halves_the_wave(oracle):
    """Most of the device is taken by another allocation and the budget is
    set far above it, so the first wave's scratch cannot be allocated: the
    call must halve its wave until it fits and return the same results."""
    n, m = 50, 4_000_000  # full solutions: ~1.2 KB per scenario of device scratch
    dist = Distribution("uniform", 1, 10, seed=11)
    inst = RoutingInstance(n, 100, True, 0.0, oracle.make_random_instance(n, 8))
    tour = np.arange(1, n + 1, dtype=np.int32)
    with Context(0) as ref_ctx:
        want = ref_ctx.split_eval(inst, tour, dist, count=m, full=True)
        assert ref_ctx.memory_info()["oom_retries"] == 0
    with Context(0, scratch_limit=1 << 40) as ctx:
        free = ctx.memory_info()["device_free"]
        hog = ctx.alloc(free - (2 << 30))  # leave ~2 GB
        try:
            got = ctx.split_eval(inst, tour, dist, count=m, full=True)
            mem = ctx.memory_info()
        finally:
            hog.free()
    assert mem["oom_retries"] > 0 and mem["last_wave"] < m
    for key in ("totals", "V", "cuts", "route_count", "feasible"):
        np.testing.assert_array_equal(want[key], got[key])
    assert want["agg"] == got["agg"]


@pytest.mark.parametrize("src", ["host", "generated", "tiled"])
def test_repeated_calls_stay_one_wave(oracle, src):
    """Without a scratch_limit a call that fits the device runs in one wave,
    also when it fits the scratch the context already holds (regression: the
    held-scratch fast path once charged the allocator's headroom against the
    held total and cut every repeated call into dozens of waves)."""
    from paper_2602_05179_b200 import Distribution
    from paper_2602_05179_b200 import _capi as A
    n, m = 200, 100_000
    inst, tour, dem = _split_case(oracle, n, m)
    dist = Distribution("uniform", 1, 10, seed=5)
    with Context(0) as ctx:
        keep = None
        if src == "host":
            scen = dem
        elif src == "generated":
            scen = dist
        else:
            keep = ctx.gen_scenarios(dist, n, m)
            scen = (keep, A.MEM_DEVICE_TILED)
        for _ in range(3):  # the same call again: its scratch is held exactly
            ctx.split_eval(inst, tour, scen, count=m)
            assert ctx.memory_info()["last_wave"] >= m
        if keep is not None:
            keep.free()
    with Context(0) as ctx:
        dd = oracle.generate(UNIFORM, 0, 33, 9, 24, m)
        for _ in range(3):
            ctx.dsirp_eval(_customers(4, 6), dd)
            assert ctx.memory_info()["last_wave"] >= m
