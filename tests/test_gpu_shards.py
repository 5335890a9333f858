"""Virtual shards on one GPU: evaluating contiguous scenario
ranges separately and combining their raw aggregates with the library's
own reduction (scendp_agg_finalize -- the buffer the NCCL all-reduce sums)
must reproduce the single-call aggregate exactly, for any shard count, and
the per-scenario totals must be the corresponding slices."""
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import TAG_SCENARIO, UNIFORM
from paper_2602_05179_b200 import Customer, Distribution, RoutingInstance, agg_finalize
from paper_2602_05179_b200 import _capi as A

pytestmark = pytest.mark.gpu


def _bounds(m, g, align=1):
    cuts = [((m * j) // g) // align * align for j in range(g)] + [m]
    return list(zip(cuts[:-1], cuts[1:]))


@pytest.mark.parametrize("shards", [1, 2, 4, 8])
def test_split_shards_generated_and_host(ctx, oracle, shards):
    n, m = 120, 20_000
    inst = RoutingInstance(n, 100, True, 0.0, oracle.make_random_instance(n, 1))
    tours = np.stack([np.arange(1, n + 1, dtype=np.int32),
                      (np.random.default_rng(5).permutation(n) + 1).astype(np.int32)])
    dist = Distribution("uniform", 1, 10, seed=oracle.derive_stream(2, TAG_SCENARIO, 0))
    whole = ctx.split_eval(inst, tours, dist, count=m)
    dem = oracle.generate(UNIFORM, 1, 10, oracle.derive_stream(2, TAG_SCENARIO, 0), n, m)
    for src in ("generated", "host"):
        raws, parts = [], []
        for lo, hi in _bounds(m, shards):
            if src == "generated":
                r = ctx.split_eval(inst, tours, dist, count=hi - lo, first_index=lo, raw=True)
            else:
                r = ctx.split_eval(inst, tours, dem[lo:hi], raw=True)
            raws.append(r["agg_raw"])
            parts.append(r["totals"])
        flat = [x for per in raws for x in per]  # [shard][k]
        assert agg_finalize(flat, 2) == whole["agg"]
        np.testing.assert_array_equal(np.concatenate(parts, axis=1), whole["totals"])


@pytest.mark.parametrize("shards", [2, 8])
def test_split_tiled_device_shards(ctx, oracle, shards):
    n, m = 64, 16_384
    inst = RoutingInstance(n, 80, True, 0.0, oracle.make_random_instance(n, 3))
    tour = np.arange(1, n + 1, dtype=np.int32)
    dist = Distribution("uniform", 1, 12, seed=17)
    scen = ctx.gen_scenarios(dist, n, m)
    whole = ctx.split_eval(inst, tour, (scen, A.MEM_DEVICE_TILED), count=m)
    raws = []
    for lo, hi in _bounds(m, shards, align=32):
        # a tile-aligned shard is a byte range of the tiled buffer
        view = SimpleNamespace(ptr=scen.ptr + ctx.tiled_bytes(n, lo))
        r = ctx.split_eval(inst, tour, (view, A.MEM_DEVICE_TILED), count=hi - lo,
                           first_index=lo, raw=True)
        raws.extend(r["agg_raw"])
    assert agg_finalize(raws, 1) == whole["agg"]
    scen.free()


def test_dsirp_shards(ctx, oracle):
    H, m = 6, 9_001
    custs = [Customer(U=80, I0=40, H=H, fixed=np.tile(30 + 5 * np.arange(3.0), (H, 1)),
                      unit=np.tile(0.5 + 0.25 * np.arange(3.0), (H, 1))) for _ in range(3)]
    dd = oracle.generate(UNIFORM, 0, 30, 4, 3 * H, m)
    whole = ctx.dsirp_eval(custs, dd)
    for shards in (2, 5):
        raws, parts = [], []
        for lo, hi in _bounds(m, shards):
            r = ctx.dsirp_eval(custs, dd[lo:hi], raw=True)
            raws.extend(r["agg_raw"])
            parts.append(r["totals"])
        assert agg_finalize(raws, 3) == whole["agg"]
        np.testing.assert_array_equal(np.concatenate(parts, axis=1), whole["totals"])
