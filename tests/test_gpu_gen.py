"""GPU parity: K4 scenario generator vs the reference's generate_scenarios
(bit-exact for uniform; poisson vs the oracle restatement; tnormal counted)."""
import numpy as np
import pytest

from oracle import POISSON, TAG_SCENARIO, TNORMAL, UNIFORM, poisson_hi
from paper_2602_05179_b200 import Distribution, tiled_to_reference

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,count,lo,hi", [(200, 5000, 1, 10), (7, 1000, 0, 1 << 31),
                                             (300, 333, 0, 33), (1, 64, 5, 5)])
def test_uniform_bit_exact(ctx, oracle, reference, rows, count, lo, hi):
    seed = oracle.derive_stream(42, TAG_SCENARIO, 0)
    ref = reference.generate(UNIFORM, lo, hi, seed, rows, 1, count)
    d = Distribution("uniform", lo, hi, seed=seed)
    buf = ctx.gen_scenarios(d, rows, count, tiled=False)
    got = buf.download(np.uint32, rows * count).reshape(count, rows)
    np.testing.assert_array_equal(got, ref)
    t = ctx.gen_scenarios(d, rows, count, tiled=True)
    flat = t.download(np.uint32, ctx.tiled_bytes(rows, count) // 4)
    np.testing.assert_array_equal(tiled_to_reference(flat, rows, count), ref)
    buf.free()
    t.free()


def test_prefix_stable_and_offset(ctx, oracle):
    seed = 9
    d = Distribution("uniform", 1, 10, seed=seed)
    full = ctx.gen_scenarios(d, 50, 1000, tiled=False).download(np.uint32, 50 * 1000)
    part = ctx.gen_scenarios(d, 50, 300, w0=500, tiled=False).download(np.uint32, 50 * 300)
    np.testing.assert_array_equal(full.reshape(1000, 50)[500:800], part.reshape(300, 50))


def test_poisson_matches_oracle(ctx, oracle):
    lam = 5.0
    hi = poisson_hi(lam)
    seed = oracle.derive_stream(1, TAG_SCENARIO, 0)
    want = oracle.generate(POISSON, 0, hi, seed, 50, 4000, mean=lam)
    d = Distribution("poisson", 0, hi, mean=lam, seed=seed)
    got = ctx.gen_scenarios(d, 50, 4000, tiled=False).download(np.uint32, 50 * 4000)
    np.testing.assert_array_equal(got.reshape(4000, 50), want)
    assert abs(want.mean() - lam) < 0.05


def test_tnormal_close_to_reference(ctx, reference):
    # CUDA libm vs glibc may differ by an ulp before llround; count mismatches
    seed = 17
    ref = reference.generate(TNORMAL, 0, 40, seed, 20, 1, 5000, mean=15.0, stddev=6.0)
    d = Distribution("tnormal", 0, 40, 15.0, 6.0, seed)
    got = ctx.gen_scenarios(d, 20, 5000, tiled=False).download(np.uint32, 20 * 5000)
    mism = int((got.reshape(5000, 20) != ref).sum())
    assert mism == 0, f"{mism} tnormal draws differ"


def test_invalid_distribution_rejected(ctx):
    from paper_2602_05179_b200._capi import InvalidArgument
    with pytest.raises(InvalidArgument):
        ctx.gen_scenarios(Distribution("uniform", 5, 1, seed=0), 3, 10)
    with pytest.raises(InvalidArgument):
        ctx.gen_scenarios(Distribution("tnormal", 0, 5, 1.0, 0.0, 0), 3, 10)
