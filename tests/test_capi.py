"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/scendp_cuda.h declares, fails loudly without a device (no CPU
fallback), and finalizes exact aggregates correctly."""
import math
import os
import re
import sys
from fractions import Fraction

import numpy as np
import pytest

from paper_2602_05179_b200 import _capi as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "scendp_cuda.h")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(scendp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = A.load()
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python mirror binds exactly these
    assert set(names) == set(A.SIGNATURES), set(names) ^ set(A.SIGNATURES)


def test_abi_version_and_tiled_bytes():
    lib = A.load()
    assert lib.scendp_abi_version() == 1
    assert lib.scendp_tiled_bytes(200, 1) == 200 * 32 * 4
    assert lib.scendp_tiled_bytes(200, 33) == 2 * 200 * 32 * 4


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device path")
def test_no_cpu_fallback_without_device():
    from paper_2602_05179_b200 import Context
    with pytest.raises(A.ScendpError) as e:
        Context(0)
    assert e.value.status == A.ERR_NO_DEVICE
    assert "no CPU fallback" in e.value.msg


# ---- exact aggregate -------------------------------------------------------
from aggref import raw_of  # noqa: E402


def finalize(raws, k=1):
    lib = A.load()
    arr = (A.AggRaw * len(raws))(*raws)
    out = (A.Agg * k)()
    A.check(lib.scendp_agg_finalize(arr, len(raws) // k, k, out))
    return out


@pytest.mark.parametrize("seed", range(6))
def test_exact_sum_is_correctly_rounded(seed):
    rng = np.random.default_rng(seed)
    scale = [1.0, 1e-12, 1e6, 1e30, 3.0, 1e-40][seed]
    vals = list(rng.random(5000) * scale)
    vals += [0.0, np.inf, 2.0 ** -180, 1e20]
    out = finalize([raw_of(vals)])[0]
    finite = [v for v in vals if math.isfinite(v)]
    want = float(sum(Fraction(v) for v in finite))
    assert out.sum == want
    assert out.finite_count == len(finite) and out.infeasible_count == 1
    assert out.mean == out.sum / len(finite)


def test_exact_sum_shard_invariant():
    rng = np.random.default_rng(9)
    vals = list(rng.random(3001) * 1234.5)
    one = finalize([raw_of(vals)])[0]
    for G in (2, 4, 8):
        cuts = [len(vals) * g // G for g in range(G + 1)]
        parts = [raw_of(vals[cuts[g]:cuts[g + 1]]) for g in range(G)]
        many = finalize(parts)[0]
        assert many.sum == one.sum and many.finite_count == one.finite_count


def test_integer_costs_match_sequential_sum():
    vals = [float(x) for x in np.random.default_rng(2).integers(1, 4000, size=100000)]
    out = finalize([raw_of(vals)])[0]
    seq = 0.0
    for v in vals:
        seq += v
    assert out.sum == seq and out.mean == seq / len(vals)


def test_best_candidate_first_minimum():
    lib = A.load()
    aggs = (A.Agg * 4)()
    for i, (mean, fc) in enumerate([(3.0, 1), (2.0, 1), (2.0, 1), (1.0, 0)]):
        aggs[i].mean = mean
        aggs[i].finite_count = fc
    assert lib.scendp_best_candidate(aggs, 4) == 1
