"""SCNB ingestion straight into HBM (scendp_scnb_load):
shards of a file land bit-identical in both device layouts, across chunk
boundaries and unaligned shard starts, and feed the evaluators with results
identical to the host-batch path and to the reference on the same file."""
import numpy as np
import pytest

from oracle import TAG_SCENARIO, UNIFORM
from paper_2602_05179_b200 import RoutingInstance, tiled_to_reference
from paper_2602_05179_b200 import _capi as A

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,count", [(50, 1000), (3, 5_000_003 // 7), (200, 65)])
def test_scnb_load_shards_both_layouts(ctx, tmp_path, rows, count):
    rng = np.random.default_rng(rows)
    data = rng.integers(0, 2**32, size=(count, rows), dtype=np.uint64).astype(np.uint32)
    path = tmp_path / "s.scnb"
    ctx.scnb_write(path, data)
    assert ctx.scnb_header(path) == (rows, count)
    for first, cnt in ((0, count), (1, count - 1), (count // 3, count // 2), (count - 1, 1)):
        ref = ctx.scnb_load(path, first, cnt, tiled=False)
        got = ref.download(np.uint32, rows * cnt).reshape(cnt, rows)
        np.testing.assert_array_equal(got, data[first:first + cnt])
        ref.free()
        til = ctx.scnb_load(path, first, cnt, tiled=True)
        flat = til.download(np.uint32, ctx.tiled_bytes(rows, cnt) // 4)
        np.testing.assert_array_equal(tiled_to_reference(flat, rows, cnt), data[first:first + cnt])
        til.free()
    with pytest.raises(A.InvalidArgument):
        ctx.scnb_load(path, count - 1, 2)


def test_scnb_multichunk_and_evaluation(ctx, oracle, reference, tmp_path):
    """A file larger than one 64 MB staging chunk; the split evaluated on the
    loaded tiled set equals the reference on the same file."""
    n, m = 200, 200_000   # 160 MB of payload: three chunks
    seed = oracle.derive_stream(3, TAG_SCENARIO, 0)
    dem = oracle.generate(UNIFORM, 1, 10, seed, n, m)
    path = tmp_path / "big.scnb"
    reference.write_scenario_file(path, dem)
    buf = ctx.scnb_load(path)
    inst = RoutingInstance(n, 100, True, 0.0, oracle.make_random_instance(n, 1))
    tour = np.arange(1, n + 1, dtype=np.int32)
    got = ctx.split_eval(inst, tour, (buf, A.MEM_DEVICE_TILED), count=m)
    tot, (mean, fc, ic) = reference.split_costs(n, 100, 1, 0.0, inst.costs, tour, dem)
    np.testing.assert_array_equal(got["totals"][0], tot)
    assert got["agg"][0]["mean"] == mean
    buf.free()


def test_scnb_narrow_then_wide_chunks(ctx, oracle, tmp_path):
    """Tiled loads narrow byte-sized values while reading; a wider value in a
    later chunk switches the rest of the load to u32 -- the tiled set is the
    file's either way (values 0..9, then one 70000 in the last chunk)."""
    n, m = 200, 200_000
    dem = oracle.generate(UNIFORM, 0, 9, 5, n, m)
    dem[m - 10, 17] = 70_000
    path = tmp_path / "mixed.scnb"
    ctx.scnb_write(path, dem)
    til = ctx.scnb_load(path, tiled=True)
    flat = til.download(np.uint32, ctx.tiled_bytes(n, m) // 4)
    np.testing.assert_array_equal(tiled_to_reference(flat, n, m), dem)
    til.free()
