"""The in-library NCCL path (dlopen'ed libnccl, one all-reduce of the raw
per-candidate aggregates) exercised on the single GPU this pool provides:
a one-rank communicator (multi-process form, scendp_comm_init_rank, and
in-process form, scendp_comm_init_all) must leave every result unchanged.
The N > 1 exchange itself is covered host-side by test_multiprocess.py."""
import ctypes as C

import numpy as np
import pytest

from oracle import TAG_SCENARIO, UNIFORM
from paper_2602_05179_b200 import Context, Customer, RoutingInstance
from paper_2602_05179_b200 import _capi as A

pytestmark = pytest.mark.gpu


def _workload(oracle):
    n, m = 50, 3000
    inst = RoutingInstance(n, 100, True, 0.0, oracle.make_random_instance(n, 1))
    tours = np.stack([np.arange(1, n + 1, dtype=np.int32),
                      (np.random.default_rng(2).permutation(n) + 1).astype(np.int32)])
    dem = oracle.generate(UNIFORM, 1, 10, oracle.derive_stream(1, TAG_SCENARIO, 0), n, m)
    return inst, tours, dem


def test_single_rank_communicator_keeps_results(oracle):
    inst, tours, dem = _workload(oracle)
    with Context(0) as plain:
        want = plain.split_eval(inst, tours, dem)
    with Context(0) as ctx:
        uid = Context.nccl_unique_id()
        assert len(uid) == A.NCCL_ID_BYTES
        ctx.comm_init_rank(uid, 1, 0)
        got = ctx.split_eval(inst, tours, dem)
        assert got["agg"] == want["agg"]
        np.testing.assert_array_equal(got["totals"], want["totals"])
        H = 6
        cust = [Customer(U=60, I0=30, H=H, fixed=np.full((H, 2), 20.0), unit=np.full((H, 2), 0.5))]
        dd = oracle.generate(UNIFORM, 0, 25, 3, H, 777)
        a = ctx.dsirp_eval(cust, dd)
        ctx.comm_destroy()
        b = ctx.dsirp_eval(cust, dd)
        assert a["agg"] == b["agg"]


def test_in_process_communicator(oracle):
    inst, tours, dem = _workload(oracle)
    lib = A.load()
    ctx = Context(0)
    try:
        want = ctx.split_eval(inst, tours, dem)
        arr = (C.c_void_p * 1)(ctx.handle)
        A.check(lib.scendp_comm_init_all(arr, 1))
        got = ctx.split_eval(inst, tours, dem)
        assert got["agg"] == want["agg"]
        A.check(lib.scendp_comm_destroy(ctx.handle))
    finally:
        ctx.close()


def test_overlapped_allreduce_path(oracle):
    """The multi-rank aggregate path (double-buffered aggregates, NCCL
    all-reduce on a second stream overlapping the next call's kernels),
    forced on a one-rank communicator: chains of asynchronous calls and
    interleaved synchronous ones give the plain results."""
    import subprocess
    import sys
    code = r'''
import numpy as np, sys
sys.path.insert(0, ".")
from oracle import Oracle, TAG_SCENARIO, UNIFORM
from paper_2602_05179_b200 import Context, Customer, RoutingInstance
from paper_2602_05179_b200 import _capi as A
o = Oracle()
n, m = 50, 3000
inst = RoutingInstance(n, 100, True, 0.0, o.make_random_instance(n, 1))
tours = np.stack([np.arange(1, n + 1, dtype=np.int32), (np.random.default_rng(2).permutation(n) + 1).astype(np.int32)])
dem = o.generate(UNIFORM, 1, 10, o.derive_stream(1, TAG_SCENARIO, 0), n, m)
with Context(0) as plain:
    want = plain.split_eval(inst, tours, dem)
    H = 6
    cust = [Customer(U=60, I0=30, H=H, fixed=np.full((H, 2), 20.0), unit=np.full((H, 2), 0.5))]
    dd = o.generate(UNIFORM, 0, 25, 3, H, 777)
    wantd = plain.dsirp_eval(cust, dd)
with Context(0) as ctx:
    ctx.comm_init_rank(Context.nccl_unique_id(), 1, 0)
    scen = ctx.alloc(m * n * 4); scen.upload(dem)
    tot = ctx.alloc(2 * m * 8)
    for rep in range(3):
        for _ in range(7):   # asynchronous chain: all-reduces overlap the next kernels
            ctx.split_eval(inst, tours, (scen, A.MEM_DEVICE), count=m, out_kind="device",
                           device_out={"totals": tot}, sync=False)
        got = ctx.split_eval(inst, tours, dem)
        assert got["agg"] == want["agg"], (got["agg"], want["agg"])
        assert np.array_equal(got["totals"], want["totals"])
        gd = ctx.dsirp_eval(cust, dd)
        assert gd["agg"] == wantd["agg"]
    ctx.timer_start()
    for _ in range(5):
        ctx.split_eval(inst, tours, (scen, A.MEM_DEVICE), count=m, out_kind="device",
                       device_out={"totals": tot}, sync=False)
    assert ctx.timer_stop() > 0
    ctx.comm_destroy()
print("overlap ok")
'''
    import os
    env = dict(os.environ, SCENDP_OVERLAP_ALLREDUCE="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "overlap ok" in r.stdout, r.stdout + r.stderr


def test_multi_context_entry_points(oracle):
    """scendp_split_eval_multi / scendp_dsirp_eval_multi: one host thread per
    context of a scendp_comm_init_all group (the deadlock-free way to drive
    one process's GPUs), each on its own scenario shard; here a one-device
    group with the shard = the whole set, equal to the plain call."""
    inst, tours, dem = _workload(oracle)
    lib = A.load()
    ctx = Context(0)
    try:
        want = ctx.split_eval(inst, tours, dem)
        arr = (C.c_void_p * 1)(ctx.handle)
        A.check(lib.scendp_comm_init_all(arr, 1))
        dem_c = np.ascontiguousarray(dem, np.uint32)
        sc = (A.Scenarios * 1)(A.Scenarios(A.MEM_HOST, dem_c.ctypes.data, dem.shape[1],
                                           dem.shape[0], 0, None))
        k, m = tours.shape[0], dem.shape[0]
        totals = np.empty((k, m))
        agg = (A.Agg * k)()
        out = (A.SplitOut * 1)(A.SplitOut(A.MEM_HOST, totals.ctypes.data, None, None, None, None,
                                          agg, None))
        rinst = inst.as_c()
        A.check(lib.scendp_split_eval_multi(arr, 1, C.byref(rinst), tours.ctypes.data, k, sc, 0,
                                            out))
        np.testing.assert_array_equal(totals, want["totals"])
        assert [agg[i].finite_count for i in range(k)] == [a["finite_count"] for a in want["agg"]]
        assert [agg[i].mean for i in range(k)] == [a["mean"] for a in want["agg"]]
        H = 6
        cust = Customer(U=60, I0=30, H=H, fixed=np.full((H, 2), 20.0), unit=np.full((H, 2), 0.5))
        dd = np.ascontiguousarray(oracle.generate(UNIFORM, 0, 25, 3, H, 777), np.uint32)
        plain = ctx.dsirp_eval([cust], dd)
        carr = (A.Customer * 1)(cust.as_c())
        sc2 = (A.Scenarios * 1)(A.Scenarios(A.MEM_HOST, dd.ctypes.data, H, dd.shape[0], 0, None))
        tot2 = np.empty(dd.shape[0])
        agg2 = (A.Agg * 1)()
        out2 = (A.DsirpOut * 1)(A.DsirpOut(A.MEM_HOST, tot2.ctypes.data, None, None, None, None,
                                           None, agg2, None))
        A.check(lib.scendp_dsirp_eval_multi(arr, 1, carr, 1, sc2, 0, out2))
        np.testing.assert_array_equal(tot2, plain["totals"][0])
        assert agg2[0].mean == plain["agg"][0]["mean"]
        # errors surface with the context index
        bad = (A.Scenarios * 1)(A.Scenarios(A.MEM_HOST, dem_c.ctypes.data, 7, dem.shape[0], 0,
                                            None))
        st = lib.scendp_split_eval_multi(arr, 1, C.byref(rinst), tours.ctypes.data, k, bad, 0, out)
        assert st == 1 and b"context 0" in lib.scendp_last_error()
        A.check(lib.scendp_comm_destroy(ctx.handle))
    finally:
        ctx.close()
