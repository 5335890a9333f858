"""N>1 host logic on CPU (gloo, world_size 2): contiguous scenario shards,
the single all-reduce of raw per-candidate aggregates (u64 digit words, the
same buffer the library hands to ncclAllReduce), and bench.py's rendezvous
helpers.  The per-scenario DP values come from the oracle restatement; the
digit conversion is the Python restatement of agg_pieces (csrc/common.cuh)
from test_capi.py."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, n, m, k, q):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from aggref import raw_words
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle, UNIFORM
    O = Oracle()
    costs = O.make_random_instance(n, 11)
    rng = np.random.default_rng(0)
    tours = [(rng.permutation(n) + 1).astype(np.int32) for _ in range(k)]
    lo, hi = rank * m // world, (rank + 1) * m // world  # contiguous shard
    dem = O.generate(UNIFORM, 1, 10, 1234, n, hi - lo, w0=lo)  # same streams as 1 GPU
    totals = [O.split_batch(n, 30, 0, 10.0, costs, t, dem) for t in tours]
    words = torch.from_numpy(raw_words(totals).astype(np.int64))  # u64 bit pattern
    dist.all_reduce(words)  # == ncclAllReduce(ncclUint64, sum) on the raw buffer
    # bench.py plumbing: max over ranks and the NCCL-id broadcast
    import bench
    d = bench.Dist.__new__(bench.Dist)
    d.rank, d.world, d.local_rank, d.pg = rank, world, rank, dist
    mx = d.max(float(rank + 1))
    uid = d.bcast_bytes(b"id-from-rank-0" if rank == 0 else b"")
    if rank == 0:
        q.put((words.numpy().astype(np.uint64), mx, uid))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_aggregate_allreduce_matches_single(world):
    from oracle import Oracle, UNIFORM
    from paper_2602_05179_b200 import _capi as A
    n, m, k = 30, 501, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, n, m, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    words, mx, uid = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert mx == float(world) and uid == b"id-from-rank-0"
    # single-process reference of the same job
    O = Oracle()
    costs = O.make_random_instance(n, 11)
    rng = np.random.default_rng(0)
    tours = [(rng.permutation(n) + 1).astype(np.int32) for _ in range(k)]
    dem = O.generate(UNIFORM, 1, 10, 1234, n, m)
    totals = [O.split_batch(n, 30, 0, 10.0, costs, t, dem) for t in tours]
    from aggref import raw_words, to_struct
    lib = A.load()
    out = (A.Agg * k)()
    A.check(lib.scendp_agg_finalize(to_struct(words), 1, k, out))
    single = (A.Agg * k)()
    A.check(lib.scendp_agg_finalize(to_struct(raw_words(totals)), 1, k, single))
    for c in range(k):
        mean, fc, ic = O.mean(totals[c])
        assert out[c].finite_count == fc == m
        assert out[c].sum == single[c].sum          # shard-invariant, bit for bit
        assert out[c].mean == mean                  # integer costs: == sequential mean
