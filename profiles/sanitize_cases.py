"""Small invocations of every kernel of the library, for compute-sanitizer
(memcheck / racecheck / synccheck) runs on the GPU box:

    compute-sanitizer --tool memcheck python profiles/sanitize_cases.py

Covers K1 (int/fp64, cost-only/full, tiled/generated, identity/permuted
tours, deque compaction, overflow to the generic kernel incl. its bitmap
path), K2-int, K2-bits (scanned and generated eligibility, compaction) and
the O(n) generic fallback, the quadratic kernel, K3 (int/fp64, cost-only/full, several
horizons), K4 (uniform/poisson/tnormal, both layouts), the tiled
transforms, SCNB loading, K5 and the DSIRP long-horizon kernel.
"""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2602_05179_b200 import (Context, Customer, Distribution, RoutingInstance,
                                       make_random_instance)
    from paper_2602_05179_b200 import _capi as A
    rng = np.random.default_rng(0)
    with Context(0) as ctx:
        for n in (7, 50):
            m = 700
            tours = np.stack([np.arange(1, n + 1), rng.permutation(n) + 1]).astype(np.int32)
            dem = rng.integers(1, 11, size=(m, n)).astype(np.uint32)
            dem[::17, n // 2] = 500                      # window empties (d > Q)
            dem[1::19] = 1                               # long windows / deque growth
            ii = make_random_instance(n, 1, 40, True)
            fc = rng.random((n + 2, n + 2)) * 9.0
            fc = np.triu(fc, 1) + np.triu(fc, 1).T
            fi = RoutingInstance(n, 40, True, 0.0, fc)
            for inst in (ii, fi):
                ctx.split_eval(inst, tours, dem)
                ctx.split_eval(inst, tours[1], dem, full=True)
                ctx.split_eval(inst, tours[0], dem, quadratic=True)
                ctx.split_eval(inst, tours, Distribution("uniform", 1, 10, seed=3), count=m)
            pen = make_random_instance(n, 1, 30, False, 10.0)
            ctx.split_eval(pen, tours, dem)
            ctx.split_eval(pen, tours[1], dem, full=True)
            ctx.split_eval(RoutingInstance(n, 30, False, 2.5, fc), tours, dem)
            # K2-bits (Q <= 127, demands in [1, 31]): scanned and generated
            pen2 = make_random_instance(n, 1, 100, False, 10.0)
            dem2 = rng.integers(1, 11, size=(m, n)).astype(np.uint32)
            ctx.split_eval(pen2, tours, dem2)
            ctx.split_eval(pen2, tours[1], dem2, full=True)
            ctx.split_eval(pen2, tours, Distribution("uniform", 1, 31, seed=4), count=m)
        # deque compaction (K1 and K2-bits) and mass hand-offs (list + bitmap)
        n3 = 203
        idx = np.arange(n3 + 2, dtype=np.float64)
        line = np.abs(idx[:, None] - idx[None, :])
        t3 = np.arange(1, n3 + 1, dtype=np.int32)
        d3 = rng.integers(3, 6, size=(300, n3)).astype(np.uint32)
        for hard in (True, False):
            ctx.split_eval(RoutingInstance(n3, 12, hard, 3.0, line), t3, d3)
            ctx.split_eval(RoutingInstance(n3, 12, hard, 3.0, line), t3, d3, full=True)
        dz = rng.integers(0, 3, size=(70_000, 60)).astype(np.uint32)
        idx = np.arange(62, dtype=np.float64)
        ctx.split_eval(RoutingInstance(60, 100, True, 0.0, np.abs(idx[:, None] - idx[None, :])),
                       np.arange(1, 61, dtype=np.int32), dz)
        for H in (1, 6, 11, 40):  # 40: the dense long-horizon kernel
            cs = [Customer(U=20, I0=5, H=H, fixed=np.full((H, 2), 7.0), unit=np.full((H, 2), 0.5)),
                  Customer(U=15, I0=3, H=H, fixed=np.full((H, 3), 3.1), unit=np.full((H, 3), 0.3))]
            dd = rng.integers(0, 25, size=(333, 2 * H)).astype(np.uint32)
            ctx.dsirp_eval(cs, dd)
            ctx.dsirp_eval(cs, dd, full=True)
            ctx.dsirp_eval(cs[:1] * 2, dd, fp64=True, full=True)
        for d in (Distribution("uniform", 0, 9, seed=1), Distribution("poisson", 0, 40, mean=4.0, seed=2),
                  Distribution("tnormal", 0, 20, mean=8.0, stddev=3.0, seed=3)):
            for tiled in (True, False):
                ctx.gen_scenarios(d, 13, 257, tiled=tiled).free()
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "s.scnb")
            ctx.scnb_write(path, rng.integers(0, 99, size=(300, 9)).astype(np.uint32))
            ctx.scnb_load(path, 5, 200).free()
            ctx.scnb_load(path, 0, 300, tiled=False).free()
        st = [rng.random((2, 37, 70)), rng.random((1, 70, 5))]
        ctx.minplus_sweep(st, rng.random((129, 37)), all_stages=True)
        ctx.minplus_sweep(st, -np.zeros((3, 37)))
        ctx.sync()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
