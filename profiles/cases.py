"""Short, fixed workloads for ncu captures (run under gpurun; never a bench).

    python profiles/cases.py <case>[,<case>...] [--reps R]

Cases (SURVEY 8d shapes; same inputs as bench.py's lines):
  c2        split hard n=200, 10^6 scenarios, tiled HBM input, cost-only (K1 int32)
  c2float   the same with non-integral costs (K1 fp64)
  c2full    C2 with full solutions (V, cuts)
  c2gen     C2 with in-kernel generation (the e2e call, batched_split_costs_generated)
  c2genr    c2gen with a random giant tour (the e2e kernel)
  c2rand    C2 with a random giant tour (the SAA case), integer costs
  c2randf   the same with non-integral costs (K1 fp64, column gather)
  c2zero    adversarial: line metric (f increasing along the identity tour:
            nothing pops), zero-heavy demands uniform:0:2, 10^5 scenarios --
            windows of ~100 positions, every deque outgrows the ring and
            takes the hand-off (generic) pass
  c2pen     C2 penalized (beta=10), 2x10^5 scenarios, identity tour
  c3        DSIRP 50 customers x 10^5 scenarios, H=6, U=100, R=3
  c3float   the non-dyadic C3 twin (K3 fp64 path)
  c3full    C3 with exact schedules (device tiled outputs)
  c4        DSIRP 200 customers x 10^6 scenarios (one GPU)
  c5        1000 tours x 10^5 scenarios, n=50, penalized beta=10
  k5        dense (min,+) sweep: 6 stages x 3 options x 101x101, 10^5 frontiers

Every case runs one warm-up launch and then R timed launches; capture with
e.g. `ncu --set full -k regex:split_linear -s 1 -c 1 python profiles/cases.py c2`.
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


HBM = 6553.6  # MEASURED_PEAKS.json hbm_gbs (GB/s)


def build(ctx, c):
    """-> (fn, algorithmic bytes per launch or None)"""
    from paper_2602_05179_b200 import (Customer, Distribution, RoutingInstance,
                                       derive_stream, make_random_instance, pinned_empty)
    from paper_2602_05179_b200 import _capi as A
    if c == "c2zero":
        n, m = 200, 100_000
        tour = np.arange(1, n + 1, dtype=np.int32)
        idx = np.arange(n + 2, dtype=np.float64)
        inst = RoutingInstance(n, 100, True, 0.0, np.abs(idx[:, None] - idx[None, :]))
        dist = Distribution("uniform", 0, 2, seed=derive_stream(1, 0x5343454E, 0))
        sc = ctx.gen_scenarios(dist, n, m)
        fn = lambda: ctx.split_eval(inst, tour, (sc, A.MEM_DEVICE_TILED), count=m, totals=False)
        return fn, None
    if c == "c2pen":
        n, m = 200, 200_000
        tour = np.arange(1, n + 1, dtype=np.int32)
        inst = make_random_instance(n, 1, 100, False, 10.0)
        dist = Distribution("uniform", 1, 10, seed=derive_stream(1, 0x5343454E, 0))
        sc = ctx.gen_scenarios(dist, n, m)
        fn = lambda: ctx.split_eval(inst, tour, (sc, A.MEM_DEVICE_TILED), count=m, totals=False)
        return fn, None
    if c.startswith("c2"):
        n, m = 200, 1_000_000
        tour = np.arange(1, n + 1, dtype=np.int32)
        if c.startswith("c2rand") or c == "c2genr":
            tour = (np.random.default_rng(7).permutation(n) + 1).astype(np.int32)
        dist = Distribution("uniform", 1, 10, seed=derive_stream(1, 0x5343454E, 0))
        nbytes = m * (4 * n + 8) + (m * 12 * (n + 1) if c == "c2full" else 0)
        if c in ("c2float", "c2randf"):
            rng = np.random.default_rng(1)
            cc = np.triu(rng.random((n + 2, n + 2)) * 20.0, 1)
            inst = RoutingInstance(n, 100, True, 0.0, cc + cc.T)
        else:
            inst = make_random_instance(n, 1, 100, True)
        tot = ctx.alloc(m * 8)
        if c in ("c2gen", "c2genr"):
            host_tot = pinned_empty(m, np.float64)
            fn = lambda: ctx.split_eval(inst, tour, dist, count=m, host_totals=host_tot)
        else:
            scen = ctx.gen_scenarios(dist, n, m)
            outs = {"totals": tot}
            full = c == "c2full"
            if full:
                outs.update(values=ctx.alloc(ctx.tiled_bytes(n + 1, m) * 2),
                            cuts=ctx.alloc(ctx.tiled_bytes(n + 1, m)),
                            route_count=ctx.alloc(m * 4), feasible=ctx.alloc(m))
            fn = lambda: ctx.split_eval(inst, tour, (scen, A.MEM_DEVICE_TILED), count=m,
                                        full=full, out_kind="device_tiled", device_out=outs,
                                        sync=False)
        return fn, nbytes
    elif c in ("c3", "c4", "c3float", "c3full"):
        nc, m, H = (200, 1_000_000, 6) if c == "c4" else (50, 100_000, 6)
        if c == "c3float":
            rng = np.random.default_rng(21)
            custs = [Customer(U=100, I0=50, H=H, h=0.5 + rng.random(), rho=1.5 + rng.random(),
                              fixed=30 + 20 * rng.random((H, 3)), unit=0.25 + rng.random((H, 3)))
                     for _ in range(nc)]
        else:
            custs = [Customer(U=100, I0=50, H=H, h=1.0, rho=2.0,
                              fixed=np.tile(40 + 5 * np.arange(3.0), (H, 1)),
                              unit=np.tile(0.5 + 0.25 * np.arange(3.0), (H, 1))) for _ in range(nc)]
        sc = ctx.gen_scenarios(Distribution("uniform", 0, 33, seed=7), nc * H, m)
        t3 = ctx.alloc(nc * m * 8)
        outs = {"totals": t3}
        if c == "c3full":  # exact schedules (deliver, quantity, end inventory, option)
            e = nc * m * H
            outs.update(evaluated=ctx.alloc(nc * m), deliver=ctx.alloc(e),
                        quantity=ctx.alloc(4 * e), end_inventory=ctx.alloc(4 * e),
                        route_option=ctx.alloc(4 * e))
        fn = lambda: ctx.dsirp_eval(custs, (sc, A.MEM_DEVICE_TILED), count=m, full=c == "c3full",
                                    out_kind="device_tiled", device_out=outs, sync=False)
        return fn, nc * m * (4 * H + 8 + (13 * H if c == "c3full" else 0))
    elif c == "c5":
        n5, m5, K5 = 50, 100_000, 1000
        inst5 = make_random_instance(n5, 5, 100, False, 10.0)
        rng = np.random.default_rng(5)
        tours5 = np.stack([rng.permutation(n5) + 1 for _ in range(K5)]).astype(np.int32)
        scen5 = ctx.gen_scenarios(Distribution("uniform", 1, 10, seed=55), n5, m5)
        fn = lambda: ctx.split_eval(inst5, tours5, (scen5, A.MEM_DEVICE_TILED), count=m5,
                                    totals=False)
        return fn, None
    elif c == "k5":
        rng = np.random.default_rng(11)
        stages = []
        for _ in range(6):
            st = np.floor(rng.random((3, 101, 101)) * 100.0)
            st[rng.random(st.shape) < 0.5] = np.inf
            stages.append(st)
        init = np.full((100_000, 101), np.inf)
        init[np.arange(100_000), rng.integers(0, 101, 100_000)] = 0.0
        fn = lambda: ctx.minplus_sweep(stages, init)
        return fn, None
    raise SystemExit(f"unknown case {c}")


def main():
    p = argparse.ArgumentParser()
    p.add_argument("case")
    p.add_argument("--reps", type=int, default=2)
    args = p.parse_args()
    from paper_2602_05179_b200 import Context

    ctx = Context(0, timing=True)
    for c in args.case.split(","):
        fn, nbytes = build(ctx, c)
        fn()
        ctx.sync()
        ctx.kernel_stats(reset=True)
        t0 = time.perf_counter()
        for _ in range(args.reps):
            fn()
        ctx.sync()
        wall_ms = (time.perf_counter() - t0) * 1e3 / args.reps
        st = ctx.kernel_stats(reset=True)
        k_ms = st["dp_ms"] / max(1, st["dp_launches"])
        frac = f" frac={nbytes / (k_ms / 1e3) / 1e9 / HBM:.3f}" if nbytes else ""
        print(f"{c}: kernel_ms={k_ms:.4f}{frac} call_ms={wall_ms:.4f} {st}", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
