"""Generate tests/golden/*.json from the REAL reference library.

Run in the dev container (needs oracle/_ref/libscendp_ref.so, built from
/root/reference/proj/src by oracle/Makefile):

    python tests/golden/make_golden.py

The fixtures are small and committed; the GPU box never reads /root/reference.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import TAG_SCENARIO, TNORMAL, UNIFORM, Customer, Reference  # noqa: E402


def main():
    R = Reference()
    # ---- split, config-1 shape (n=50, Q=100), 64 scenarios ------------------
    n, Q, m = 50, 100, 64
    costs = R.make_random_instance(n, 1)
    sseed = R.derive_stream(1, TAG_SCENARIO, 0)
    dem = R.generate(UNIFORM, 1, 10, sseed, n, 1, m)
    rng = np.random.default_rng(2026)
    cases = []
    for tour, hard, beta in ((np.arange(1, n + 1), 1, 0.0),
                             (rng.permutation(n) + 1, 1, 0.0),
                             (rng.permutation(n) + 1, 0, 10.0)):
        tour = tour.astype(np.int32)
        tot, (mean, fc, ic) = R.split_costs(n, Q, hard, beta, costs, tour, dem)
        cases.append({"tour": tour.tolist(), "hard": hard, "beta": beta,
                      "totals": tot.tolist(), "mean": mean, "finite": fc, "infeasible": ic})
    with open(os.path.join(HERE, "split_c1.json"), "w") as f:
        json.dump({"n": n, "Q": Q, "m": m, "instance_seed": 1, "scenario_seed": sseed,
                   "costs": costs.ravel().tolist(), "demand_sum": int(dem.sum()),
                   "cases": cases}, f)

    # ---- dsirp: a few customers, U=100 H=6 R=3 pins -----------
    dcases = []
    rng = np.random.default_rng(7)
    for k in range(4):
        U, H, R_ = 100, 6, 3
        fixed = np.tile(40 + 5 * np.arange(R_, dtype=float), (H, 1)) + (rng.random((H, R_)) if k % 2 else 0)
        unit = np.tile(0.5 + 0.25 * np.arange(R_, dtype=float), (H, 1))
        cust = Customer(U, U // 2, H, 1.0 + 0.1 * k, 2.0, fixed=fixed, unit=unit)
        d = rng.integers(0, 34, size=(16, H)).astype(np.uint32)
        tot, dl, q, ei, ro, ev, agg = R.expected_cost(cust, d)
        dcases.append({"U": U, "I0": U // 2, "H": H, "h": cust.h, "rho": 2.0,
                       "fixed": fixed.tolist(), "unit": unit.tolist(),
                       "demand": d.ravel().tolist(), "totals": tot.tolist(),
                       "deliver": dl.tolist(), "route_option": ro.tolist()})
    with open(os.path.join(HERE, "dsirp_small.json"), "w") as f:
        json.dump({"cases": dcases}, f)

    # ---- generator samples ------------------------------------------------
    gcases = []
    for kind, lo, hi, mean, std, seed in ((UNIFORM, 1, 10, 0.0, 1.0, 11),
                                         (UNIFORM, 0, 33, 0.0, 1.0, 12),
                                         (TNORMAL, 0, 40, 15.0, 6.0, 13)):
        data = R.generate(kind, lo, hi, seed, 9, 1, 20, mean=mean, stddev=std)
        gcases.append({"kind": kind, "lo": lo, "hi": hi, "mean": mean, "stddev": std,
                       "seed": seed, "rows": 9, "count": 20, "data": data.ravel().tolist()})
    with open(os.path.join(HERE, "generator.json"), "w") as f:
        json.dump({"cases": gcases}, f)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
