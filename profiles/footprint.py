"""Device footprint model vs measured device memory (SPEC
acceptance 12: measured peak within 2x of the model).

    python profiles/footprint.py > profiles/r02_footprint.txt   (on the GPU box)

For each call shape at 10^4 and 10^5 scenarios, on a fresh context: the
model's fixed + per-scenario x wave bytes (scendp_*_footprint), the scratch
high-water mark the library allocated, and the cudaMemGetInfo delta across
the call (includes allocation granularity and the CUDA context's own growth).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2602_05179_b200 import (Context, Customer, Distribution, make_random_instance,
                                       pinned_empty)
    rows = []
    H = 6
    custs = [Customer(U=100, I0=50, H=H, h=1.0, rho=2.0,
                      fixed=np.tile(40 + 5 * np.arange(3.0), (H, 1)),
                      unit=np.tile(0.5 + 0.25 * np.arange(3.0), (H, 1))) for _ in range(50)]
    for m in (10_000, 100_000):
        n = 200
        inst = make_random_instance(n, 1, 100, True)
        tour = np.arange(1, n + 1, dtype=np.int32)
        rng = np.random.default_rng(1)
        dem = rng.integers(1, 11, size=(m, n)).astype(np.uint32)
        dd = rng.integers(0, 34, size=(m, 50 * H)).astype(np.uint32)
        cases = [
            ("split cost-only, pageable host batch + totals", lambda c, fp: c.split_eval(
                inst, tour, dem, footprint=fp)),
            ("split full solutions, pageable host", lambda c, fp: c.split_eval(
                inst, tour, dem, full=True, footprint=fp)),
            ("split generated (fused), host totals", lambda c, fp: c.split_eval(
                inst, tour, Distribution("uniform", 1, 10, seed=5), count=m, footprint=fp)),
            ("dsirp C3-shape, 50 customers, cost-only, pageable host", lambda c, fp: c.dsirp_eval(
                custs, dd, footprint=fp)),
            ("dsirp C3-shape, 50 customers, schedules, pageable host", lambda c, fp: c.dsirp_eval(
                custs, dd, full=True, footprint=fp)),
        ]
        for name, fn in cases:
            with Context(0) as ctx:
                before = ctx.memory_info()
                fp = fn(ctx, True)
                fn(ctx, False)
                after = ctx.memory_info()
            model = fp["fixed"] + fp["per_scenario"] * min(fp["wave"], m)
            peak = after["scratch_peak"]
            delta = before["device_free"] - after["device_free"]
            rows.append((m, name, fp["fixed"], fp["per_scenario"], fp["wave"], model, peak, delta))
    print("# device footprint model vs measured (B200, fresh context per call)")
    print(f"{'m':>7}  {'fixed MB':>9} {'B/scen':>7} {'wave':>8} {'model MB':>9} "
          f"{'peak MB':>8} {'peak/model':>10} {'memgetinfo MB':>13}  call")
    for m, name, fixed, per, wave, model, peak, delta in rows:
        print(f"{m:>7}  {fixed / 2**20:9.1f} {per:7d} {wave:8d} {model / 2**20:9.1f} "
              f"{peak / 2**20:8.1f} {peak / model:10.3f} {delta / 2**20:13.1f}  {name}")


if __name__ == "__main__":
    main()
