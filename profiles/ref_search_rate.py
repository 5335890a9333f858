"""Reference CPU rate of improve_first_stage (saa.cpp:106-189) on the
profiles/facade_bench.cpp search workload (n = 50, beta = 10, 10^5 training
scenarios), all host threads, a bounded number of evaluations.  Test/bench
infrastructure (runs oracle/_ref)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import UNIFORM, Reference  # noqa: E402

R = Reference()
n, m, evals = 50, 100_000, int(sys.argv[1]) if len(sys.argv) > 1 else 60
costs = R.make_random_instance(n, 5)
train = R.generate(UNIFORM, 1, 10, 11, n, 1, m)
threads = os.cpu_count() or 1
t0 = time.perf_counter()
res = R.improve_first_stage(n, 100, 10.0, costs, train, evals, threads=threads)
dt = time.perf_counter() - t0
print(f"reference improve_first_stage n=50 m=1e5, {threads} threads: {evals} evaluations in "
      f"{dt * 1e3:.0f} ms ({dt * 1e3 / evals:.1f} ms/evaluation)")
