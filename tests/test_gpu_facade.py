"""The C++ drop-in facade (include/scendp/*.hpp) used by a C++ program
(tests/cpp/facade_main.cpp, built by csrc/Makefile) must reproduce the real
reference library (oracle/_ref) on identical inputs -- including the
reference's sequential-order means and the SAA search trajectory."""
import os
import subprocess

import numpy as np
import pytest

from oracle import POISSON, TNORMAL, UNIFORM, Customer

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "facade_main")
GAMMA, MASK = 0x9E3779B97F4A7C15, (1 << 64) - 1


def run(*args):
    if not os.path.exists(BIN):
        pytest.fail("tests/cpp/_build/facade_main not built (make -C paper_2602_05179_b200/csrc)")
    out = subprocess.run([BIN, *map(str, args)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    res = {}
    for line in out.stdout.splitlines():
        t = line.split()
        if t[0] == "failure":
            res["failure"] = line
        elif t[0] in ("totals", "V4", "gen_totals", "trajectory", "frontiers", "batch_last"):
            res[t[0]] = np.array([float(x) for x in t[2:]])
        elif t[0] in ("cuts4", "route_count", "tour", "deliver", "quantity", "end_inventory",
                      "route_option", "data", "col3", "timings_sharded", "timings_one",
                      "timings_full"):
            res[t[0]] = np.array([int(x) for x in t[2:]])
        elif t[0] == "route":
            res.setdefault("routes", []).append((int(t[1]), int(t[2])))
        else:
            for k in range(0, len(t) - 1, 2):
                res[t[k]] = float(t[k + 1])
    return res


def mix64(z):
    z = (z + GAMMA) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def fisher_yates(n, seed):
    order = list(range(1, n + 1))
    st = seed
    for i in range(n - 1, 0, -1):
        x = mix64(st)
        st = (st + GAMMA) & MASK
        j = (x * (i + 1)) >> 64
        order[i], order[j] = order[j], order[i]
    return np.array(order, np.int32)


@pytest.mark.parametrize("n,Q,hard,beta,m,tseed", [(50, 100, 1, 0.0, 1024, 0),
                                                   (60, 40, 1, 0.0, 777, 99),
                                                   (40, 30, 0, 10.0, 600, 5)])
def test_facade_split_matches_reference(reference, n, Q, hard, beta, m, tseed):
    got = run("split", n, Q, hard, beta, 3, 4, m, tseed)
    costs = reference.make_random_instance(n, 3)
    dem = reference.generate(UNIFORM, 1, 10, 4, n, 1, m)
    assert got["demand_sum"] == dem.sum()
    tour = fisher_yates(n, tseed) if tseed else np.arange(1, n + 1, dtype=np.int32)
    tot, (mean, fc, ic) = reference.split_costs(n, Q, hard, beta, costs, tour, dem, threads=4)
    np.testing.assert_array_equal(got["totals"], tot)
    np.testing.assert_array_equal(got["gen_totals"], tot)
    assert got["mean"] == mean            # BatchResultSet: reference-order mean
    assert got["finite"] == fc and got["infeasible"] == ic
    t2, V, cuts, rc, feas, (mean2, _, _) = reference.expected_split(n, Q, hard, beta, costs, tour, dem)
    np.testing.assert_array_equal(got["V4"], V[:4].ravel())
    np.testing.assert_array_equal(got["cuts4"], cuts[:4].ravel())
    np.testing.assert_array_equal(got["route_count"], rc)
    assert got["full_mean"] == mean2
    assert got["sharded_equal"] == 1  # devices {0, 0}, batch_size 300: same bits
    # one BatchTiming per batch: the reference's batches of 300 on one device
    # (engine.hpp:150-192), and per device shard in the sharded call
    ref_batches = [min(300, m - lo) for lo in range(0, m, 300)]
    assert list(got["timings_one"]) == ref_batches and got["timings_one_ok"] == 1
    assert list(got["timings_full"]) == ref_batches and got["timings_full_ok"] == 1
    half = [m // 2, m - m // 2]
    assert list(got["timings_sharded"]) == [min(300, h - lo) for h in half for lo in range(0, h, 300)]
    assert got["timings_sharded_ok"] == 1


def test_facade_dsirp_matches_reference(reference):
    U, I0, H, R, seed, m = 100, 50, 6, 3, 21, 900
    got = run("dsirp", U, I0, H, R, seed, m)
    fixed = np.array([[40.0 + 5.0 * r + 0.125 * t for r in range(R)] for t in range(H)])
    unit = np.array([[0.5 + 0.25 * r for r in range(R)] for t in range(H)])
    cust = Customer(U, I0, H, 1.25, 2.5, fixed=fixed, unit=unit)
    dem = reference.generate(UNIFORM, 0, 33, seed, 1, H, m)
    tot, dl, q, ei, ro, ev, (mean, fc, ic) = reference.expected_cost(cust, dem)
    np.testing.assert_array_equal(got["totals"], tot)
    np.testing.assert_array_equal(got["deliver"], dl.ravel())
    np.testing.assert_array_equal(got["quantity"], q.ravel())
    np.testing.assert_array_equal(got["end_inventory"], ei.ravel())
    np.testing.assert_array_equal(got["route_option"], ro.ravel())
    assert got["mean"] == mean and got["errors"] == 0
    assert got["one"] == tot[0] and got["replay"] == tot[0]


@pytest.mark.parametrize("kbatch", [1, 7, 256])
def test_facade_improve_first_stage_trajectory(reference, kbatch):
    """Batched candidate scoring keeps the reference's exact trajectory."""
    n, Q, beta, m, evals = 14, 30, 10.0, 300, 400
    got = run("saa", n, Q, beta, 8, 9, m, evals, kbatch)
    costs = reference.make_random_instance(n, 8)
    train = reference.generate(UNIFORM, 1, 10, 9, n, 1, m)
    tour, value, ev, bf, traj = reference.improve_first_stage(n, Q, beta, costs, train, evals)
    np.testing.assert_array_equal(got["tour"], tour)
    assert got["value"] == value and got["evaluations"] == ev and got["best_found_at"] == bf
    np.testing.assert_array_equal(got["trajectory"], traj)


def test_facade_generator(reference, oracle):
    got = run("gen", 0, 1, 10, 0, 1, 77, 5, 3, 40)
    ref = reference.generate(UNIFORM, 1, 10, 77, 5, 3, 40)
    np.testing.assert_array_equal(got["data"], ref.ravel())
    np.testing.assert_array_equal(got["col3"], ref[3])
    got = run("gen", 1, 0, 40, 15.0, 6.0, 78, 4, 2, 30)
    np.testing.assert_array_equal(got["data"], reference.generate(TNORMAL, 0, 40, 78, 4, 2, 30,
                                                                  mean=15.0, stddev=6.0).ravel())
    got = run("gen", 2, 0, 47, 5.0, 1, 79, 6, 1, 30)
    np.testing.assert_array_equal(got["data"], oracle.generate(POISSON, 0, 47, 79, 6, 30,
                                                               mean=5.0).ravel())


# ---- SAA experiment suite (saa.cpp:191-443) ---------------------------------
EXP_N, EXP_Q, EXP_BETA, EXP_SEED = 12, 30, 5.0, 1


def _exp(reference, tmp_path, which, m_list, reps, eval_size, ref_size, evals, seed=7,
         dist=(UNIFORM, 1, 10, 0.0, 1.0)):
    costs = reference.make_random_instance(EXP_N, EXP_SEED)
    want = reference.experiment(which, EXP_N, EXP_Q, EXP_BETA, costs, dist, m_list, reps,
                                eval_size, ref_size, seed, evals, tmp_path / "ref.csv")
    kind, lo, hi, mean, sd = dist
    run("exp", which, EXP_N, EXP_Q, EXP_BETA, EXP_SEED, kind, lo, hi, mean, sd, seed, evals,
        reps, eval_size, ref_size, tmp_path / "ours.csv", *m_list)
    return (tmp_path / "ours.csv").read_text(), want


@pytest.mark.parametrize("which,m_list,reps,eval_size,ref_size", [
    (0, [20, 300], 2, 700, 1500),      # bias, with the reference-value row
    (1, [10, 100, 1000], 3, 0, 0),     # convergence (two decades) + log-log slope
    (2, [50, 400], 2, 900, 0),         # quality vs scenarios
])
def test_saa_experiment_reports_match_reference(reference, tmp_path, which, m_list, reps,
                                                eval_size, ref_size):
    """Report CSVs (write_report_csv) of the GPU experiment suite equal the
    reference's byte for byte: same training/evaluation streams, searches,
    out-of-sample means and statistics."""
    got, want = _exp(reference, tmp_path, which, m_list, reps, eval_size, ref_size, evals=40)
    assert got == want


def test_saa_experiment_poisson_free_tnormal(reference, tmp_path):
    """tnormal training sets are generated on the GPU (CUDA libm); the
    quality report must still match when no draw straddles a rounding edge."""
    got, want = _exp(reference, tmp_path, 2, [60], 2, 300, 0, evals=25,
                     dist=(TNORMAL, 0, 12, 5.0, 2.0))
    assert got == want


def test_time_budget_and_scaling_reports(reference, tmp_path):
    """Wall-clock experiments: same row schema and labels as the reference's
    (the values are timings of different hardware)."""
    def rows(text):
        return [ln.split(",") for ln in text.splitlines() if ln and not ln.startswith("#")][1:]
    for which, ms, size in ((3, [100, 1000, 10000], 20000), (4, [], 300)):
        got, want = _exp(reference, tmp_path, which, ms or [1], 1, size, 0, evals=0)
        g, w = rows(got), rows(want)
        assert len(g) == len(w)
        for a, b in zip(g, w):
            assert a[0] == b[0] and a[2] == b[2] and a[3] == b[3]
            assert a[4].split("_", 1)[1] == b[4].split("_", 1)[1]   # gpu1_* vs single_*
            assert float(a[5]) >= 0.0
