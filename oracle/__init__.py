"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this package.  The product path (``paper_2602_05179_b200``) never
does: it fails loudly when its CUDA library is missing.

* ``Oracle``    -- oracle/_build/liboracle.so, the plain-C restatement
                   (oracle/scendp_oracle.c), always buildable with gcc.
* ``Reference`` -- oracle/_ref/libscendp_ref.so, the real reference compiled
                   from /root/reference/proj/src by oracle/Makefile.  Built in
                   the dev container; the prebuilt .so travels to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libscendp_ref.so")

TAG_SCENARIO = 0x5343454E
TAG_EVALUATION = 0x4556414C
TAG_INSTANCE = 0x494E5354
TAG_EXPERIMENT = 0x45585054

UNIFORM, TNORMAL, POISSON = 0, 1, 2

_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    """Compile the C restatement and, when /root/reference exists, the
    reference library (oracle/Makefile)."""
    targets = ["all"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


class OrDist(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lo", C.c_int64), ("hi", C.c_int64),
                ("mean", C.c_double), ("stddev", C.c_double),
                ("seed", C.c_uint64)]


class OrCustomer(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("initial_inventory", C.c_int32),
                ("horizon", C.c_int32), ("holding", C.c_double),
                ("stockout_multiplier", C.c_double), ("options", C.c_int32),
                ("fixed", C.c_void_p), ("unit", C.c_void_p),
                ("delivery_tabular", C.c_int32),
                ("delivery_table", C.c_void_p),
                ("holding_tabular", C.c_int32),
                ("holding_table", C.c_void_p)]


class RefCustomer(C.Structure):
    """CustomerArgs of ref_shim.cpp."""
    _fields_ = [("U", C.c_int), ("I0", C.c_int), ("H", C.c_int),
                ("h", C.c_double), ("rho", C.c_double), ("R", C.c_int),
                ("fixed", C.c_void_p), ("unit", C.c_void_p),
                ("delivery_tabular", C.c_int), ("delivery_table", C.c_void_p),
                ("holding_tabular", C.c_int), ("holding_table", C.c_void_p)]


def poisson_hi(lam: float) -> int:
    """Default truncation point of poisson:lambda."""
    return int(np.ceil(lam + 12.0 * np.sqrt(lam) + 10.0))


class Customer:
    """Plain container mirroring CustomerSpec + DeliveryCostModel +
    HoldingPenaltyModel (oudp.hpp:15-65)."""

    def __init__(self, U, I0, H, h=1.0, rho=2.0, fixed=None, unit=None,
                 delivery_table=None, holding_table=None, R=None):
        self.U, self.I0, self.H, self.h, self.rho = int(U), int(I0), int(H), float(h), float(rho)
        if delivery_table is not None:
            self.delivery_table = np.ascontiguousarray(delivery_table, np.float64).reshape(H, U + 1)
            self.R = int(R or 1)
            self.fixed = np.zeros((H, self.R))
            self.unit = np.zeros((H, self.R))
        else:
            self.delivery_table = None
            self.fixed = np.ascontiguousarray(fixed, np.float64).reshape(H, -1)
            self.unit = np.ascontiguousarray(unit, np.float64).reshape(H, -1)
            self.R = self.fixed.shape[1]
        self.holding_table = (None if holding_table is None else
                              np.ascontiguousarray(holding_table, np.float64))

    def _ptr(self, a):
        return None if a is None else a.ctypes.data

    def as_oracle(self):
        return OrCustomer(self.U, self.I0, self.H, self.h, self.rho, self.R,
                          self._ptr(self.fixed), self._ptr(self.unit),
                          int(self.delivery_table is not None),
                          self._ptr(self.delivery_table),
                          int(self.holding_table is not None),
                          self._ptr(self.holding_table))

    def as_ref(self):
        return RefCustomer(self.U, self.I0, self.H, self.h, self.rho, self.R,
                           self._ptr(self.fixed), self._ptr(self.unit),
                           int(self.delivery_table is not None),
                           self._ptr(self.delivery_table),
                           int(self.holding_table is not None),
                           self._ptr(self.holding_table))


class Oracle:
    """The plain-C restatement (oracle/scendp_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.or_mix64.restype = C.c_uint64
        L.or_mix64.argtypes = [C.c_uint64]
        L.or_derive_stream.restype = C.c_uint64
        L.or_derive_stream.argtypes = [C.c_uint64] * 3
        L.or_poisson_table.restype = C.c_int64
        L.or_poisson_table.argtypes = [C.c_double, C.c_int64, _f64p]
        L.or_generate_scenarios.argtypes = [C.POINTER(OrDist), C.c_void_p,
                                            C.c_uint64, C.c_uint64, C.c_uint64, _u32p]
        L.or_make_random_instance.argtypes = [C.c_int32, C.c_uint64, _f64p]
        L.or_split_linear.restype = C.c_double
        L.or_split_linear.argtypes = [C.c_int32, C.c_int64, _f64p, _i32p, _u32p,
                                      C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_split_quadratic.restype = C.c_double
        L.or_split_quadratic.argtypes = [C.c_int32, C.c_int64, C.c_int32, C.c_double,
                                         _f64p, _i32p, _u32p, C.c_void_p, C.c_void_p]
        L.or_brute_force_split.restype = C.c_double
        L.or_brute_force_split.argtypes = [C.c_int32, C.c_int64, C.c_int32, C.c_double,
                                           _f64p, _i32p, _u32p]
        L.or_split_batch.argtypes = [C.c_int32, C.c_int64, C.c_int32, C.c_double,
                                     _f64p, _i32p, _u32p, C.c_uint64, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_dsirp_scenario.restype = C.c_int32
        L.or_dsirp_scenario.argtypes = [C.POINTER(OrCustomer), _u32p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_dsirp_simulate.restype = C.c_double
        L.or_dsirp_simulate.argtypes = [C.POINTER(OrCustomer), _u32p, _u8p, _i32p]
        L.or_dsirp_brute_force.restype = C.c_double
        L.or_dsirp_brute_force.argtypes = [C.POINTER(OrCustomer), _u32p]
        L.or_mean.argtypes = [_f64p, C.c_void_p, C.c_uint64, C.POINTER(C.c_double),
                              C.POINTER(C.c_int32), C.POINTER(C.c_uint64),
                              C.POINTER(C.c_uint64)]

    # ---- streams / generator -------------------------------------------
    def mix64(self, z):
        return self.lib.or_mix64(z)

    def derive_stream(self, seed, tag, index):
        return self.lib.or_derive_stream(seed, tag, index)

    def poisson_table(self, lam, hi=None):
        hi = poisson_hi(lam) if hi is None else int(hi)
        out = np.zeros(hi + 1, np.float64)
        self.lib.or_poisson_table(lam, hi, out)
        return out

    def generate(self, kind, lo, hi, seed, rows, count, w0=0, mean=0.0, stddev=1.0):
        """Reference layout (count x rows), columns [w0, w0+count)."""
        cdf = None
        if kind == POISSON:
            cdf = self.poisson_table(mean, hi)
        d = OrDist(kind, lo, hi, mean, stddev, seed)
        out = np.zeros(rows * count, np.uint32)
        self.lib.or_generate_scenarios(C.byref(d), None if cdf is None else cdf.ctypes.data,
                                       rows, w0, count, out)
        return out.reshape(count, rows)

    def make_random_instance(self, n, seed):
        c = np.zeros((n + 2) * (n + 2), np.float64)
        self.lib.or_make_random_instance(n, seed, c)
        return c.reshape(n + 2, n + 2)

    # ---- split -----------------------------------------------------------
    def split_linear(self, n, Q, costs, tour, demand):
        V = np.zeros(n + 1, np.float64)
        cuts = np.zeros(n + 1, np.int32)
        dq = C.c_int32()
        t = self.lib.or_split_linear(n, Q, np.ascontiguousarray(costs, np.float64).ravel(),
                                     np.ascontiguousarray(tour, np.int32),
                                     np.ascontiguousarray(demand, np.uint32),
                                     V.ctypes.data, cuts.ctypes.data, C.addressof(dq))
        return t, V, cuts, dq.value

    def split_quadratic(self, n, Q, hard, beta, costs, tour, demand):
        V = np.zeros(n + 1, np.float64)
        cuts = np.zeros(n + 1, np.int32)
        t = self.lib.or_split_quadratic(n, Q, int(hard), beta,
                                        np.ascontiguousarray(costs, np.float64).ravel(),
                                        np.ascontiguousarray(tour, np.int32),
                                        np.ascontiguousarray(demand, np.uint32),
                                        V.ctypes.data, cuts.ctypes.data)
        return t, V, cuts

    def brute_force_split(self, n, Q, hard, beta, costs, tour, demand):
        return self.lib.or_brute_force_split(n, Q, int(hard), beta,
                                             np.ascontiguousarray(costs, np.float64).ravel(),
                                             np.ascontiguousarray(tour, np.int32),
                                             np.ascontiguousarray(demand, np.uint32))

    def split_batch(self, n, Q, hard, beta, costs, tour, demand, full=False):
        """demand: (m, n) reference layout.  Returns totals[, V, cuts, rc]."""
        demand = np.ascontiguousarray(demand, np.uint32)
        m = demand.shape[0]
        totals = np.zeros(m, np.float64)
        V = np.zeros((m, n + 1), np.float64) if full else None
        cuts = np.zeros((m, n + 1), np.int32) if full else None
        rc = np.zeros(m, np.int32)
        self.lib.or_split_batch(n, Q, int(hard), beta,
                                np.ascontiguousarray(costs, np.float64).ravel(),
                                np.ascontiguousarray(tour, np.int32), demand.ravel(), m,
                                totals.ctypes.data,
                                None if V is None else V.ctypes.data,
                                None if cuts is None else cuts.ctypes.data,
                                rc.ctypes.data)
        if full:
            return totals, V, cuts, rc
        return totals

    # ---- dsirp -------------------------------------------------------------
    def dsirp_scenario(self, cust: Customer, demands):
        H = cust.H
        total = C.c_double()
        dl = np.zeros(H, np.uint8)
        q = np.zeros(H, np.int32)
        ei = np.zeros(H, np.int32)
        ro = np.zeros(H, np.int32)
        oc = cust.as_oracle()
        rc = self.lib.or_dsirp_scenario(C.byref(oc), np.ascontiguousarray(demands, np.uint32),
                                        C.addressof(total), dl.ctypes.data, q.ctypes.data,
                                        ei.ctypes.data, ro.ctypes.data)
        if rc != 0:
            return None
        return total.value, dl, q, ei, ro

    def dsirp_simulate(self, cust, demands, deliver, route_option):
        oc = cust.as_oracle()
        return self.lib.or_dsirp_simulate(C.byref(oc), np.ascontiguousarray(demands, np.uint32),
                                          np.ascontiguousarray(deliver, np.uint8),
                                          np.ascontiguousarray(route_option, np.int32))

    def dsirp_brute_force(self, cust, demands):
        oc = cust.as_oracle()
        return self.lib.or_dsirp_brute_force(C.byref(oc), np.ascontiguousarray(demands, np.uint32))

    def mean(self, totals, evaluated=None):
        totals = np.ascontiguousarray(totals, np.float64)
        mean, has, fc, ic = C.c_double(), C.c_int32(), C.c_uint64(), C.c_uint64()
        ev = None if evaluated is None else np.ascontiguousarray(evaluated, np.uint8)
        self.lib.or_mean(totals, None if ev is None else ev.ctypes.data, totals.size,
                         C.byref(mean), C.byref(has), C.byref(fc), C.byref(ic))
        return (mean.value if has.value else None), fc.value, ic.value


class Reference:
    """The real reference library (oracle/_ref/libscendp_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_make_random_instance.argtypes = [C.c_int, C.c_ulonglong, _f64p]
        L.ref_generate_scenarios.argtypes = [C.c_int, C.c_longlong, C.c_longlong, C.c_double,
                                             C.c_double, C.c_ulonglong, C.c_size_t,
                                             C.c_size_t, C.c_size_t, _u32p]
        L.ref_derive_stream.restype = C.c_ulonglong
        L.ref_derive_stream.argtypes = [C.c_ulonglong] * 3
        agg = [C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_ulonglong),
               C.POINTER(C.c_ulonglong)]
        L.ref_split_costs.argtypes = [C.c_int, C.c_longlong, C.c_int, C.c_double, _f64p, _i32p,
                                      _u32p, C.c_size_t, C.c_uint, C.c_void_p] + agg
        L.ref_split_costs_generated.argtypes = [C.c_int, C.c_longlong, C.c_int, C.c_double,
                                                _f64p, _i32p, C.c_int, C.c_longlong,
                                                C.c_longlong, C.c_double, C.c_double,
                                                C.c_ulonglong, C.c_size_t, C.c_uint,
                                                C.c_void_p] + agg
        L.ref_expected_split.argtypes = [C.c_int, C.c_longlong, C.c_int, C.c_double, _f64p,
                                         _i32p, _u32p, C.c_size_t, C.c_uint, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p] + agg
        L.ref_split_scenario.argtypes = [C.c_int, C.c_int, C.c_longlong, C.c_int, C.c_double,
                                         _f64p, _i32p, _u32p, _f64p, _i32p, C.POINTER(C.c_int)]
        L.ref_brute_force_split.restype = C.c_double
        L.ref_brute_force_split.argtypes = [C.c_int, C.c_longlong, C.c_int, C.c_double,
                                            _f64p, _i32p, _u32p]
        L.ref_expected_cost.argtypes = [C.POINTER(RefCustomer), _u32p, C.c_size_t, C.c_uint,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p] + agg
        L.ref_sweep_customer.argtypes = [C.POINTER(RefCustomer), _u32p, _f64p]
        L.ref_solve_customer.argtypes = [C.POINTER(RefCustomer), _u32p, C.POINTER(C.c_double),
                                         _u8p, _i32p, _i32p, _i32p]
        L.ref_minplus_apply.argtypes = [C.c_size_t, C.c_size_t, _f64p, _f64p, _f64p]
        L.ref_oracle_trials.restype = C.c_ulonglong
        L.ref_oracle_trials.argtypes = [C.c_int, C.c_size_t, C.c_ulonglong, C.c_int]
        L.ref_improve_first_stage.argtypes = [C.c_int, C.c_longlong, C.c_double, _f64p, _u32p,
                                              C.c_size_t, C.c_uint, C.c_ulonglong, _i32p,
                                              C.POINTER(C.c_double), C.POINTER(C.c_ulonglong),
                                              C.POINTER(C.c_ulonglong), _f64p, C.c_size_t]

        L.ref_write_scenario_file.argtypes = [C.c_char_p, _u32p, C.c_size_t, C.c_size_t]
        L.ref_read_scenario_file.argtypes = [C.c_char_p, C.POINTER(C.c_size_t),
                                             C.POINTER(C.c_size_t), C.c_void_p, C.c_size_t]
        L.ref_parse_instance_file.argtypes = [C.c_char_p, C.c_char_p]
        L.ref_write_routing_instance.argtypes = [C.c_int, C.c_longlong, C.c_int, C.c_double,
                                                 _f64p, C.c_char_p]
        L.ref_experiment.argtypes = [C.c_int, C.c_int, C.c_longlong, C.c_double, _f64p,
                                     C.c_int, C.c_longlong, C.c_longlong, C.c_double,
                                     C.c_double, C.POINTER(C.c_size_t), C.c_size_t, C.c_int,
                                     C.c_size_t, C.c_size_t, C.c_ulonglong, C.c_ulonglong,
                                     C.c_uint, C.c_char_p]

        L.ref_forward_sweep.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]

    def forward_sweep(self, stages, init):
        """stages: list of [depth][rows][cols] arrays; returns every frontier."""
        init = np.ascontiguousarray(init, np.float64)
        rows = np.array([a.shape[1] for a in stages], np.uint64)
        cols = np.array([a.shape[2] for a in stages], np.uint64)
        depth = np.array([a.shape[0] for a in stages], np.uint64)
        ent = np.concatenate([np.ascontiguousarray(a, np.float64).ravel() for a in stages]) \
            if stages else np.zeros(1)
        out = np.zeros(init.size + int(cols.sum()), np.float64)
        self._check(self.lib.ref_forward_sweep(len(stages), rows.ctypes.data, cols.ctypes.data,
                                               depth.ctypes.data, ent.ctypes.data,
                                               init.ctypes.data, init.size, out.ctypes.data))
        return out

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    # ---- io.hpp --------------------------------------------------------------
    def write_scenario_file(self, path, data):
        data = np.ascontiguousarray(data, np.uint32)
        self._check(self.lib.ref_write_scenario_file(str(path).encode(), data.ravel(),
                                                     data.shape[1], data.shape[0]))

    def read_scenario_file(self, path):
        """(rows, count, data[count][rows]) or raises RuntimeError(message)."""
        rows, count = C.c_size_t(), C.c_size_t()
        self._check(self.lib.ref_read_scenario_file(str(path).encode(), C.byref(rows),
                                                    C.byref(count), None, 0))
        out = np.zeros(rows.value * count.value, np.uint32)
        self._check(self.lib.ref_read_scenario_file(str(path).encode(), C.byref(rows),
                                                    C.byref(count), out.ctypes.data, out.size))
        return rows.value, count.value, out.reshape(count.value, rows.value)

    def parse_instance_file(self, path, out_path):
        self.lib.ref_parse_instance_file(str(path).encode(), str(out_path).encode())
        return open(out_path).read()

    def write_routing_instance(self, n, Q, hard, beta, costs, out_path):
        self.lib.ref_write_routing_instance(n, Q, hard, beta,
                                            np.ascontiguousarray(costs, np.float64).ravel(),
                                            str(out_path).encode())
        return open(out_path).read()

    def experiment(self, which, n, Q, beta, costs, dist, m_list, reps, eval_size, ref_size,
                   seed, evals, out_path, threads=1):
        kind, lo, hi, mean, sd = dist
        ms = (C.c_size_t * len(m_list))(*m_list)
        self._check(self.lib.ref_experiment(
            which, n, Q, beta, np.ascontiguousarray(costs, np.float64).ravel(), kind, lo, hi,
            mean, sd, ms, len(m_list), reps, eval_size, ref_size, seed, evals, threads,
            str(out_path).encode()))
        return open(out_path).read()

    @staticmethod
    def _agg():
        return C.c_double(), C.c_int(), C.c_ulonglong(), C.c_ulonglong()

    @staticmethod
    def _aggout(a):
        return (a[0].value if a[1].value else None), a[2].value, a[3].value

    def make_random_instance(self, n, seed):
        c = np.zeros((n + 2) * (n + 2), np.float64)
        self.lib.ref_make_random_instance(n, seed, c)
        return c.reshape(n + 2, n + 2)

    def derive_stream(self, seed, tag, index):
        return self.lib.ref_derive_stream(seed, tag, index)

    def generate(self, kind, lo, hi, seed, entities, steps, count, mean=0.0, stddev=1.0):
        out = np.zeros(entities * steps * count, np.uint32)
        self.lib.ref_generate_scenarios(kind, lo, hi, mean, stddev, seed, entities, steps,
                                        count, out)
        return out.reshape(count, entities * steps)

    def split_costs(self, n, Q, hard, beta, costs, tour, demand, threads=1):
        demand = np.ascontiguousarray(demand, np.uint32)
        m = demand.shape[0]
        totals = np.zeros(m, np.float64)
        a = self._agg()
        self._check(self.lib.ref_split_costs(n, Q, int(hard), beta,
                                             np.ascontiguousarray(costs, np.float64).ravel(),
                                             np.ascontiguousarray(tour, np.int32),
                                             demand.ravel(), m, threads, totals.ctypes.data,
                                             *[C.byref(x) for x in a]))
        return totals, self._aggout(a)

    def split_costs_generated(self, n, Q, hard, beta, costs, tour, kind, lo, hi, seed, m,
                              threads=1, mean=0.0, stddev=1.0, want_totals=True):
        totals = np.zeros(m, np.float64) if want_totals else None
        a = self._agg()
        self._check(self.lib.ref_split_costs_generated(
            n, Q, int(hard), beta, np.ascontiguousarray(costs, np.float64).ravel(),
            np.ascontiguousarray(tour, np.int32), kind, lo, hi, mean, stddev, seed, m,
            threads, None if totals is None else totals.ctypes.data,
            *[C.byref(x) for x in a]))
        return totals, self._aggout(a)

    def expected_split(self, n, Q, hard, beta, costs, tour, demand, threads=1):
        demand = np.ascontiguousarray(demand, np.uint32)
        m = demand.shape[0]
        totals = np.zeros(m, np.float64)
        V = np.zeros((m, n + 1), np.float64)
        cuts = np.zeros((m, n + 1), np.int32)
        rc = np.zeros(m, np.int32)
        feas = np.zeros(m, np.uint8)
        a = self._agg()
        self._check(self.lib.ref_expected_split(
            n, Q, int(hard), beta, np.ascontiguousarray(costs, np.float64).ravel(),
            np.ascontiguousarray(tour, np.int32), demand.ravel(), m, threads,
            totals.ctypes.data, V.ctypes.data, cuts.ctypes.data, rc.ctypes.data,
            feas.ctypes.data, *[C.byref(x) for x in a]))
        return totals, V, cuts, rc, feas, self._aggout(a)

    def split_scenario(self, linear, n, Q, hard, beta, costs, tour, demand):
        V = np.zeros(n + 1, np.float64)
        cuts = np.zeros(n + 1, np.int32)
        rc = C.c_int()
        self._check(self.lib.ref_split_scenario(int(linear), n, Q, int(hard), beta,
                                                np.ascontiguousarray(costs, np.float64).ravel(),
                                                np.ascontiguousarray(tour, np.int32),
                                                np.ascontiguousarray(demand, np.uint32),
                                                V, cuts, C.byref(rc)))
        return V, cuts, rc.value

    def expected_cost(self, cust: Customer, demand, threads=1):
        demand = np.ascontiguousarray(demand, np.uint32)
        m = demand.shape[0]
        H = cust.H
        totals = np.zeros(m, np.float64)
        dl = np.zeros((m, H), np.uint8)
        q = np.zeros((m, H), np.int32)
        ei = np.zeros((m, H), np.int32)
        ro = np.zeros((m, H), np.int32)
        ev = np.zeros(m, np.uint8)
        a = self._agg()
        rcst = cust.as_ref()
        self._check(self.lib.ref_expected_cost(C.byref(rcst), demand.ravel(), m, threads,
                                               totals.ctypes.data, dl.ctypes.data,
                                               q.ctypes.data, ei.ctypes.data, ro.ctypes.data,
                                               ev.ctypes.data, *[C.byref(x) for x in a]))
        return totals, dl, q, ei, ro, ev, self._aggout(a)

    def sweep_customer(self, cust: Customer, demand):
        out = np.zeros((cust.H + 1) * (cust.U + 1), np.float64)
        rcst = cust.as_ref()
        self._check(self.lib.ref_sweep_customer(C.byref(rcst),
                                                np.ascontiguousarray(demand, np.uint32), out))
        return out.reshape(cust.H + 1, cust.U + 1)

    def solve_customer(self, cust: Customer, demand):
        H = cust.H
        total = C.c_double()
        dl = np.zeros(H, np.uint8)
        q = np.zeros(H, np.int32)
        ei = np.zeros(H, np.int32)
        ro = np.zeros(H, np.int32)
        rcst = cust.as_ref()
        self._check(self.lib.ref_solve_customer(C.byref(rcst),
                                                np.ascontiguousarray(demand, np.uint32),
                                                C.byref(total), dl, q, ei, ro))
        return total.value, dl, q, ei, ro

    def minplus_apply(self, a, j):
        a = np.ascontiguousarray(a, np.float64)
        out = np.zeros(a.shape[1], np.float64)
        self._check(self.lib.ref_minplus_apply(a.shape[0], a.shape[1], a.ravel(),
                                               np.ascontiguousarray(j, np.float64), out))
        return out

    def oracle_trials(self, which, trials, seed, max_n=120):
        mism = self.lib.ref_oracle_trials(which, trials, seed, max_n)
        return mism, self.lib.ref_last_error().decode()

    def improve_first_stage(self, n, Q, beta, costs, train, max_evals, threads=1):
        train = np.ascontiguousarray(train, np.uint32)
        tour = np.zeros(n, np.int32)
        value, ev, bf = C.c_double(), C.c_ulonglong(), C.c_ulonglong()
        cap = int(max_evals) + 16
        traj = np.zeros(cap, np.float64)
        self._check(self.lib.ref_improve_first_stage(
            n, Q, beta, np.ascontiguousarray(costs, np.float64).ravel(), train.ravel(),
            train.shape[0], threads, max_evals, tour, C.byref(value), C.byref(ev),
            C.byref(bf), traj, cap))
        return tour, value.value, ev.value, bf.value, traj[:ev.value]
