"""B200-native scenario-batched second-stage DP engine (host-side mirror).

Python mirror of the reference's evaluator interface (proj/include/scendp/
split.hpp, oudp.hpp, scenario.hpp) over the C-ABI in include/scendp_cuda.h.
The C++ drop-in facade (include/scendp/*.hpp) is the primary host API; this
module exists so tests and bench.py can drive the same C-ABI from Python.

Everything runs on the GPU through libscendp_b200.so; there is no fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi as A

__all__ = [
    "RoutingInstance", "Distribution", "Customer", "Context", "DeviceBuffer",
    "make_random_instance", "poisson_hi", "tiled_to_reference", "reference_to_tiled",
]

KIND = {"uniform": A.DIST_UNIFORM, "tnormal": A.DIST_TNORMAL, "poisson": A.DIST_POISSON}
GAMMA = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1
TAG_SCENARIO = 0x5343454E
TAG_EVALUATION = 0x4556414C
TAG_INSTANCE = 0x494E5354
TAG_EXPERIMENT = 0x45585054


def mix64(z: int) -> int:
    """scenario.hpp:12-17"""
    z = (z + GAMMA) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def derive_stream(seed: int, tag: int, index: int) -> int:
    """scenario.hpp:54-57"""
    return mix64(mix64(mix64(seed) ^ tag) ^ index)


def poisson_hi(lam: float) -> int:
    return int(np.ceil(lam + 12.0 * np.sqrt(lam) + 10.0))


@dataclass
class RoutingInstance:
    """split.hpp:17-29"""
    n: int
    capacity: int
    hard: bool
    penalty_beta: float
    costs: np.ndarray  # (n+2, n+2) float64

    def as_c(self):
        self._costs = np.ascontiguousarray(self.costs, np.float64).ravel()
        return A.Routing(self.n, self.capacity, 1 if self.hard else 0, self.penalty_beta,
                         self._costs.ctypes.data)


def make_random_instance(n: int, seed: int, capacity: int, hard: bool = True,
                         penalty_beta: float = 0.0) -> RoutingInstance:
    """split.cpp:390-409 (host construction; integer costs 1..20)."""
    side = n + 2
    costs = np.zeros((side, side), np.float64)
    st = derive_stream(seed, TAG_INSTANCE, 0)
    for a in range(side):
        for b in range(a + 1, side):
            x = mix64(st)
            st = (st + GAMMA) & MASK64
            c = float(1 + ((x * 20) >> 64))
            costs[a, b] = c
            costs[b, a] = c
    return RoutingInstance(n, capacity, hard, penalty_beta, costs)


@dataclass
class Distribution:
    """DistributionSpec (scenario.hpp:60-76) + poisson."""
    kind: str
    lo: int = 0
    hi: int = 0
    mean: float = 0.0
    stddev: float = 1.0
    seed: int = 0

    @staticmethod
    def parse(text: str, seed: int) -> "Distribution":
        p = text.split(":")
        if p[0] == "uniform" and len(p) == 3:
            return Distribution("uniform", int(p[1]), int(p[2]), seed=seed)
        if p[0] == "tnormal" and len(p) == 5:
            return Distribution("tnormal", int(p[3]), int(p[4]), float(p[1]), float(p[2]), seed)
        if p[0] == "poisson" and len(p) in (2, 3):
            lam = float(p[1])
            hi = int(p[2]) if len(p) == 3 else poisson_hi(lam)
            return Distribution("poisson", 0, hi, lam, 1.0, seed)
        raise ValueError(f"distribution spec '{text}': expected uniform:lo:hi, "
                         "tnormal:mean:std:lo:hi or poisson:lambda[:hi]")

    def as_c(self) -> A.Dist:
        return A.Dist(KIND[self.kind], self.lo, self.hi, self.mean, self.stddev, self.seed)


@dataclass
class Customer:
    """CustomerSpec + DeliveryCostModel + HoldingPenaltyModel (oudp.hpp:15-65)."""
    U: int
    I0: int
    H: int
    h: float = 1.0
    rho: float = 2.0
    fixed: Optional[np.ndarray] = None  # (H, R)
    unit: Optional[np.ndarray] = None   # (H, R)
    delivery_table: Optional[np.ndarray] = None  # (H, U+1)
    holding_table: Optional[np.ndarray] = None   # (U+1,)
    R: int = 1

    def __post_init__(self):
        if self.delivery_table is not None:
            self.delivery_table = np.ascontiguousarray(self.delivery_table, np.float64).reshape(
                self.H, self.U + 1)
            self.fixed = np.zeros((self.H, self.R))
            self.unit = np.zeros((self.H, self.R))
        else:
            self.fixed = np.ascontiguousarray(self.fixed, np.float64).reshape(self.H, -1)
            self.unit = np.ascontiguousarray(self.unit, np.float64).reshape(self.H, -1)
            self.R = self.fixed.shape[1]
        if self.holding_table is not None:
            self.holding_table = np.ascontiguousarray(self.holding_table, np.float64)

    def as_c(self) -> A.Customer:
        p = lambda a: None if a is None else a.ctypes.data  # noqa: E731
        return A.Customer(self.U, self.I0, self.H, self.h, self.rho, self.R, p(self.fixed),
                          p(self.unit), int(self.delivery_table is not None),
                          p(self.delivery_table), int(self.holding_table is not None),
                          p(self.holding_table))


class DeviceBuffer:
    """Device allocation owned by a Context."""

    def __init__(self, ctx: "Context", nbytes: int):
        self.ctx = ctx
        self.nbytes = int(nbytes)
        p = C.c_void_p()
        A.check(ctx.lib.scendp_device_alloc(ctx.handle, max(1, self.nbytes), C.byref(p)))
        self.ptr = p.value

    def free(self):
        if self.ptr:
            self.ctx.lib.scendp_device_free(self.ctx.handle, self.ptr)
            self.ptr = None

    def upload(self, arr: np.ndarray):
        arr = np.ascontiguousarray(arr)
        assert arr.nbytes <= self.nbytes
        A.check(self.ctx.lib.scendp_memcpy(self.ctx.handle, self.ptr, arr.ctypes.data,
                                           arr.nbytes, 0, 0))

    def download(self, dtype, count: int) -> np.ndarray:
        out = np.empty(count, dtype)
        A.check(self.ctx.lib.scendp_memcpy(self.ctx.handle, out.ctypes.data, self.ptr,
                                           out.nbytes, 1, 0))
        return out


def reference_to_tiled(arr: np.ndarray) -> np.ndarray:
    """(count, rows) reference layout -> tiled [count/32][rows][32] (host helper)."""
    count, rows = arr.shape
    tiles = (count + 31) // 32
    pad = np.zeros((tiles * 32, rows), arr.dtype)
    pad[:count] = arr
    return np.ascontiguousarray(pad.reshape(tiles, 32, rows).transpose(0, 2, 1))


def tiled_to_reference(flat: np.ndarray, rows: int, count: int) -> np.ndarray:
    tiles = (count + 31) // 32
    t = flat[: tiles * rows * 32].reshape(tiles, rows, 32).transpose(0, 2, 1)
    return np.ascontiguousarray(t.reshape(tiles * 32, rows)[:count])


def _fp_dict(f: A.Footprint) -> dict:
    return {"fixed": f.fixed_bytes, "per_scenario": f.per_scenario_bytes, "wave": f.wave,
            "budget": f.budget}


def _agg_dict(a: A.Agg) -> dict:
    return {"sum": a.sum, "mean": a.mean if a.finite_count else None,
            "finite_count": a.finite_count, "infeasible_count": a.infeasible_count,
            "error_count": a.error_count, "range_errors": a.range_errors}


class Context:
    """One CUDA device + stream (scendp_ctx)."""

    def __init__(self, device: int = 0, timing: bool = False, max_batch: int = 0,
                 scratch_limit: int = 0):
        self.lib = A.load()
        o = A.Opts(device, scratch_limit, max_batch, A.CTX_KERNEL_TIMING if timing else 0)
        h = C.c_void_p()
        A.check(self.lib.scendp_ctx_create(C.byref(o), C.byref(h)))
        self.handle = h.value
        dev, sms, stream = C.c_int32(), C.c_int32(), C.c_void_p()
        A.check(self.lib.scendp_ctx_info(self.handle, C.byref(dev), C.byref(sms), C.byref(stream)))
        self.device, self.sm_count, self.stream = dev.value, sms.value, stream.value

    def close(self):
        if self.handle:
            self.lib.scendp_ctx_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- memory ---------------------------------------------------------------
    def alloc(self, nbytes: int) -> DeviceBuffer:
        return DeviceBuffer(self, nbytes)

    def sync(self):
        A.check(self.lib.scendp_ctx_sync(self.handle))

    def set_max_batch(self, m: int):
        A.check(self.lib.scendp_ctx_set_max_batch(self.handle, m))

    def tiled_bytes(self, rows: int, count: int) -> int:
        return self.lib.scendp_tiled_bytes(rows, count)

    # ---- K4 -------------------------------------------------------------------
    def gen_scenarios(self, dist: Distribution, rows: int, count: int, w0: int = 0,
                      tiled: bool = True, out: Optional[DeviceBuffer] = None) -> DeviceBuffer:
        nbytes = self.tiled_bytes(rows, count) if tiled else rows * count * 4
        buf = out or self.alloc(nbytes)
        d = dist.as_c()
        A.check(self.lib.scendp_gen_scenarios(self.handle, C.byref(d), rows, w0, count,
                                              A.MEM_DEVICE_TILED if tiled else A.MEM_DEVICE,
                                              buf.ptr))
        return buf

    # ---- SCNB files (io.cpp:276-344) ------------------------------------------
    @staticmethod
    def scnb_header(path: str):
        """(rows, count) of an SCNB file (reference header checks and messages)."""
        lib = A.load()
        h = A.ScnbHeader()
        A.check(lib.scendp_scnb_header_read(str(path).encode(), C.byref(h)))
        return h.rows, h.count

    @staticmethod
    def scnb_write(path: str, data: np.ndarray):
        """write_scenario_binary of a (count, rows) host array."""
        lib = A.load()
        arr = np.ascontiguousarray(data, np.uint32)
        A.check(lib.scendp_scnb_write(str(path).encode(), arr.ctypes.data, arr.shape[1],
                                      arr.shape[0]))

    def scnb_load(self, path: str, first: int = 0, count: Optional[int] = None,
                  tiled: bool = True) -> DeviceBuffer:
        """Stream scenarios [first, first+count) of an SCNB file into HBM."""
        rows, total = self.scnb_header(path)
        count = total - first if count is None else count
        buf = self.alloc(self.tiled_bytes(rows, count) if tiled else rows * count * 4)
        A.check(self.lib.scendp_scnb_load(self.handle, str(path).encode(), first, count,
                                          A.MEM_DEVICE_TILED if tiled else A.MEM_DEVICE,
                                          buf.ptr))
        return buf

    # ---- K5: dense (min,+) sweep (minplus.cpp) -------------------------------
    def minplus_sweep(self, stages, init: np.ndarray, all_stages: bool = False,
                      exact_ties: bool = False) -> np.ndarray:
        """forward_sweep of a batch of frontiers (init [B][n]) through `stages`
        ([depth][rows][cols] arrays).  Returns [B][n + sum cols] (all_stages)
        or the last frontiers [B][cols]."""
        init = np.ascontiguousarray(np.atleast_2d(init), np.float64)
        keep = [np.ascontiguousarray(a, np.float64) for a in stages]
        cs = (A.MinplusStage * max(1, len(keep)))()
        for s, a in enumerate(keep):
            cs[s] = A.MinplusStage(a.shape[1], a.shape[2], a.shape[0], a.ctypes.data)
        width = init.shape[1] + (sum(a.shape[2] for a in keep) if all_stages else 0)
        if not all_stages:
            width = keep[-1].shape[2] if keep else init.shape[1]
        out = np.empty((init.shape[0], width), np.float64)
        flags = (A.MINPLUS_ALL_STAGES if all_stages else 0) | (A.MINPLUS_EXACT_TIES if exact_ties else 0)
        A.check(self.lib.scendp_minplus_sweep(self.handle, cs, len(keep), init.ctypes.data,
                                              init.shape[1], init.shape[0], A.MEM_HOST, flags,
                                              out.ctypes.data))
        return out

    def to_tiled(self, src: DeviceBuffer, rows: int, count: int) -> DeviceBuffer:
        dst = self.alloc(self.tiled_bytes(rows, count))
        A.check(self.lib.scendp_scenarios_to_tiled(self.handle, src.ptr, rows, count, dst.ptr))
        return dst

    @staticmethod
    def _scenarios(scen, rows: int, count: Optional[int], first_index: int):
        """scen: host ndarray (count, rows) | (DeviceBuffer, kind) | Distribution."""
        keep = []
        if isinstance(scen, np.ndarray):
            arr = np.ascontiguousarray(np.atleast_2d(scen), np.uint32)
            keep.append(arr)
            # the array's own row count: the C-ABI rejects a mismatch with the
            # instance (split.cpp:128-138, oudp.cpp:402-407)
            sc = A.Scenarios(A.MEM_HOST, arr.ctypes.data, arr.shape[1], arr.shape[0],
                             first_index, None)
        elif isinstance(scen, Distribution):
            d = scen.as_c()
            keep.append(d)
            sc = A.Scenarios(A.MEM_GENERATED, None, rows, count, first_index, C.pointer(d))
        else:
            buf, kind = scen
            sc = A.Scenarios(kind, buf.ptr, rows, count, first_index, None)
        return sc, keep

    # ---- split (K1/K2/K6) -------------------------------------------------------
    def split_eval(self, inst: RoutingInstance, tours, scenarios, count: Optional[int] = None,
                   first_index: int = 0, full: bool = False, totals: bool = True,
                   quadratic: bool = False, out_kind: str = "host",
                   device_out: Optional[dict] = None, sync: bool = True,
                   host_totals: Optional[np.ndarray] = None, raw: bool = False,
                   prepare: bool = False, footprint: bool = False):
        """Evaluate tours (k x n, 1-based ids) on a scenario set.

        Returns totals [k][m] (host), V/cuts [m][n+1], route_count, feasible
        (full mode) and per-tour aggregates.  out_kind 'device_tiled' writes
        into caller DeviceBuffers (device_out) and returns only aggregates.
        prepare=True returns a callable that issues this exact call again;
        footprint=True returns the call's device footprint model instead.
        """
        tours = np.ascontiguousarray(np.atleast_2d(np.asarray(tours, np.int32)))
        k, n = tours.shape
        rinst = inst.as_c()
        sc, keep = self._scenarios(scenarios, n, count, first_index)
        m = sc.count
        flags = (A.SPLIT_FULL if full else 0) | (A.QUADRATIC if quadratic else 0)
        if not sync:
            flags |= A.ASYNC
        res = {}
        agg = (A.Agg * k)()
        if out_kind == "host":
            o = A.SplitOut(A.MEM_HOST, None, None, None, None, None, agg, None)
            if totals:
                res["totals"] = (host_totals.reshape(k, m) if host_totals is not None
                                 else np.empty((k, m), np.float64))
                o.totals = res["totals"].ctypes.data
            if full:
                res["V"] = np.empty((m, n + 1), np.float64)
                res["cuts"] = np.empty((m, n + 1), np.int32)
                res["route_count"] = np.empty(m, np.int32)
                res["feasible"] = np.empty(m, np.uint8)
                o.values = res["V"].ctypes.data
                o.cuts = res["cuts"].ctypes.data
                o.route_count = res["route_count"].ctypes.data
                o.feasible = res["feasible"].ctypes.data
        else:
            kind = A.MEM_DEVICE_TILED if out_kind == "device_tiled" else A.MEM_DEVICE
            dv = device_out or {}
            ptr = lambda key: dv[key].ptr if key in dv else None  # noqa: E731
            o = A.SplitOut(kind, ptr("totals"), ptr("values"), ptr("cuts"), ptr("route_count"),
                           ptr("feasible"), agg if sync else None, None)
        if raw:
            raws = (A.AggRaw * k)()
            o.agg_raw = raws
            res["agg_raw"] = raws
        if footprint:
            fp = A.Footprint()
            A.check(self.lib.scendp_split_footprint(self.handle, C.byref(rinst), k, C.byref(sc),
                                                    flags, C.byref(o), C.byref(fp)))
            return _fp_dict(fp)
        if prepare:
            # the same C call, argument structs built once (bench loops: the
            # Python marshalling would otherwise dominate short device calls)
            lib, h, held = self.lib, self.handle, (rinst, tours, sc, keep, o, agg, inst)
            return lambda: A.check(lib.scendp_split_eval(
                h, C.byref(held[0]), held[1].ctypes.data, k, C.byref(held[2]), flags,
                C.byref(held[4])))
        A.check(self.lib.scendp_split_eval(self.handle, C.byref(rinst), tours.ctypes.data, k,
                                           C.byref(sc), flags, C.byref(o)))
        if sync or out_kind == "host":
            res["agg"] = [_agg_dict(agg[i]) for i in range(k)]
            res["best"] = int(self.lib.scendp_best_candidate(agg, k))
        return res

    # ---- DSIRP (K3) -------------------------------------------------------------
    def dsirp_eval(self, customers: Sequence[Customer], scenarios, count: Optional[int] = None,
                   first_index: int = 0, full: bool = False, totals: bool = True,
                   out_kind: str = "host", device_out: Optional[dict] = None,
                   sync: bool = True, fp64: bool = False,
                   host_totals: Optional[np.ndarray] = None, raw: bool = False,
                   prepare: bool = False, footprint: bool = False):
        nc = len(customers)
        H = customers[0].H
        carr = (A.Customer * nc)(*[c.as_c() for c in customers])
        sc, keep = self._scenarios(scenarios, nc * H, count, first_index)
        m = sc.count
        flags = (A.DSIRP_FULL if full else 0) | (0 if sync else A.ASYNC) | (A.DSIRP_FP64 if fp64 else 0)
        agg = (A.Agg * nc)()
        res = {}
        if out_kind == "host":
            o = A.DsirpOut(A.MEM_HOST, None, None, None, None, None, None, agg, None)
            if totals:
                res["totals"] = (host_totals.reshape(nc, m) if host_totals is not None
                                 else np.empty((nc, m), np.float64))
                res["evaluated"] = np.empty((nc, m), np.uint8)
                o.totals = res["totals"].ctypes.data
                o.evaluated = res["evaluated"].ctypes.data
            if full:
                for key, dt in (("deliver", np.uint8), ("quantity", np.int32),
                                ("end_inventory", np.int32), ("route_option", np.int32)):
                    res[key] = np.empty((nc, m, H), dt)
                    setattr(o, key, res[key].ctypes.data)
        else:
            kind = A.MEM_DEVICE_TILED if out_kind == "device_tiled" else A.MEM_DEVICE
            dv = device_out or {}
            ptr = lambda key: dv[key].ptr if key in dv else None  # noqa: E731
            o = A.DsirpOut(kind, ptr("totals"), ptr("evaluated"), ptr("deliver"),
                           ptr("quantity"), ptr("end_inventory"), ptr("route_option"),
                           agg if sync else None, None)
        if raw:
            raws = (A.AggRaw * nc)()
            o.agg_raw = raws
            res["agg_raw"] = raws
        if footprint:
            fp = A.Footprint()
            A.check(self.lib.scendp_dsirp_footprint(self.handle, carr, nc, C.byref(sc), flags,
                                                    C.byref(o), C.byref(fp)))
            return _fp_dict(fp)
        if prepare:
            lib, h, held = self.lib, self.handle, (carr, sc, keep, o, agg, list(customers))
            return lambda: A.check(lib.scendp_dsirp_eval(h, held[0], nc, C.byref(held[1]), flags,
                                                         C.byref(held[3])))
        A.check(self.lib.scendp_dsirp_eval(self.handle, carr, nc, C.byref(sc), flags,
                                           C.byref(o)))
        if sync or out_kind == "host":
            res["agg"] = [_agg_dict(agg[i]) for i in range(nc)]
        return res

    # ---- timing ---------------------------------------------------------------------
    def timer_start(self):
        A.check(self.lib.scendp_timer_start(self.handle))

    def timer_stop(self) -> float:
        ms = C.c_double()
        A.check(self.lib.scendp_timer_stop(self.handle, C.byref(ms)))
        return ms.value

    def memory_info(self) -> dict:
        """Scratch held / high-water mark, cudaMemGetInfo, wave retries."""
        mi = A.MemoryInfo()
        A.check(self.lib.scendp_ctx_memory(self.handle, C.byref(mi)))
        return {k: getattr(mi, k) for k, _ in A.MemoryInfo._fields_}

    def kernel_stats(self, reset: bool = False) -> dict:
        s = A.KernelStats()
        A.check(self.lib.scendp_kernel_stats_get(self.handle, C.byref(s), 1 if reset else 0))
        return {"launches": s.launches, "dp_launches": s.dp_launches, "dp_ms": s.dp_ms,
                "gen_launches": s.gen_launches, "gen_ms": s.gen_ms,
                "h2d_bytes": s.h2d_bytes, "d2h_bytes": s.d2h_bytes}

    def flush_l2(self):
        A.check(self.lib.scendp_flush_l2(self.handle))

    # ---- NCCL -----------------------------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = A.load()
        buf = (C.c_uint8 * A.NCCL_ID_BYTES)()
        A.check(lib.scendp_nccl_unique_id(buf))
        return bytes(buf)

    def comm_init_rank(self, uid: bytes, nranks: int, rank: int):
        buf = (C.c_uint8 * A.NCCL_ID_BYTES).from_buffer_copy(uid)
        A.check(self.lib.scendp_comm_init_rank(self.handle, buf, nranks, rank))

    def comm_destroy(self):
        A.check(self.lib.scendp_comm_destroy(self.handle))


def pinned_empty(count: int, dtype) -> np.ndarray:
    """numpy view of page-locked host memory (cudaMallocHost); freed at exit."""
    lib = A.load()
    dt = np.dtype(dtype)
    p = C.c_void_p()
    A.check(lib.scendp_host_alloc_pinned(max(1, count * dt.itemsize), C.byref(p)))
    buf = (C.c_char * (count * dt.itemsize)).from_address(p.value)
    return np.frombuffer(buf, dtype=dt, count=count)


def agg_finalize(raws: List[A.AggRaw], k: int) -> List[dict]:
    lib = A.load()
    n = len(raws) // k
    arr = (A.AggRaw * len(raws))(*raws)
    out = (A.Agg * k)()
    A.check(lib.scendp_agg_finalize(arr, n, k, out))
    return [_agg_dict(out[i]) for i in range(k)]
