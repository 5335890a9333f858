"""ctypes declarations of the C-ABI (include/scendp_cuda.h).

The shared library is built in-tree (``paper_2602_05179_b200/libscendp_b200.so``,
see csrc/Makefile).  Loading fails loudly when it is missing: there is no
Python or CPU fallback for any evaluator.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libscendp_b200.so")
# A/B measurements of another in-tree build (profiles/ scripts only)
LIB_PATH = os.environ.get("SCENDP_LIB", LIB_PATH)

OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_CUDA = 2
ERR_NCCL = 3
ERR_OUT_OF_MEMORY = 4
ERR_NO_DEVICE = 5
ERR_LOGIC = 6
ERR_RUNTIME = 7
ERR_UNSUPPORTED = 8

DIST_UNIFORM, DIST_TNORMAL, DIST_POISSON = 0, 1, 2
MEM_HOST, MEM_DEVICE, MEM_DEVICE_TILED, MEM_GENERATED = 0, 1, 2, 3
CTX_KERNEL_TIMING = 0x1
SPLIT_COST_ONLY, SPLIT_FULL = 0, 1
DSIRP_COST_ONLY, DSIRP_FULL = 0, 1
DSIRP_FP64 = 0x400
ASYNC = 0x100
QUADRATIC = 0x200
AGG_DIGITS = 12
NCCL_ID_BYTES = 128


class Opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("scratch_limit", C.c_uint64),
                ("max_batch", C.c_uint64), ("flags", C.c_uint32)]


class Dist(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lo", C.c_int64), ("hi", C.c_int64),
                ("mean", C.c_double), ("stddev", C.c_double), ("seed", C.c_uint64)]


class Scenarios(C.Structure):
    _fields_ = [("mem_kind", C.c_uint32), ("data", C.c_void_p), ("rows", C.c_uint64),
                ("count", C.c_uint64), ("first_index", C.c_uint64),
                ("dist", C.POINTER(Dist))]


class AggRaw(C.Structure):
    _fields_ = [("digits", C.c_uint64 * AGG_DIGITS), ("finite_count", C.c_uint64),
                ("infeasible_count", C.c_uint64), ("error_count", C.c_uint64),
                ("range_errors", C.c_uint64)]


class Agg(C.Structure):
    _fields_ = [("sum", C.c_double), ("mean", C.c_double), ("finite_count", C.c_uint64),
                ("infeasible_count", C.c_uint64), ("error_count", C.c_uint64),
                ("range_errors", C.c_uint64)]


class Routing(C.Structure):
    _fields_ = [("n", C.c_int32), ("capacity", C.c_int64), ("hard", C.c_int32),
                ("penalty_beta", C.c_double), ("costs", C.c_void_p)]


class SplitOut(C.Structure):
    _fields_ = [("mem_kind", C.c_uint32), ("totals", C.c_void_p), ("values", C.c_void_p),
                ("cuts", C.c_void_p), ("route_count", C.c_void_p), ("feasible", C.c_void_p),
                ("agg", C.POINTER(Agg)), ("agg_raw", C.POINTER(AggRaw))]


class Customer(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("initial_inventory", C.c_int32),
                ("horizon", C.c_int32), ("holding", C.c_double),
                ("stockout_multiplier", C.c_double), ("options", C.c_int32),
                ("fixed", C.c_void_p), ("unit", C.c_void_p),
                ("delivery_tabular", C.c_int32), ("delivery_table", C.c_void_p),
                ("holding_tabular", C.c_int32), ("holding_table", C.c_void_p)]


class DsirpOut(C.Structure):
    _fields_ = [("mem_kind", C.c_uint32), ("totals", C.c_void_p), ("evaluated", C.c_void_p),
                ("deliver", C.c_void_p), ("quantity", C.c_void_p),
                ("end_inventory", C.c_void_p), ("route_option", C.c_void_p),
                ("agg", C.POINTER(Agg)), ("agg_raw", C.POINTER(AggRaw))]


class KernelStats(C.Structure):
    _fields_ = [("launches", C.c_uint64), ("dp_launches", C.c_uint64), ("dp_ms", C.c_double),
                ("gen_launches", C.c_uint64), ("gen_ms", C.c_double),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64)]


class MinplusStage(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("depth", C.c_uint64),
                ("entries", C.c_void_p)]


MINPLUS_ALL_STAGES = 0x1
MINPLUS_EXACT_TIES = 0x2


class ScnbHeader(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("count", C.c_uint64)]


class Footprint(C.Structure):
    _fields_ = [("fixed_bytes", C.c_uint64), ("per_scenario_bytes", C.c_uint64),
                ("wave", C.c_uint64), ("budget", C.c_uint64)]


class MemoryInfo(C.Structure):
    _fields_ = [("scratch_bytes", C.c_uint64), ("scratch_peak", C.c_uint64),
                ("device_free", C.c_uint64), ("device_total", C.c_uint64),
                ("oom_retries", C.c_uint64), ("last_wave", C.c_uint64),
                ("tnormal_host_columns", C.c_uint64)]


# Every symbol include/scendp_cuda.h declares, with its ctypes signature.
SIGNATURES = {
    "scendp_ctx_create": (C.c_int, [C.POINTER(Opts), C.POINTER(C.c_void_p)]),
    "scendp_ctx_destroy": (None, [C.c_void_p]),
    "scendp_last_error": (C.c_char_p, []),
    "scendp_abi_version": (C.c_int32, []),
    "scendp_ctx_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_void_p)]),
    "scendp_ctx_sync": (C.c_int, [C.c_void_p]),
    "scendp_ctx_set_max_batch": (C.c_int, [C.c_void_p, C.c_uint64]),
    "scendp_device_alloc": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p)]),
    "scendp_device_free": (C.c_int, [C.c_void_p, C.c_void_p]),
    "scendp_host_alloc_pinned": (C.c_int, [C.c_uint64, C.POINTER(C.c_void_p)]),
    "scendp_host_free_pinned": (C.c_int, [C.c_void_p]),
    "scendp_memcpy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32,
                                C.c_uint32]),
    "scendp_memset": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_uint64]),
    "scendp_tiled_bytes": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "scendp_gen_scenarios": (C.c_int, [C.c_void_p, C.POINTER(Dist), C.c_uint64, C.c_uint64,
                                       C.c_uint64, C.c_uint32, C.c_void_p]),
    "scendp_scenarios_to_tiled": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                            C.c_void_p]),
    "scendp_scnb_header_read": (C.c_int, [C.c_char_p, C.POINTER(ScnbHeader)]),
    "scendp_scnb_load": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint32,
                                   C.c_void_p]),
    "scendp_scnb_write": (C.c_int, [C.c_char_p, C.c_void_p, C.c_uint64, C.c_uint64]),
    "scendp_agg_finalize": (C.c_int, [C.POINTER(AggRaw), C.c_uint32, C.c_uint32,
                                      C.POINTER(Agg)]),
    "scendp_split_eval": (C.c_int, [C.c_void_p, C.POINTER(Routing), C.c_void_p, C.c_uint32,
                                    C.POINTER(Scenarios), C.c_uint32, C.POINTER(SplitOut)]),
    "scendp_best_candidate": (C.c_int64, [C.POINTER(Agg), C.c_uint32]),
    "scendp_dsirp_eval": (C.c_int, [C.c_void_p, C.POINTER(Customer), C.c_uint32,
                                    C.POINTER(Scenarios), C.c_uint32, C.POINTER(DsirpOut)]),
    "scendp_minplus_sweep": (C.c_int, [C.c_void_p, C.POINTER(MinplusStage), C.c_uint32,
                                       C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32,
                                       C.c_uint32, C.c_void_p]),
    "scendp_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "scendp_comm_init_rank": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]),
    "scendp_comm_init_all": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32]),
    "scendp_comm_destroy": (C.c_int, [C.c_void_p]),
    "scendp_timer_start": (C.c_int, [C.c_void_p]),
    "scendp_timer_stop": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "scendp_kernel_stats_get": (C.c_int, [C.c_void_p, C.POINTER(KernelStats), C.c_int32]),
    "scendp_flush_l2": (C.c_int, [C.c_void_p]),
    "scendp_split_footprint": (C.c_int, [C.c_void_p, C.POINTER(Routing), C.c_uint32,
                                         C.POINTER(Scenarios), C.c_uint32, C.POINTER(SplitOut),
                                         C.POINTER(Footprint)]),
    "scendp_dsirp_footprint": (C.c_int, [C.c_void_p, C.POINTER(Customer), C.c_uint32,
                                         C.POINTER(Scenarios), C.c_uint32, C.POINTER(DsirpOut),
                                         C.POINTER(Footprint)]),
    "scendp_ctx_memory": (C.c_int, [C.c_void_p, C.POINTER(MemoryInfo)]),
    "scendp_split_eval_multi": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(Routing),
                                          C.c_void_p, C.c_uint32, C.POINTER(Scenarios),
                                          C.c_uint32, C.POINTER(SplitOut)]),
    "scendp_dsirp_eval_multi": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32,
                                          C.POINTER(Customer), C.c_uint32, C.POINTER(Scenarios),
                                          C.c_uint32, C.POINTER(DsirpOut)]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libscendp_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} not found: build it with `make -C paper_2602_05179_b200/csrc` "
            "(or __graft_entry__.build()); the engine has no CPU fallback")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class ScendpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"scendp status {status}: {msg}")
        self.status = status
        self.msg = msg


class InvalidArgument(ScendpError, ValueError):
    pass


def check(status: int) -> None:
    if status == OK:
        return
    msg = _lib.scendp_last_error().decode(errors="replace")
    if status == ERR_INVALID_ARGUMENT:
        raise InvalidArgument(status, msg)
    raise ScendpError(status, msg)
