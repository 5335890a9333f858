#!/usr/bin/env python
"""bench.py -- scenario-batched DP throughput on B200 (contract in the task).

Headline (BASELINE.json configs[1], "C2"): CVRPSD split, n=200, Q=100, hard
capacities, identity giant tour, make_random_instance(200, seed=1) costs,
uniform:1:10 demands (the reference default), 10^6 scenarios in total,
STRONG-sharded over the N GPUs: rank g owns the contiguous scenario range
[g*m/N, (g+1)*m/N), generated on its own device with the
reference's streams, so every shard is bit-identical to the 1-GPU run.

  value  one step = one scendp_split_eval per rank over its HBM-resident
         (tiled) shard: K1 DP kernel (+ hand-off pass) + the NCCL all-reduce
         of the 128-byte exact aggregate when N > 1 (overlapped with the next
         step's kernel; the timer ends after the last one); device-timed with
         CUDA events, max over ranks.  Inputs (800 MB) exceed the 126 MB L2,
         so no flush.
  e2e    the reference's own benchmark call, batched_split_costs_generated
         (saa.cpp:366-375), through the C-ABI with host buffers, as an SAA
         caller makes it: every step evaluates a DIFFERENT (instance, giant
         tour) pair -- 4 cost matrices x 8 random tours, cycled -- so each step
         validates its cost matrix, builds its tour tables in pinned memory and
         copies them host->device (nothing is cached across steps), generates
         its shard's demands in-kernel, and reads all per-scenario totals and
         the aggregate back to host memory.  `e2e_host_batch` is the same
         metric with a materialized host ScenarioBatch (800 MB of pinned
         demands H2D per step, batched_split_costs).
  --impl reference  the reference's own CPU implementation (oracle/_ref,
         compiled from /root/reference sources) running the same call with all
         host threads (rank 0 only under torchrun).

--gpus N without torchrun re-launches itself under torch.distributed.run with
N ranks (one process per GPU; fails loudly when fewer than N GPUs are
visible).  NCCL's INIT lines (nRanks) go to stderr.

Secondary lines (weak-scaled C2, random-tour C2 int/fp64, float-cost and
full-solution C2, penalized C2, SAA C5 candidate sweep, DSIRP C3/C4 and the
non-dyadic C3 twin, K5 min-plus, SCNB ingestion) ride in the same JSON object
under "secondary"; at N = 1 each split/DSIRP line carries "cpu_reference",
the reference's own evaluator (oracle/_ref) on a bounded sample of that
workload with all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scenario DP evals/sec (split & DSIRP, 10^6 scen) at 1/2/4/8 B200 vs host CPU"
UNIT = "scenario-evals/s"
N_C2, Q_C2, M_C2 = 200, 100, 1_000_000
TAG_SCENARIO = 0x5343454E
DRY = os.environ.get("SCENDP_BENCH_DRY_RUN") == "1"  # launcher test without a GPU


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=4000)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--scenarios", type=int, default=M_C2, help="scenarios in total (C2)")
    p.add_argument("--no-secondary", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def shard(m: int, rank: int, world: int):
    """[g*m/G, (g+1)*m/G): contiguous scenario range of rank g."""
    return m * rank // world, m * (rank + 1) // world


# ---- launcher ------------------------------------------------------------------
def visible_gpus() -> int:
    import torch
    return torch.cuda.device_count()


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn(args) -> int:
    """Re-run this script under torch.distributed.run with args.gpus ranks."""
    if not DRY and args.impl == "ours":  # the reference arm uses no GPU
        n = visible_gpus()
        if n < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {n}",
                  file=sys.stderr, flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, cwd=ROOT)


# ---- distributed plumbing (gloo: barrier, id broadcast, max over ranks) -------
class Dist:
    def __init__(self):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=self.rank, world_size=self.world)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def bcast_bytes(self, b: bytes) -> bytes:
        if not self.pg:
            return b
        obj = [b]
        self.pg.broadcast_object_list(obj, src=0)
        return obj[0]

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ---- clocks during the timed region --------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # the timed region must be covered: wait for the sampler's first line
        t_end = time.time() + 5.0
        while time.time() < t_end and self.proc.poll() is None:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                pass
            time.sleep(0.02)

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                try:
                    rows.append((float(parts[1]), float(parts[2]), float(parts[3]), parts[5:9]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        smax = max(r[1] for r in rows)
        load = [r for r in rows if r[2] > 250.0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[3]) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": smax,
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(load),
                "power_w_max": max(r[2] for r in rows)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(name: str):
    """dram bytes per launch from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(name)
    except Exception:
        return None


def workload_config(args, world):
    return {"workload": "C2: CVRPSD split n=200 Q=100 hard, identity giant tour, "
                        "make_random_instance(200, seed=1), uniform:1:10 demands, "
                        f"{args.scenarios} scenarios in total",
            "n": N_C2, "Q": Q_C2, "scenarios": args.scenarios, "tours": 1,
            "mode": "hard (linear deque)",
            "parallelism": f"scenario shards x{world}: rank g owns [g*m/{world}, (g+1)*m/{world})",
            "l2": "inputs (4n B/scenario = 800 MB) exceed the 126 MB L2; no flush"}


def base_line(args, world, value, ms_step, scaling, dtype):
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": dtype,
            "data": "synthetic (seeded generator, bit-identical to the reference's)",
            "config": workload_config(args, world)}


# ---- reference (CPU) arm -------------------------------------------------------
def reference_rate(m: int, threads: int, reps: int, warmup: int, budget_s: float = 60.0):
    from oracle import UNIFORM, Reference
    R = Reference()
    costs = R.make_random_instance(N_C2, 1)
    tour = np.arange(1, N_C2 + 1, dtype=np.int32)
    seed = R.derive_stream(1, TAG_SCENARIO, 0)
    # warm-up like run_scaling_benchmark (saa.cpp:364-368)
    R.split_costs_generated(N_C2, Q_C2, 1, 0.0, costs, tour, UNIFORM, 1, 10, seed,
                            min(m, 1000), threads, want_totals=False)
    for _ in range(warmup):
        R.split_costs_generated(N_C2, Q_C2, 1, 0.0, costs, tour, UNIFORM, 1, 10, seed, m,
                                threads, want_totals=False)
    times = []
    t_end = time.perf_counter() + budget_s
    for _ in range(reps):
        t0 = time.perf_counter()
        R.split_costs_generated(N_C2, Q_C2, 1, 0.0, costs, tour, UNIFORM, 1, 10, seed, m,
                                threads, want_totals=True)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end:
            break
    return m / (sum(times) / len(times)), len(times)


def run_reference(args, d: Dist):
    if d.rank != 0:
        return
    threads = os.cpu_count() or 1
    # bounded sample: the full 10^6 scenarios per step unless that would
    # exceed ~60 s for the requested steps
    probe, _ = reference_rate(100_000, threads, 1, 0)
    m = args.scenarios
    if args.steps * m / probe > 60.0:
        m = max(10_000, int(60.0 * probe / max(1, args.steps)))
    rate, done = reference_rate(m, threads, args.steps, min(args.warmup, 3))
    line = base_line(args, d.world, rate, m / rate * 1e3, "strong", "f64")
    line["steps"] = done
    line["impl"] = "reference"
    line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                            "sample": f"batched_split_costs_generated, {m} scenarios per step, "
                                      f"{threads} threads (BackendConfig::multi_thread)"}
    line["e2e"] = {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


# ---- our arm -------------------------------------------------------------------
def timed(ctx, d: Dist, fn, steps: int, warmup: int):
    """W untimed steps, then K steps between barrier + device sync on both
    sides, CUDA events on the library stream; returns (max over ranks, local,
    kernel stats of the timed region)."""
    for i in range(warmup):
        fn(i)
    ctx.sync()
    ctx.kernel_stats(reset=True)
    d.barrier()
    ctx.sync()
    ctx.timer_start()
    for i in range(steps):
        fn(warmup + i)
    ms = ctx.timer_stop()  # synchronizes (and waits for the last all-reduce)
    st = ctx.kernel_stats(reset=True)
    d.barrier()
    return d.max(ms), ms, st


def run_dry(args, d: Dist):
    """SCENDP_BENCH_DRY_RUN=1: the launcher / rank plumbing without a GPU
    (tests/test_bench_launcher.py): barrier, max over ranks, one line."""
    lo, hi = shard(args.scenarios, d.rank, d.world)
    d.barrier()
    ms = d.max(1.0 + 0.5 * d.rank)
    total = d.max(float(hi - lo)) * d.world  # equal shards in the test
    line = base_line(args, d.world, args.scenarios / (ms / 1e3), ms, "strong", "f64")
    line["dry_run"] = {"shard": [lo, hi], "sum_of_shards_le": total}
    if d.rank == 0:
        print(json.dumps(line), flush=True)


def run_ours(args, d: Dist):
    from paper_2602_05179_b200 import (Context, Distribution, derive_stream,
                                       make_random_instance, pinned_empty)
    from paper_2602_05179_b200 import _capi as A
    import ctypes
    ctx = Context(d.local_rank, timing=True)
    if d.world > 1:
        uid = d.bcast_bytes(Context.nccl_unique_id() if d.rank == 0 else b"")
        ctx.comm_init_rank(uid, d.world, d.rank)
    hbm_peak, peak_src = peaks()
    n = N_C2
    lo, hi = shard(args.scenarios, d.rank, d.world)
    m = hi - lo
    inst = make_random_instance(n, 1, Q_C2, True)
    tour = np.arange(1, n + 1, dtype=np.int32)
    dist = Distribution("uniform", 1, 10, seed=derive_stream(1, TAG_SCENARIO, 0))
    scen = ctx.gen_scenarios(dist, n, m, w0=lo)          # HBM-resident, tiled
    tot = ctx.alloc(m * 8)

    call = ctx.split_eval(inst, tour, (scen, A.MEM_DEVICE_TILED), count=m, first_index=lo,
                          out_kind="device_tiled", device_out={"totals": tot}, sync=False,
                          prepare=True)  # the C-ABI call, argument structs built once

    def step(_):
        call()

    clocks = Clocks(d.local_rank)
    clocks.start()
    ms_max, ms_local, st = timed(ctx, d, step, args.steps, args.warmup)
    clk = clocks.stop()
    ms_step = ms_max / args.steps
    value = args.scenarios / (ms_step / 1e3)
    k_ms = st["dp_ms"] / max(1, st["dp_launches"])
    bytes_per_launch = m * (4 * n + 8)
    achieved = bytes_per_launch / (k_ms / 1e3) / 1e9
    # the timed path's aggregate, all-reduced over the ranks (exact)
    chk = ctx.split_eval(inst, tour, (scen, A.MEM_DEVICE_TILED), count=m, first_index=lo,
                         totals=False)

    # ---- e2e: reference-facing call with host buffers, new inputs each step --
    host_tot = pinned_empty(max(1, m), np.float64)
    insts = [make_random_instance(n, s, Q_C2, True) for s in (1, 2, 3, 4)]
    rng = np.random.default_rng(17)
    tours = [(rng.permutation(n) + 1).astype(np.int32) for _ in range(8)]
    c_insts = [x.as_c() for x in insts]
    c_dist = dist.as_c()
    c_sc = A.Scenarios(A.MEM_GENERATED, None, n, m, lo, ctypes.pointer(c_dist))
    c_agg = (A.Agg * 1)()
    c_out = A.SplitOut(A.MEM_HOST, host_tot.ctypes.data, None, None, None, None, c_agg, None)

    def e2e_step(i):
        A.check(ctx.lib.scendp_split_eval(ctx.handle, ctypes.byref(c_insts[i % 4]),
                                          tours[i % 8].ctypes.data, 1, ctypes.byref(c_sc), 0,
                                          ctypes.byref(c_out)))

    e2e_steps = max(8, min(args.steps, 400))
    e_ms_max, _, est = timed(ctx, d, e2e_step, e2e_steps, max(3, args.warmup))
    e2e = {"value": args.scenarios / (e_ms_max / e2e_steps / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": est["h2d_bytes"] // e2e_steps,
           "d2h_bytes_per_step": est["d2h_bytes"] // e2e_steps,
           "steps": e2e_steps,
           "call": "scendp_split_eval(GENERATED uniform:1:10 shard, host totals) == "
                   "batched_split_costs_generated; a different (instance, random giant tour) "
                   "each step: validation, tour tables built and copied H2D every step",
           "gpu_launches": est["launches"]}
    # materialized host ScenarioBatch (reference layout, pinned) of this shard
    ref_layout = ctx.gen_scenarios(dist, n, m, w0=lo, tiled=False)
    host_batch = pinned_empty(m * n, np.uint32)
    A.check(ctx.lib.scendp_memcpy(ctx.handle, host_batch.ctypes.data, ref_layout.ptr,
                                  m * n * 4, 1, 0))
    ref_layout.free()
    hb = host_batch.reshape(m, n)

    def host_step(i):
        ctx.split_eval(insts[i % 4], tours[i % 8], hb, host_totals=host_tot, first_index=lo)

    h_steps = max(3, min(args.steps, 20))
    h_ms_max, _, hst = timed(ctx, d, host_step, h_steps, 1)
    e2e_host = {"value": args.scenarios / (h_ms_max / h_steps / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": hst["h2d_bytes"] // h_steps,
                "d2h_bytes_per_step": hst["d2h_bytes"] // h_steps,
                "call": "scendp_split_eval(HOST pinned ScenarioBatch shard) == batched_split_costs"}
    pageable = np.array(hb, copy=True)
    p_ms_max, _, pst = timed(ctx, d, lambda i: ctx.split_eval(
        insts[i % 4], tours[i % 8], pageable, host_totals=host_tot, first_index=lo), h_steps, 1)
    e2e_host_pageable = {"value": args.scenarios / (p_ms_max / h_steps / 1e3), "unit": UNIT,
                         "h2d_bytes_per_step": pst["h2d_bytes"] // h_steps,
                         "d2h_bytes_per_step": pst["d2h_bytes"] // h_steps,
                         "call": "scendp_split_eval(HOST pageable ScenarioBatch shard)"}
    del pageable
    scen_tot_check = float(np.sum(host_tot[:m]))  # keep the D2H result live

    line = base_line(args, d.world, value, ms_step, "strong",
                     "f64 (exact int32 path: integral costs, bit-identical to fp64)")
    line.update({
        "gpu_launches": st["launches"],
        "kernel_ms": k_ms,
        "bellman_state_updates_per_s": value * n,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": ncu_traffic("split_linear_c2"),
                     "kernel": "split_linear_kernel<cost-only, tiled, int32, identity tour>",
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "unit_bytes": "4n+8 per scenario (demand column read once, total written once)",
                     "peak_source": peak_src},
        "clocks": clk,
        "e2e": e2e,
        "e2e_host_batch": e2e_host,
        "e2e_host_batch_pageable": e2e_host_pageable,
        "check": {"mean_cost": chk["agg"][0]["mean"], "finite": chk["agg"][0]["finite_count"],
                  "host_totals_sum_rank0": scen_tot_check},
    })
    scen.free()
    tot.free()
    if d.world == 1 and not args.no_cpu_baseline and d.rank == 0:
        line["cpu_baseline"] = cpu_baseline()
    if not args.no_secondary:
        line["secondary"] = secondary(ctx, d, args)
        if d.world == 1 and not args.no_cpu_baseline:
            try:
                for k, v in cpu_reference_secondary().items():
                    if k in line["secondary"]:
                        v["unit"] = line["secondary"][k]["unit"]
                        line["secondary"][k]["cpu_reference"] = v
            except Exception as e:  # reference library missing on this box
                line["secondary_cpu_reference"] = f"unavailable: {e}"
    if d.world > 1:
        ctx.comm_destroy()
    ctx.close()
    if d.rank == 0:
        print(json.dumps(line), flush=True)


def cpu_baseline():
    threads = os.cpu_count() or 1
    try:
        rate, reps = reference_rate(M_C2, threads, 20, 1, budget_s=15.0)
        rate1, _ = reference_rate(50_000, 1, 3, 0, budget_s=10.0)
    except Exception as e:  # reference library missing on this box
        return {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"unavailable: {e}"}
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"batched_split_costs_generated C2, {M_C2} scenarios x {reps} reps, "
                      f"{threads} threads",
            "single_thread_value": rate1}


def secondary(ctx, d: Dist, args):
    from paper_2602_05179_b200 import (Customer, Distribution, RoutingInstance, derive_stream,
                                       make_random_instance, pinned_empty)
    from paper_2602_05179_b200 import _capi as A
    out = {}
    hbm_peak, _ = peaks()
    n, G, g = N_C2, d.world, d.rank

    def kernel_rate(fn, steps, warm=2):
        """fn: a prepared C-ABI call (argument structs built once) or any callable"""
        ms_max, ms, st = timed(ctx, d, lambda i: fn(), steps, warm)
        return ms_max / steps, st["dp_ms"] / max(1, st["dp_launches"])

    def frac(nbytes, k_ms):
        return nbytes / (k_ms / 1e3) / 1e9 / hbm_peak

    # C2 weak-scaled: 10^6 scenarios per GPU (rank g owns [g*10^6, (g+1)*10^6))
    mw = M_C2
    distw = Distribution("uniform", 1, 10, seed=0x5eed)
    scen = ctx.gen_scenarios(distw, n, mw, w0=g * mw)
    tot = ctx.alloc(mw * 8)
    iinst = make_random_instance(n, 1, Q_C2, True)
    ident = np.arange(1, n + 1, dtype=np.int32)
    step_ms, k_ms = kernel_rate(ctx.split_eval(
        iinst, ident, (scen, A.MEM_DEVICE_TILED), count=mw, first_index=g * mw,
        out_kind="device_tiled", device_out={"totals": tot}, sync=False, prepare=True), 50)
    out["split_c2_weak"] = {"value": G * mw / (step_ms / 1e3), "unit": UNIT, "kernel_ms": k_ms,
                            "scaling": "weak", "scenarios_per_gpu": mw,
                            "roofline_frac": frac(mw * (4 * n + 8), k_ms)}

    # strong shards of the 10^6-scenario sets below
    lo, hi = shard(M_C2, g, G)
    m = hi - lo
    dist = Distribution("uniform", 1, 10, seed=77)
    scen2 = ctx.gen_scenarios(dist, n, m, w0=lo)
    rng = np.random.default_rng(1)
    c = rng.random((n + 2, n + 2)) * 20.0
    c = np.triu(c, 1)
    c = c + c.T
    finst = RoutingInstance(n, Q_C2, True, 0.0, c)
    rtour = (np.random.default_rng(7).permutation(n) + 1).astype(np.int32)
    for name, inst_, tour_ in (("split_c2_float_costs", finst, ident),
                               ("split_c2_random_tour", iinst, rtour),
                               ("split_c2_random_tour_float", finst, rtour)):
        step_ms, k_ms = kernel_rate(ctx.split_eval(
            inst_, tour_, (scen2, A.MEM_DEVICE_TILED), count=m, first_index=lo,
            out_kind="device_tiled", device_out={"totals": tot}, sync=False, prepare=True), 50)
        out[name] = {"value": M_C2 / (step_ms / 1e3), "unit": UNIT, "kernel_ms": k_ms,
                     "dtype": "f64" if inst_ is finst else "int32-exact",
                     "tour": "identity" if tour_ is ident else "random permutation (SAA case)",
                     "roofline_frac": frac(m * (4 * n + 8), k_ms), "scaling": "strong"}
    V = ctx.alloc(ctx.tiled_bytes(n + 1, m) * 2)
    cuts = ctx.alloc(ctx.tiled_bytes(n + 1, m))
    rc = ctx.alloc(m * 4)
    fe = ctx.alloc(m)
    step_ms, k_ms = kernel_rate(ctx.split_eval(
        iinst, ident, (scen2, A.MEM_DEVICE_TILED), count=m, first_index=lo, full=True,
        out_kind="device_tiled",
        device_out={"totals": tot, "values": V, "cuts": cuts, "route_count": rc, "feasible": fe},
        sync=False, prepare=True), 10)
    out["split_c2_full_solution"] = {
        "value": M_C2 / (step_ms / 1e3), "unit": UNIT, "kernel_ms": k_ms, "scaling": "strong",
        "roofline_frac": frac(m * (4 * n + 8 + 12 * (n + 1)), k_ms)}
    for b in (V, cuts, rc, fe):
        b.free()
    # penalized split (K2-int, O(n) exact form), n = 200
    pinst = make_random_instance(n, 1, Q_C2, False, 10.0)
    mp = min(m, 200_000)
    step_ms, k_ms = kernel_rate(ctx.split_eval(
        pinst, ident, (scen2, A.MEM_DEVICE_TILED), count=mp, first_index=lo,
        out_kind="device_tiled", device_out={"totals": tot}, sync=False, prepare=True), 5, 1)
    out["split_c2_penalized"] = {"value": G * mp / (step_ms / 1e3), "unit": UNIT,
                                 "kernel_ms": k_ms, "scenarios_per_gpu": mp, "scaling": "weak",
                                 "dense_candidates_per_s": G * mp * n * (n + 1) / 2 / (step_ms / 1e3)}
    # adversarial hand-off cliff: a line metric (f increases along the
    # identity tour, nothing pops) with zero-heavy demands uniform:0:2 keeps
    # ~100 entries in every deque -- no scenario fits K1's ring, all 10^5
    # take the hand-off (generic) pass.  Timed per call (K1 + the pass).
    ma = min(m, 100_000)
    idx = np.arange(n + 2, dtype=np.float64)
    ainst = RoutingInstance(n, Q_C2, True, 0.0, np.abs(idx[:, None] - idx[None, :]))
    scena = ctx.gen_scenarios(Distribution("uniform", 0, 2, seed=91), n, ma, w0=lo)
    step_ms, k_ms = kernel_rate(ctx.split_eval(
        ainst, ident, (scena, A.MEM_DEVICE_TILED), count=ma, first_index=lo,
        out_kind="device_tiled", device_out={"totals": tot}, sync=False, prepare=True), 5, 1)
    out["split_c2_adversarial_handoff"] = {
        "value": G * ma / (step_ms / 1e3), "unit": UNIT, "ms_per_call": step_ms,
        "k1_kernel_ms": k_ms, "scenarios_per_gpu": ma, "scaling": "weak",
        "config": "n=200 Q=100 line metric, identity tour, uniform:0:2: every scenario handed off"}
    scena.free()
    scen.free()
    scen2.free()
    tot.free()

    # C1 (BASELINE configs[0], the reference's CPU-runnable case): n = 50,
    # Q = 100, one fixed giant tour, 1,024 seeded Poisson(5) scenarios
    # generated inside the DP kernel; a synchronous call with host totals --
    # launch-latency-bound at this size, so timed per call
    from paper_2602_05179_b200 import poisson_hi
    n1, m1 = 50, 1024
    inst1 = make_random_instance(n1, 1, Q_C2, True)
    d1 = Distribution("poisson", 0, poisson_hi(5.0), mean=5.0, seed=derive_stream(1, 0x5343454E, 0))
    t1 = np.arange(1, n1 + 1, dtype=np.int32)
    h1 = pinned_empty(m1, np.float64)
    c1 = ctx.split_eval(inst1, t1, d1, count=m1, host_totals=h1, prepare=True)
    step_ms, _ = kernel_rate(c1, 200, 5)
    out["split_c1"] = {"value": m1 / (step_ms / 1e3), "unit": UNIT, "ms_per_call": step_ms,
                       "scaling": "replicated (whole C1 per rank)",
                       "config": "C1: n=50 Q=100 hard, identity tour, 1024 Poisson(5) scenarios, "
                                 "generated in-kernel, host totals"}

    # C5: 1000 giant tours x 10^5 scenarios, n = 50, penalized beta = 10, one
    # launch per rank over its scenario shard; the K x 16-word exact aggregate
    # is all-reduced, so the argmin is over the whole 10^5
    n5, m5, K5 = 50, 100_000, 1000
    inst5 = make_random_instance(n5, 5, Q_C2, False, 10.0)
    rng = np.random.default_rng(5)
    tours5 = np.stack([rng.permutation(n5) + 1 for _ in range(K5)]).astype(np.int32)
    lo5, hi5 = shard(m5, g, G)
    scen5 = ctx.gen_scenarios(Distribution("uniform", 1, 10, seed=55), n5, hi5 - lo5, w0=lo5)
    # the C-ABI call with its argument structs built once (the aggregates of
    # all 1000 tours are read back and all-reduced every call); the argmin
    # comes from one more call through the Python mirror afterwards
    c5 = ctx.split_eval(inst5, tours5, (scen5, A.MEM_DEVICE_TILED), count=hi5 - lo5,
                        first_index=lo5, totals=False, prepare=True)
    step_ms, k_ms = kernel_rate(c5, 3, 1)
    best5 = ctx.split_eval(inst5, tours5, (scen5, A.MEM_DEVICE_TILED), count=hi5 - lo5,
                           first_index=lo5, totals=False)["best"]
    out["saa_c5_candidates"] = {
        "value": K5 * m5 / (step_ms / 1e3), "unit": "(tour, scenario)-evals/s",
        "candidates_per_s": K5 / (step_ms / 1e3), "ms_per_launch": step_ms, "kernel_ms": k_ms,
        "best_tour": best5, "scaling": "strong",
        "config": "K=1000 tours x 1e5 scenarios, n=50, beta=10"}
    scen5.free()

    # DSIRP C3 (50 customers, H=6, 1e5; weak), C4 (200 customers, H=6, 1e6
    # sharded over the ranks) and the non-dyadic C3 twin (K3 fp64 path)
    H = 6
    rngf = np.random.default_rng(21)
    fcusts = [Customer(U=100, I0=50, H=H, h=0.5 + rngf.random(), rho=1.5 + rngf.random(),
                       fixed=30 + 20 * rngf.random((H, 3)), unit=0.25 + rngf.random((H, 3)))
              for _ in range(50)]
    for name, nc, mtot, steps, scaling in (("dsirp_c3", 50, 100_000, 20, "weak"),
                                           ("dsirp_c4", 200, 1_000_000, 5, "strong"),
                                           ("dsirp_c3_float", 50, 100_000, 20, "weak")):
        if scaling == "strong":
            l3, h3 = shard(mtot, g, G)
        else:
            l3, h3 = g * mtot, (g + 1) * mtot
        m3 = h3 - l3
        custs = fcusts if name == "dsirp_c3_float" else [
            Customer(U=100, I0=50, H=H, h=1.0, rho=2.0,
                     fixed=np.tile(40 + 5 * np.arange(3.0), (H, 1)),
                     unit=np.tile(0.5 + 0.25 * np.arange(3.0), (H, 1))) for _ in range(nc)]
        sc = ctx.gen_scenarios(Distribution("uniform", 0, 33, seed=7), nc * H, m3, w0=l3)
        t3 = ctx.alloc(nc * m3 * 8)
        step_ms, k_ms = kernel_rate(ctx.dsirp_eval(
            custs, (sc, A.MEM_DEVICE_TILED), count=m3, first_index=l3, out_kind="device_tiled",
            device_out={"totals": t3}, sync=False, prepare=True), steps)
        units = nc * (mtot if scaling == "strong" else G * mtot)
        out[name] = {"value": units / (step_ms / 1e3), "unit": "(customer, scenario)-evals/s",
                     "kernel_ms": k_ms, "customers": nc, "scenarios": units // nc,
                     "bellman_state_updates_per_s": units * H * 101 / (step_ms / 1e3),
                     "roofline_frac": frac(nc * m3 * (4 * H + 8), k_ms),
                     "unit_bytes": "4H+8 per (customer, scenario)", "scaling": scaling,
                     "dtype": "f64" if name == "dsirp_c3_float" else "int32-exact (dyadic pins)"}
        sc.free()
        t3.free()
    if G > 1:
        return out

    # K5: generic dense (min,+) sweep -- the DSIRP dense chain shape (H = 6
    # stages of 101 x 101, option depth 3) for 10^5 frontiers
    rng = np.random.default_rng(11)
    stages = []
    for _ in range(6):
        st = np.floor(rng.random((3, 101, 101)) * 100.0)
        st[rng.random(st.shape) < 0.5] = np.inf
        stages.append(st)
    B = 100_000
    init = np.full((B, 101), np.inf)
    init[np.arange(B), rng.integers(0, 101, B)] = 0.0
    ctx.minplus_sweep(stages, init[:1000])
    ctx.kernel_stats(reset=True)
    t0 = time.perf_counter()
    ctx.minplus_sweep(stages, init)
    wall = time.perf_counter() - t0
    st1 = ctx.kernel_stats(reset=True)
    cand = B * 6 * 3 * 101 * 101
    out["minplus_k5"] = {"value": cand / (st1["dp_ms"] / 1e3), "unit": "candidate updates/s",
                         "kernel_ms": st1["dp_ms"], "wall_ms_with_host_copies": wall * 1e3,
                         "fp64_ops_per_s": 2 * cand / (st1["dp_ms"] / 1e3),
                         "config": "6 stages x 3 options x 101x101, 1e5 frontiers (FP64 add+min)"}

    # SCNB ingestion (io.cpp:276-344): the C2 scenario set as an 800 MB file
    # streamed into the tiled HBM layout (parallel pread -> pinned double
    # buffers -> H2D -> to_tiled)
    import tempfile
    nf, mf = 200, 1_000_000
    host = ctx.gen_scenarios(Distribution("uniform", 1, 10, seed=3), nf, mf, tiled=False)
    arr = host.download(np.uint32, nf * mf).reshape(mf, nf)
    host.free()
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "c2.scnb")
        ctx.scnb_write(path, arr)
        ctx.scnb_load(path).free()  # warm the page cache and staging buffers
        wall = float("inf")
        for _ in range(3):  # best of 3 (the host page cache is shared)
            t0 = time.perf_counter()
            buf = ctx.scnb_load(path)
            wall = min(wall, time.perf_counter() - t0)
            buf.free()
    out["scnb_ingest"] = {"value": arr.nbytes / wall / 1e9, "unit": "GB/s (file -> tiled HBM)",
                          "bytes": arr.nbytes, "wall_ms": wall * 1e3,
                          "note": "page-cached 800 MB file (C2 set), best of 3"}
    return out


def cpu_reference_secondary():
    """The reference's own evaluators (oracle/_ref) on bounded samples of the
    secondary workloads (SURVEY 8d "CPU reference timing"), all host threads;
    rate = units of the sample / wall time of one call after a warm-up."""
    from oracle import UNIFORM, Customer as RefCust, Reference
    R = Reference()
    threads = os.cpu_count() or 1
    out = {}

    def rate(fn, units):
        fn()  # warm-up (saa.cpp:364-368)
        t0 = time.perf_counter()
        fn()
        return units / (time.perf_counter() - t0)

    n = N_C2
    tour = np.arange(1, n + 1, dtype=np.int32)
    rtour = (np.random.default_rng(7).permutation(n) + 1).astype(np.int32)
    ms = 20_000
    dem = R.generate(UNIFORM, 1, 10, 77, n, 1, ms)
    rng = np.random.default_rng(1)
    c = rng.random((n + 2, n + 2)) * 20.0
    c = np.triu(c, 1)
    c = c + c.T
    icost = R.make_random_instance(n, 1)
    out["split_c2_weak"] = (rate(lambda: R.split_costs(n, Q_C2, 1, 0.0, icost, tour, dem,
                                                        threads), ms),
                            f"batched_split_costs, {ms} scenarios")
    out["split_c2_float_costs"] = (rate(lambda: R.split_costs(n, Q_C2, 1, 0.0, c, tour, dem,
                                                               threads), ms),
                                   f"batched_split_costs, float-cost twin, {ms} scenarios")
    out["split_c2_random_tour"] = (rate(lambda: R.split_costs(n, Q_C2, 1, 0.0, icost, rtour, dem,
                                                               threads), ms),
                                   f"batched_split_costs, random tour, {ms} scenarios")
    out["split_c2_random_tour_float"] = (rate(lambda: R.split_costs(n, Q_C2, 1, 0.0, c, rtour,
                                                                     dem, threads), ms),
                                         f"batched_split_costs, random tour, float costs, "
                                         f"{ms} scenarios")
    out["split_c2_full_solution"] = (rate(lambda: R.expected_split(n, Q_C2, 1, 0.0, icost, tour,
                                                                    dem, threads), ms),
                                     f"batched_expected_split, {ms} scenarios")
    mp = 2_000
    out["split_c2_penalized"] = (rate(lambda: R.split_costs(n, Q_C2, 0, 10.0, icost, tour,
                                                             dem[:mp], threads), mp),
                                 f"batched_split_costs penalized beta=10, {mp} scenarios")
    idx = np.arange(n + 2, dtype=np.float64)
    lcost = np.abs(idx[:, None] - idx[None, :])
    dema = R.generate(UNIFORM, 0, 2, 91, n, 1, ms)
    out["split_c2_adversarial_handoff"] = (rate(lambda: R.split_costs(n, Q_C2, 1, 0.0, lcost, tour,
                                                                       dema, threads), ms),
                                           f"batched_split_costs, line metric, uniform:0:2, "
                                           f"{ms} scenarios")
    # C1: the reference's batched_split_costs on the same 1,024 Poisson(5)
    # scenarios (the reference has no Poisson kind; the oracle restatement
    # samples them -- cpu-baseline leg only)
    from oracle import POISSON, Oracle
    from paper_2602_05179_b200 import poisson_hi
    O = Oracle()
    dem1 = O.generate(POISSON, 0, poisson_hi(5.0), R.derive_stream(1, 0x5343454E, 0), 50, 1024,
                      mean=5.0)
    c1 = R.make_random_instance(50, 1)
    t1 = np.arange(1, 51, dtype=np.int32)
    out["split_c1"] = (rate(lambda: R.split_costs(50, Q_C2, 1, 0.0, c1, t1, dem1, threads), 1024),
                       "batched_split_costs, C1 (n=50, 1024 Poisson(5) scenarios)")
    # C5: K calls of batched_split_costs (saa.cpp:127-131), timed on 4 tours
    n5, m5, k5 = 50, 100_000, 4
    cost5 = R.make_random_instance(n5, 5)
    dem5 = R.generate(UNIFORM, 1, 10, 55, n5, 1, m5)
    rng5 = np.random.default_rng(5)
    tours5 = [(rng5.permutation(n5) + 1).astype(np.int32) for _ in range(k5)]
    out["saa_c5_candidates"] = (rate(lambda: [R.split_costs(n5, Q_C2, 0, 10.0, cost5, t, dem5,
                                                            threads) for t in tours5], k5 * m5),
                                f"{k5} tours x batched_split_costs (n=50, beta=10, 10^5 scenarios)")
    # DSIRP: batched_expected_cost per customer (the reference has no
    # multi-customer call), 4 customers x 10^5 scenarios
    H, m3, nc = 6, 100_000, 4
    cust = RefCust(U=100, I0=50, H=H, h=1.0, rho=2.0,
                   fixed=np.tile(40 + 5 * np.arange(3.0), (H, 1)),
                   unit=np.tile(0.5 + 0.25 * np.arange(3.0), (H, 1)))
    d3 = R.generate(UNIFORM, 0, 33, 7, 1, H, m3)
    r3 = rate(lambda: [R.expected_cost(cust, d3, threads) for _ in range(nc)], nc * m3)
    for name in ("dsirp_c3", "dsirp_c4"):
        out[name] = (r3, f"{nc} customers x batched_expected_cost (U=100, H=6, R=3, 10^5)")
    rngf = np.random.default_rng(21)
    fc = RefCust(U=100, I0=50, H=H, h=0.5 + rngf.random(), rho=1.5 + rngf.random(),
                 fixed=30 + 20 * rngf.random((H, 3)), unit=0.25 + rngf.random((H, 3)))
    out["dsirp_c3_float"] = (rate(lambda: [R.expected_cost(fc, d3, threads) for _ in range(nc)],
                                  nc * m3),
                             f"{nc} customers x batched_expected_cost, non-dyadic costs")
    return {k: {"value": v, "cores": threads, "kind": "reference", "sample": smp}
            for k, (v, smp) in out.items()}


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn(args))
    if args.gpus > 1 or int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # NCCL's communicator lines (nRanks, rings, NVLS) on stderr; stdout
        # keeps the single JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    d = Dist()
    if d.world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={d.world}", file=sys.stderr, flush=True)
        d.close()
        sys.exit(2)
    try:
        if args.impl == "reference":
            run_reference(args, d)
        elif DRY:
            run_dry(args, d)
        else:
            run_ours(args, d)
    finally:
        d.close()


if __name__ == "__main__":
    main()
