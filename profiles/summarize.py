"""Summarize ncu captures (.ncu-rep from gpurun_out/) into the tracked text
files under profiles/.  Usage:

    python profiles/summarize.py <round> gpurun_out/<rep>.ncu-rep[:<name>] ...
    python profiles/summarize.py <round> --launches gpurun_out/launches.csv

Each summary lists duration, DRAM traffic, issue/pipe utilisation, occupancy,
instruction counts and the top stall reasons of the captured launch.  The
DRAM bytes per launch also go to profiles/ncu_traffic.json (read by bench.py
for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = [
    ("Kernel Name", "kernel"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_fp64.sum", "FP64 warp instructions"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
    ("launch__occupancy_limit_registers", "CTA limit (regs)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp instr"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep):
    # a .csv is the raw page exported on the GPU box (capture.sh), else ncu -i
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def summarize(rep, name, rnd):
    h, u, rows = raw(rep)
    r = rows[0]
    lines = [f"# ncu --set full summary: {os.path.basename(rep)} (round {rnd})", ""]
    for key, label in METRICS:
        if key in h:
            i = h.index(key)
            lines.append(f"{label:32s} {r[i]} {u[i]}")
    stalls = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(r[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    lines += ["", "top stall reasons (warps per issue-active cycle):"]
    lines += [f"  {v:7.3f} {k}" for v, k in sorted(stalls, reverse=True)[:8]]
    rd = to_bytes(r[h.index("dram__bytes_read.sum")], u[h.index("dram__bytes_read.sum")])
    wr = to_bytes(r[h.index("dram__bytes_write.sum")], u[h.index("dram__bytes_write.sum")])
    path = os.path.join(HERE, f"r{rnd:02d}_{name}.txt")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    return rd + wr


def launches(csv_path, rnd, suffix=""):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    kn, mv = h.index("Kernel Name"), h.index("Metric Value")
    tot = {}
    cnt = {}
    for r in rows[hi + 1:]:
        if len(r) <= mv:
            continue
        k = r[kn].split("(")[0].replace("void ", "")
        t = float(r[mv].replace(",", ""))
        tot[k] = tot.get(k, 0.0) + t
        cnt[k] = cnt.get(k, 0) + 1
    allt = sum(tot.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none), round {rnd}",
             "# cold-cache, serialised per launch: compare shares, not absolutes", "",
             f"{'kernel':70s} {'launches':>8s} {'total':>12s} {'share':>7s}"]
    for k, t in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k[:70]:70s} {cnt[k]:8d} {t:12.0f} {100 * t / allt:6.1f}%")
    with open(os.path.join(HERE, f"r{rnd:02d}_launches{suffix}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")


def main():
    rnd = int(sys.argv[1])
    args = sys.argv[2:]
    if args and args[0] == "--launches":
        # optional third argument: file suffix (e.g. _headline)
        launches(args[1], rnd, args[2] if len(args) > 2 else "")
        return
    tj = os.path.join(HERE, "ncu_traffic.json")
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    for a in args:
        rep, _, name = a.partition(":")
        name = name or os.path.basename(rep).split(".")[0]
        traffic[name] = summarize(rep, name, rnd)
    with open(tj, "w") as f:
        json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main()
