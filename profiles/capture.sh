#!/usr/bin/env bash
# capture.sh -- one GPU call that produces every measurement under profiles/:
#   1. the benchmark line (no profiler attached)          gpurun_out/bench.json
#   2. the launch list of a short bench run (ncu, gpu__time_duration.sum,
#      --clock-control none; cold-cache, serialised -- shares, not absolutes)
#   3. one `ncu --set full` capture per hot kernel on the fixed workloads of
#      profiles/cases.py (-lineinfo builds: the source page maps to csrc/).
# Run from the repo root under gpurun:
#   gpurun --timeout 3000 -- 'bash profiles/capture.sh r02'
# then, in the container:
#   python profiles/summarize.py 2 --launches gpurun_out/launches.csv
#   python profiles/summarize.py 2 gpurun_out/k1_r02.ncu-rep:split_linear_c2 ...
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p "$OUT"
NCU="ncu --clock-control none --import-source on"

# SKIP_BENCH=1: captures only; CASES=k1,k2: only the named captures
if [ -z "${SKIP_BENCH:-}" ]; then
  python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench rc=$?"
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file "$OUT/launches.csv" \
      python bench.py --steps 2 --warmup 1 > "$OUT/bench_ncu.log" 2>&1
  echo "launch list rc=$?"
fi

cap() {  # cap <name> <kernel regex> <case>
  [ -z "${CASES:-}" ] || [[ ",$CASES," == *",$1,"* ]] || return 0
  timeout 900 $NCU --set full -k "regex:$2" -s 1 -c 1 -f -o "$OUT/$1_$TAG" \
      python profiles/cases.py "$3" > "$OUT/$1.log" 2>&1
  echo "$1 rc=$?"
  # the reports exceed gpurun's copy-back limit together: export the raw and
  # source pages (text) and keep the report itself outside gpurun_out/
  if [ -f "$OUT/$1_$TAG.ncu-rep" ]; then
    ncu -i "$OUT/$1_$TAG.ncu-rep" --page raw --csv > "$OUT/$1_$TAG.raw.csv" 2>/dev/null
    ncu -i "$OUT/$1_$TAG.ncu-rep" --page source --csv --print-source sass \
        > "$OUT/$1_$TAG.sass.csv" 2>/dev/null
    mkdir -p /tmp/ncu_reps && mv "$OUT/$1_$TAG.ncu-rep" /tmp/ncu_reps/
  fi
}
cap k1 split_linear_kernel c2
cap k1gen split_linear_kernel c2gen
cap k1f split_linear_kernel c2float
cap k1r split_linear_kernel c2rand
cap k1rf split_linear_kernel c2randf
cap k2 split_penal c5
cap k3 dsirp_fast_kernel c3
cap k3f dsirp_fast_kernel c3float
cap k3c4 dsirp_fast_kernel c4
cap k5 minplus_stage_kernel k5
if [ -z "${SKIP_BENCH:-}" ]; then
  python profiles/footprint.py > "$OUT/footprint.txt" 2>&1
  echo "footprint rc=$?"
fi
