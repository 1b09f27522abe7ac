#!/bin/bash
# Per-kernel warm-cache launch times of compile-time variants (experiment harness).
# usage: BENCH_ARGS="--config 2" tools/diag_launch.sh "NAME:DEFINES" ...
# (the bench may fail after the kernels of interest ran: the list is kept)
set -u
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  PBSM_LIB_NAME=libpbsm_$name.so PBSM_DEFINES="$defs" PBSM_FORCE_BUILD=1 python -c "from paper_1908_11740_b200 import _build; _build.build_library(force=True)" > /dev/null 2>&1
done
for spec in "$@"; do
  name=${spec%%:*}
  PBSM_LIB_NAME=libpbsm_$name.so ncu --metrics gpu__time_duration.sum --clock-control none \
    --cache-control none --csv --log-file gpurun_out/diag_$name.csv \
    python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 3 ${BENCH_ARGS:-} > /dev/null 2>&1
  python tools/summarize_ncu.py --launches gpurun_out/diag_$name.csv --title "$name" | sed -n '5,30p' | sed "s/^/$name /"
done
