#!/bin/bash
# Build and bench compile-time variants of libpbsm (experiment harness).
# usage: tools_variants.sh "NAME:DEFINES" ...
set -e
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  PBSM_LIB_NAME=libpbsm_$name.so PBSM_DEFINES="$defs" PBSM_FORCE_BUILD=1 python -c "import __graft_entry__ as g; from paper_1908_11740_b200 import _build; _build.build_library(force=True)" > /dev/null 2>&1
done
for spec in "$@"; do
  name=${spec%%:*}
  PBSM_LIB_NAME=libpbsm_$name.so python bench.py --no-e2e --no-cpu-baseline --steps 10 ${BENCH_ARGS} > gpurun_out/var_$name.json 2>gpurun_out/var_$name.err || true
  python -c "import json,sys; d=json.load(open('gpurun_out/var_$name.json')); print('$name', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})" || tail -3 gpurun_out/var_$name.err
done
