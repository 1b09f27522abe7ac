#!/bin/bash
# usage: tools/join_variants.sh CONFIG "NAME:DEFINES" ...   (phase times via tools/phase_probe.py)
cfg=$1; shift
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  PBSM_LIB_NAME=libpbsm_$name.so PBSM_DEFINES="$defs" PBSM_FORCE_BUILD=1 python -c "from paper_1908_11740_b200 import _build; _build.build_library(force=True)" > /dev/null 2>&1
  echo -n "$name "; PBSM_LIB_NAME=libpbsm_$name.so PBSM_SPECULATE=0 python tools/phase_probe.py --config $cfg 2>&1 | tail -1
done
