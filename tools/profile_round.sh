#!/bin/bash
# GPU-box side of a profiling round (run under gpurun).  Outputs in gpurun_out/.
# usage: tools/profile_round.sh TAG CONFIG
set -u
tag=${1:-r01}; cfg=${2:-2}; kre=${3:-k_join|k_scatter|k_count}; skip=${4:-12}
CMD="python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --sub-configs none --no-parity"
mkdir -p gpurun_out
$CMD > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/${tag}_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_cfg${cfg}_launches.csv $CMD > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"$kre" \
    -s $skip -c 5 -o gpurun_out/${tag}_cfg${cfg}_full $CMD > gpurun_out/${tag}_ncu_full.log 2>&1
echo "full rc=$?"
