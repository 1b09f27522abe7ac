# GPU box: bench lines for configs 3-5, an ncu --set full capture of every kernel of one
# cfg2 join step, and launch lists for configs 3-5.  usage: bash tools/profile_all.sh TAG
tag=${1:-r01}
mkdir -p gpurun_out
for c in 3 4 5; do
  python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench_cfg$c.json 2> gpurun_out/${tag}_bench_cfg$c.err
  echo "bench cfg$c rc=$?"
done
CMD="python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
# warm-up: 3 joins (+ 1 untimed probe join in bench) before the timed step; skip them
ncu --set full --clock-control none --import-source on -s 40 -c 12 \
    -o gpurun_out/${tag}_cfg2_allk $CMD > gpurun_out/${tag}_allk.log 2>&1
echo "all-kernel capture rc=$?"
for c in 3 4 5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${tag}_cfg${c}_launches.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo "launch list cfg$c rc=$?"
done
