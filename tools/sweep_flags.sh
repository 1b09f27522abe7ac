# Bench prebuilt library variants (paper_1908_11740_b200/_lib/libpbsm_NAME.so, built in
# the container with PBSM_DEFINES) on configs 2 and 3.  usage: bash tools/sweep_flags.sh NAME...
mkdir -p gpurun_out
for c in ${SWEEP_CFGS:-2 3}; do
  for name in "$@"; do
    PBSM_LIB_NAME=libpbsm_$name.so python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 \
      > gpurun_out/sw_${name}_$c.json 2> gpurun_out/sw_${name}_$c.err
    python -c "import json; d=json.load(open('gpurun_out/sw_${name}_$c.json')); print('cfg$c $name', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})" || tail -2 gpurun_out/sw_${name}_$c.err
  done
done 2>&1 | tee gpurun_out/sweep.txt
