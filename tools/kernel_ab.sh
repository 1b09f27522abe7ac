# per-kernel device times (ncu launch list, gpu__time_duration) of two library builds
# usage: tools/kernel_ab.sh CONFIG NAME...   (paper_1908_11740_b200/_lib/libpbsm_NAME.so)
cfg=$1; shift
mkdir -p gpurun_out
for name in "$@"; do
  PBSM_LIB_NAME=libpbsm_$name.so ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/kab_${name}_c${cfg}.csv python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo "== $name cfg$cfg"; python tools/summarize_ncu.py --launches gpurun_out/kab_${name}_c${cfg}.csv | grep '^| `'
done
