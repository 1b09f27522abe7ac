# HEAD check in the re-created container + cfg4 binning/compact-entry A/B
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r02zx_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02zx_pytest.log
for v in bin nobin_nosplit nobin_split; do
  case $v in
    bin) env="PBSM_SPLIT=1";;
    nobin_nosplit) env="PBSM_BIN_BYTES=1000000000000000 PBSM_SPLIT=0";;
    nobin_split) env="PBSM_BIN_BYTES=1000000000000000 PBSM_SPLIT=1";;
  esac
  env $env timeout 600 python bench.py --config 4 --no-e2e --no-cpu-baseline --sub-configs none --steps 5 > gpurun_out/r02zx_${v}_4.json 2> gpurun_out/r02zx_${v}_4.err
  python -c "
import json; d=json.load(open('gpurun_out/r02zx_${v}_4.json'))
print('cfg4 $v', round(d['ms_per_step'],4), 'parity', (d.get('parity') or {}).get('match'), {k: round(v,3) for k,v in d['phases_ms'].items()})" || tail -3 gpurun_out/r02zx_${v}_4.err
done 2>&1 | tee gpurun_out/r02zx_variants.txt
