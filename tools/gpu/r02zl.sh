timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r02zl_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02zl_pytest.log
for c in 2 5 3; do
  for sp in 0 1 r1; do
    if [ $sp = r1 ]; then env="PBSM_SPLIT=1 PBSM_SPLIT_PAIR_RATIO=1.0"; else env="PBSM_SPLIT=$sp"; fi
    env $env timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --sub-configs none --steps 10 > gpurun_out/r02zl_${sp}_$c.json 2> gpurun_out/r02zl_${sp}_$c.err
    python -c "
import json; d=json.load(open('gpurun_out/r02zl_${sp}_$c.json'))
print('cfg$c split=$sp', round(d['ms_per_step'],4), 'parity', (d.get('parity') or {}).get('match'), {k: round(v,3) for k,v in d['phases_ms'].items()})" || tail -3 gpurun_out/r02zl_${sp}_$c.err
  done
done 2>&1 | tee gpurun_out/r02zl_variants.txt
