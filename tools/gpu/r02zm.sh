for c in 5 4; do
  for sp in 0 1; do
    PBSM_SPLIT=$sp timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --sub-configs none --steps 10 > gpurun_out/r02zm_${sp}_$c.json 2> gpurun_out/r02zm_${sp}_$c.err
    python -c "
import json; d=json.load(open('gpurun_out/r02zm_${sp}_$c.json'))
print('cfg$c split=$sp', round(d['ms_per_step'],4), 'parity', (d.get('parity') or {}).get('match'), {k: round(v,3) for k,v in d['phases_ms'].items()})" || tail -3 gpurun_out/r02zm_${sp}_$c.err
  done
done 2>&1 | tee gpurun_out/r02zm_variants.txt
