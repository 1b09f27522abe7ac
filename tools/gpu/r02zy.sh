# cfg4 with compact entries preferred over the row-band copy; phases of cfg3/cfg5 at HEAD
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r02zy_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02zy_pytest.log
for c in 4 3 5 2; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --sub-configs none --steps 10 > gpurun_out/r02zy_$c.json 2> gpurun_out/r02zy_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/r02zy_$c.json'))
print('cfg$c', round(d['ms_per_step'],4), 'parity', (d.get('parity') or {}).get('match'), {k: round(v,3) for k,v in d['phases_ms'].items()})" || tail -3 gpurun_out/r02zy_$c.err
done 2>&1 | tee gpurun_out/r02zy_variants.txt
