# fast replay (host path of a repeated join) + no memset node in the bounded emit
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r03c_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r03c_pytest.log
for f in 0 1; do
  for c in 2 5; do
    PBSM_FAST_REPLAY=$f timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --sub-configs none --steps 20 > gpurun_out/r03c_f${f}_$c.json 2> gpurun_out/r03c_f${f}_$c.err
    python -c "
import json; d=json.load(open('gpurun_out/r03c_f${f}_$c.json'))
print('fast=$f cfg$c', round(d['ms_per_step'],4), 'parity', (d.get('parity') or {}).get('match'))" || tail -3 gpurun_out/r03c_f${f}_$c.err
  done
  PBSM_FAST_REPLAY=$f python tools/fixed_cost.py 1000 graph 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print('fast=$f fixed', d['k'], d['rows'], d['us_per_join'])
    except Exception: print(l.rstrip())"
done 2>&1 | tee gpurun_out/r03c_fast_replay_ab.txt
python tools/timeline.py 2 > gpurun_out/r03c_timeline_cfg2.jsonl 2>/dev/null; tail -14 gpurun_out/r03c_timeline_cfg2.jsonl
