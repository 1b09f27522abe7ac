# large work item -> tile table written by the plan (k_join skips its 32-ary search)
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r03o_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r03o_pytest.log
for name in _base ""; do
  for c in 2 3; do
    PBSM_LIB_NAME=libpbsm$name.so python tools/timeline.py $c 2>/dev/null | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
print('lib$name cfg$c span', rows[-1]['span_us'], 'plan', [r['dur_us'] for r in rows[:-1]][3:6], 'tail', [r['dur_us'] for r in rows[:-1]][-3:], 'last starts', [r['start_us'] for r in rows[-4:-1]])"
  done
  for c in 2 3 4; do PBSM_LIB_NAME=libpbsm$name.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --sub-configs none --steps 50 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('lib$name cfg$c bench', round(d['ms_per_step'],4), d['parity']['match'])"; done
done 2>&1 | tee gpurun_out/r03o_item_table_ab.txt
