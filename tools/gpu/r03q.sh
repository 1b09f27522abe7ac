# count pass with two rectangles per thread and step (16-byte column loads): c2v0 = off, lib = on at 3 CTAs/SM, c2v4 = on at 4 CTAs/SM
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r03q_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r03q_pytest.log
for name in _c2v0 "" _c2v4; do
  for c in 2 3 5; do
    PBSM_LIB_NAME=libpbsm$name.so python tools/timeline.py $c 2>/dev/null | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
print('lib$name cfg$c span', rows[-1]['span_us'], 'first', [(r['start_us'], r['dur_us']) for r in rows[:-1]][:4])"
  done
  for c in 2 3 5 4; do PBSM_LIB_NAME=libpbsm$name.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --sub-configs none --steps 50 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('lib$name cfg$c bench', round(d['ms_per_step'],4), d['parity']['match'])"; done
done 2>&1 | tee gpurun_out/r03q_count2v_ab.txt
