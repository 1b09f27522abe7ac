# large work items: per-lead hit bitmaps, every pair tested once (base = 4096-entry hit list + second test pass)
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r03r_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r03r_pytest.log
for name in _base ""; do
  for c in 2 3 4; do
    PBSM_LIB_NAME=libpbsm$name.so python tools/timeline.py $c 2>/dev/null | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
print('lib$name cfg$c span', rows[-1]['span_us'], 'tail', [r['dur_us'] for r in rows[:-1]][-3:], 'last starts', [r['start_us'] for r in rows[-4:-1]])"
  done
  for c in 2 3 4; do PBSM_LIB_NAME=libpbsm$name.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --sub-configs none --steps 50 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('lib$name cfg$c bench', round(d['ms_per_step'],4), d['parity']['match'])"; done
done 2>&1 | tee gpurun_out/r03r_large_bitmap_ab.txt
