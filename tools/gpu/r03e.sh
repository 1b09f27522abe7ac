# k_join occupancy variants: kernel timeline (durations in launch order) + bench
for name in "" _jm3 _jm4 _lh2k; do
  for c in 2 3; do
    PBSM_LIB_NAME=libpbsm$name.so python tools/timeline.py $c 2>/dev/null | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
print('lib$name cfg$c span', rows[-1]['span_us'], 'durs', [r['dur_us'] for r in rows[:-1]], 'last starts', [r['start_us'] for r in rows[-4:-1]])"
  done
  PBSM_LIB_NAME=libpbsm$name.so timeout 600 python bench.py --config 2 --no-e2e --no-cpu-baseline --sub-configs none --steps 100 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('lib$name cfg2 bench', round(d['ms_per_step'],4), d['parity']['match'])"
done 2>&1 | tee gpurun_out/r03e_kjoin_occupancy_ab.txt
