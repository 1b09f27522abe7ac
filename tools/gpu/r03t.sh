# cache policies re-checked with compact 32-byte entries: record stores plain (rh0) / .cs (rh2) instead of L2 evict_first; atomics without evict_last (ah0)
for name in "" _rh0 _rh2 _ah0; do
  for c in 2 3 5; do
    PBSM_LIB_NAME=libpbsm$name.so python tools/timeline.py $c 2>/dev/null | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
d=[r['dur_us'] for r in rows[:-1]]
print('lib$name cfg$c span', rows[-1]['span_us'], 'all', d)"
  done
done 2>&1 | tee gpurun_out/r03t_cache_policy_ab.txt
