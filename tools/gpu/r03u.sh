# write guard fused into the nested join for up to 128 tiles per thread (g128) vs 32 (cfg3/cfg4 run k_guard on its own at 32)
for name in "" _g128; do
  for c in 3 4; do
    PBSM_LIB_NAME=libpbsm$name.so python tools/timeline.py $c 2>/dev/null | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
d=[r['dur_us'] for r in rows[:-1]]
print('lib$name cfg$c span', rows[-1]['span_us'], 'tail', d[-4:])"
  done
done 2>&1 | tee gpurun_out/r03u_guard_fused_ab.txt
