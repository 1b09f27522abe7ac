for name in "" _pm3 _pm2; do
  for c in 2 3 4; do
    PBSM_LIB_NAME=libpbsm$name.so python tools/timeline.py $c 2>/dev/null | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
print('lib$name cfg$c span', rows[-1]['span_us'], 'plan', [r['dur_us'] for r in rows[:-1]][3:6])"
  done
done 2>&1 | tee gpurun_out/r03s_plan_minb_ab.txt
