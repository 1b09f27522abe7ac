# nested join occupancy re-check at HEAD: few7 = 7 CTAs/SM for the few-pairs instance (shipped 8), m27 / m25 = 7 / 5 for the other (shipped 6)
for name in "" _few7 _m27 _m25; do
  for c in 2 3 5; do
    PBSM_LIB_NAME=libpbsm$name.so python tools/timeline.py $c 2>/dev/null | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
d=[r['dur_us'] for r in rows[:-1]]
print('lib$name cfg$c span', rows[-1]['span_us'], 'nested', d[-2] if $c==5 else d[-3])"
  done
done 2>&1 | tee gpurun_out/r03x_nested_occupancy_ab.txt
