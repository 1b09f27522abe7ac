# fast replay A/B, interleaved repeats, 100 steps
for i in 1 2 3; do for f in 0 1; do
  PBSM_FAST_REPLAY=$f timeout 600 python bench.py --config 2 --no-e2e --no-cpu-baseline --sub-configs none --no-parity --steps 100 > gpurun_out/r03d_f${f}_$i.json 2> gpurun_out/r03d_f${f}_$i.err
  python -c "
import json; d=json.load(open('gpurun_out/r03d_f${f}_$i.json'))
print('rep $i fast=$f cfg2', round(d['ms_per_step'],4), d['clocks'])" || tail -3 gpurun_out/r03d_f${f}_$i.err
done; done 2>&1 | tee gpurun_out/r03d_fast_replay_ab.txt
