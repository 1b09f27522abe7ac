timeout 900 python -m pytest tests/test_gpu_units.py -x -q > gpurun_out/r02c_units.log 2>&1; echo units rc=$?
tail -15 gpurun_out/r02c_units.log
timeout 600 python tools/unit_probe.py 2,5 10 > gpurun_out/r02c_probe.jsonl 2>&1; echo probe rc=$?
cat gpurun_out/r02c_probe.jsonl | cut -c1-1500
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch
from paper_1908_11740_b200 import device as dev
from paper_1908_11740_b200.synth import make_config
r, s, k = make_config(2)
R, S = dev.to_device(r), dev.to_device(s)
for _ in range(4):
    res = dev.run_join(R, S, k, k, pipeline="units")
torch.cuda.synchronize()
print(res.count)
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_ncu.csv python /tmp/one.py > gpurun_out/r02c_ncu.log 2>&1; echo ncu rc=$?
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(l for l in open('gpurun_out/r02c_ncu.csv') if l.startswith('"')))
d = collections.defaultdict(list)
for r in rows:
    if r.get('Metric Name') == 'gpu__time_duration.sum':
        d[r['Kernel Name'][:60]].append(float(r['Metric Value']))
for k, v in d.items(): print(f"{k:60s} n={len(v)} last={v[-1]/1e3:.1f}us mean={sum(v)/len(v)/1e3:.1f}us")
PY
