timeout 900 python tools/strip_emulation.py --config 2 --ns 1 2 4 8 > gpurun_out/r02ze_strips_cfg2.jsonl 2>&1; echo rc=$?
timeout 1200 python tools/strip_emulation.py --config 3 --ns 1 8 > gpurun_out/r02ze_strips_cfg3.jsonl 2>&1; echo rc=$?
python tools/fixed_cost.py 1000 graph > gpurun_out/r02ze_fixed_graph.jsonl 2>&1
python -c "
import json
for f in ('gpurun_out/r02ze_strips_cfg2.jsonl','gpurun_out/r02ze_strips_cfg3.jsonl'):
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l); print(d['config'], d['n'], d['projected_ms'], round(d['mean_ms'],4))
"
grep '^{' gpurun_out/r02ze_fixed_graph.jsonl | cut -c1-120
