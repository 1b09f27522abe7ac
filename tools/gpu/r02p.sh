timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r02p_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r02p_pytest.log
bash tools/multirank_smoke.sh 2>&1 | tail -8
timeout 900 python tools/strip_emulation.py --config 2 --ns 1 2 4 8 > gpurun_out/r02p_strips_cfg2.jsonl 2>&1; echo strips rc=$?
python -c "
import json
for l in open('gpurun_out/r02p_strips_cfg2.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['projected_ms'], round(d['mean_ms'],4))"
