timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02f_pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/r02f_pytest.log
timeout 300 python tools/unit_probe.py 2,3 10 > gpurun_out/r02f_probe.jsonl 2>&1; echo probe rc=$?
python - <<'PY'
import json
for l in open('gpurun_out/r02f_probe.jsonl'):
    d = json.loads(l); t = d['tiles']; print(d['cfg'], t['ms'], t['phases_ms'])
PY
