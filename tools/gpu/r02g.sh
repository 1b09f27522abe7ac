timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "large or strategy or synthetic or instances or configs" > gpurun_out/r02g_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r02g_pytest.log
timeout 300 python tools/unit_probe.py 2,3 10 > gpurun_out/r02g_probe.jsonl 2>&1; echo probe rc=$?
python - <<'PY'
import json
for l in open('gpurun_out/r02g_probe.jsonl'):
    d = json.loads(l); t = d['tiles']; print(d['cfg'], t['ms'], t['phases_ms'])
PY
python tools/one_join.py 3 3 tiles > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g_ncu3.csv python tools/one_join.py 3 3 tiles > /dev/null 2>&1; python tools/ncu_kernels.py gpurun_out/r02g_ncu3.csv 1
