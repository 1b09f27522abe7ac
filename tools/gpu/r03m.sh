# self-join partitioned once: GPU tests + cfg5 A/B + strips
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r03m_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r03m_pytest.log
for f in 0 1; do
  PBSM_SELF_ONCE=$f timeout 600 python bench.py --config 5 --no-e2e --no-cpu-baseline --sub-configs none --steps 50 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('self_once=$f cfg5 bench', round(d['ms_per_step'],4), d['parity']['match'], {k: round(v,3) for k,v in d['phases_ms'].items()}, round(d['step_roofline']['frac'],3))"
done 2>&1 | tee gpurun_out/r03m_self_once_ab.txt
python bench.py --config 2 --no-e2e --no-cpu-baseline --sub-configs none --steps 50 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('cfg2 bench', round(d['ms_per_step'],4), d['parity']['match'])"
