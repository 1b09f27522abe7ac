timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "graph or speculative or strategy" > gpurun_out/r02o_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r02o_pytest.log
python tools/fixed_cost.py 1000 eager 2>&1 | tee gpurun_out/r02o_fixed_eager.jsonl
python tools/fixed_cost.py 1000 graph 2>&1 | tee gpurun_out/r02o_fixed_graph.jsonl
python bench.py --no-e2e --no-cpu-baseline --sub-configs 5,3,4 > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/r02o_bench.json')); print('cfg2', d['ms_per_step'], d['parity']['match'], d['phases_ms'])
for c,v in d['sub_configs'].items(): print(c, v['ms_per_step'], v.get('parity',{}).get('match'))"
