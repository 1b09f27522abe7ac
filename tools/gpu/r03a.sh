# (record of a reverted experiment: the PBSM_CHAIN / PBSM_CHAIN_PDL switches existed only in that build; see profiles/r03a_join_chain_pdl_ab.txt)
# join chain (one stream, fused R+S count / scatter launches, PDL at every boundary) vs the two-stream graph
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r03a_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r03a_pytest.log
for mode in "0 0" "1 0" "1 1"; do
  set -- $mode
  for c in 2 5 3; do
    PBSM_CHAIN=$1 PBSM_CHAIN_PDL=$2 timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --sub-configs none --steps 20 > gpurun_out/r03a_${1}${2}_$c.json 2> gpurun_out/r03a_${1}${2}_$c.err
    python -c "
import json; d=json.load(open('gpurun_out/r03a_${1}${2}_$c.json'))
print('chain=$1 pdl=$2 cfg$c', round(d['ms_per_step'],4), 'parity', (d.get('parity') or {}).get('match'))" || tail -3 gpurun_out/r03a_${1}${2}_$c.err
  done
  PBSM_CHAIN=$1 PBSM_CHAIN_PDL=$2 python tools/fixed_cost.py 1000 graph 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print('chain=$1 pdl=$2 fixed', d['k'], d['rows'], d['us_per_join'])
    except Exception: print(l.rstrip())"
done 2>&1 | tee gpurun_out/r03a_chain_ab.txt
