# Bench prebuilt library variants (_lib/libpbsm_NAME.so) on several configs:
# ms/step, phases and the parity gate.  usage: CFGS="2 3 5" bash tools/gpu/variants.sh TAG NAME...
tag=$1; shift
mkdir -p gpurun_out
for c in ${CFGS:-2 3 5}; do
  for name in "$@"; do
    PBSM_LIB_NAME=libpbsm_$name.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline \
      --sub-configs "" --steps ${STEPS:-10} > gpurun_out/${tag}_${name}_$c.json 2> gpurun_out/${tag}_${name}_$c.err
    python -c "
import json; d=json.load(open('gpurun_out/${tag}_${name}_$c.json'))
print('cfg$c ${name}', round(d['ms_per_step'],4), 'parity', (d.get('parity') or {}).get('match'), {k: round(v,3) for k,v in d['phases_ms'].items()})" || tail -3 gpurun_out/${tag}_${name}_$c.err
  done
done 2>&1 | tee gpurun_out/${tag}_variants.txt
