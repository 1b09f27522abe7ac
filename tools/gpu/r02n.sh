python tools/fixed_cost.py 1000 2>&1 | tee gpurun_out/r02n_fixed.jsonl
