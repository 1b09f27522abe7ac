python -c "from paper_1908_11740_b200 import _build; _build.build_library()" 
timeout 900 python -m pytest tests/test_gpu_units.py -x -q > gpurun_out/r02b_units.log 2>&1; echo units rc=$?
tail -30 gpurun_out/r02b_units.log
timeout 600 python tools/unit_probe.py 2,5,3,4 10 > gpurun_out/r02b_probe.jsonl 2>&1; echo probe rc=$?
cat gpurun_out/r02b_probe.jsonl | cut -c1-3000
