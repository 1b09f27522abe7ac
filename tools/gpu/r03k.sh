timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r03k_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r03k_pytest.log
