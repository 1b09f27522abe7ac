PBSM_LIB_NAME=libpbsm_pipe.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extra_truth.py -m gpu -x -q > gpurun_out/r02y_pytest.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/r02y_pytest.log
CFGS="2 5 3 4" bash tools/gpu/variants.sh r02y base pipe
