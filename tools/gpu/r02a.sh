set -x
python -c "import torch;print(torch.cuda.get_device_name())"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02a_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r02a_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo bench rc=$?
tail -3 gpurun_out/r02a_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02a_ref.json 2>&1; echo ref rc=$?
