# re-entry check of HEAD: GPU tests, smoke, both bench arms
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r02zz_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02zz_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02zz_smoke.log 2>&1; tail -1 gpurun_out/r02zz_smoke.log
python bench.py > gpurun_out/r02zz_bench_main.json 2> gpurun_out/r02zz_bench_main.err; cut -c1-600 gpurun_out/r02zz_bench_main.json
python bench.py --impl reference > gpurun_out/r02zz_bench_ref.json 2> gpurun_out/r02zz_bench_ref.err; cut -c1-600 gpurun_out/r02zz_bench_ref.json
