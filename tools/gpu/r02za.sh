timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r02za_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r02za_pytest.log
CFGS="4" bash tools/gpu/variants.sh r02za base pipe5
python -c "import __graft_entry__ as g; g.smoke()"
