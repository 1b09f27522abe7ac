# GPU-box side of an end-of-iteration check (run under gpurun from the repo root).
# usage: bash tools/round_cmd.sh TAG
set -x
tag=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${tag}_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
python bench.py > gpurun_out/${tag}_bench_main.json 2> gpurun_out/${tag}_bench_main.err; cat gpurun_out/${tag}_bench_main.json
python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; cat gpurun_out/${tag}_bench_ref.json
bash tools/profile_round.sh ${tag} 2
