set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; cat gpurun_out/bench_main.json
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
bash tools/profile_round.sh r01h 2
cp paper_1908_11740_b200/_lib/libpbsm.so gpurun_out/libpbsm_r01h.so
