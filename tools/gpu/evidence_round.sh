# Final evidence round at HEAD: GPU tests, smoke, both bench arms, launch list + full captures, all-kernel
# captures, strip emulation, fixed cost, timelines.
tag=r04
bash tools/round_cmd.sh $tag 2>&1 | tail -30
bash tools/gpu/ncu_all.sh $tag 2>&1 | tail -8
bash tools/gpu/ncu_misc2.sh $tag 2>&1 | tail -3
python tools/strip_emulation.py --config 2 > gpurun_out/${tag}_strip_emulation_cfg2.jsonl 2> gpurun_out/${tag}_strip2.err; cut -c1-120 gpurun_out/${tag}_strip_emulation_cfg2.jsonl
python tools/strip_emulation.py --config 3 --ns 1 8 > gpurun_out/${tag}_strip_emulation_cfg3.jsonl 2> gpurun_out/${tag}_strip3.err; cut -c1-120 gpurun_out/${tag}_strip_emulation_cfg3.jsonl
python tools/fixed_cost.py 1000 graph > gpurun_out/${tag}_fixed_cost_graph.jsonl 2>&1; cut -c1-100 gpurun_out/${tag}_fixed_cost_graph.jsonl
for c in 2 3 4 5; do python tools/timeline.py $c > gpurun_out/${tag}_timeline_cfg$c.jsonl 2>/dev/null; tail -1 gpurun_out/${tag}_timeline_cfg$c.jsonl; done
