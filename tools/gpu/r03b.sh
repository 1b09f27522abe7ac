python tools/timeline.py 2 > gpurun_out/r03b_timeline_cfg2.jsonl 2> gpurun_out/r03b_timeline_cfg2.err; tail -25 gpurun_out/r03b_timeline_cfg2.jsonl; tail -3 gpurun_out/r03b_timeline_cfg2.err
python tools/timeline.py 2 895 1344 > gpurun_out/r03b_timeline_cfg2_strip.jsonl 2> gpurun_out/r03b_timeline_cfg2_strip.err; tail -25 gpurun_out/r03b_timeline_cfg2_strip.jsonl
python tools/plan_stats.py 2 3 5 > gpurun_out/r03b_plan_stats.txt 2>&1; cat gpurun_out/r03b_plan_stats.txt
