# ncu --set full with source: nested join, scatter, count, plan_apply (cfg2)
CMD="python bench.py --config 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --sub-configs none --no-parity"
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_join_nested_pipe$|^k_scatter$|^k_count$|^k_plan_apply$|^k_plan_reduce$' -s 25 -c 7 -o gpurun_out/r03i_cfg2_src -f $CMD > gpurun_out/r03i_ncu.log 2>&1; echo rc=$?; tail -2 gpurun_out/r03i_ncu.log
