# ncu --set full with source of k_join (cfg2, cfg3)
for c in 2 3; do
CMD="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --sub-configs none --no-parity"
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_join$' -s 4 -c 1 -o gpurun_out/r03h_kjoin_cfg$c -f $CMD > gpurun_out/r03h_ncu_$c.log 2>&1; echo rc=$?; tail -2 gpurun_out/r03h_ncu_$c.log
done
