tag=${1:-r02}
mkdir -p gpurun_out /tmp/ncu_all
python tools/ncu_workload.py misc2 > gpurun_out/${tag}_misc2_plain.log 2>&1 || { tail -5 gpurun_out/${tag}_misc2_plain.log; exit 1; }
timeout 1500 ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled \
  --kernel-id "::regex:k_group|k_route|k_count|k_scatter|k_join_nested|k_map_ids:3" \
  -o /tmp/ncu_all/${tag}_misc2_all python tools/ncu_workload.py misc2 > gpurun_out/${tag}_misc2_ncu.log 2>&1
echo "misc2 ncu rc=$?"; tail -2 gpurun_out/${tag}_misc2_ncu.log
python tools/summarize_ncu.py --full /tmp/ncu_all/${tag}_misc2_all.ncu-rep \
  --title "$tag misc2: --set full, warm launch of the ε-join / routing-pack / pair-group kernels" > gpurun_out/${tag}_misc2_all.md
ncu -i /tmp/ncu_all/${tag}_misc2_all.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/${tag}_misc2_all_raw.csv.gz
cat gpurun_out/${tag}_misc2_all.md | cut -c1-200
