# ncu --set full of (the 3rd, warm) launch of EVERY kernel of each workload;
# summarised ON the box (the reports themselves exceed gpurun's return size).
# usage: bash tools/gpu/ncu_all.sh TAG   → gpurun_out/TAG_{cfg2,cfg4,misc}_all.{md,csv}
tag=${1:-r02}
mkdir -p gpurun_out /tmp/ncu_all
for w in cfg2 cfg4 misc; do
  python tools/ncu_workload.py $w > gpurun_out/${tag}_${w}_plain.log 2>&1 || { echo "$w plain failed"; tail -5 gpurun_out/${tag}_${w}_plain.log; continue; }
  timeout 1500 ncu -f --set full --clock-control none --import-source on --kernel-id ::regex:^.*k_:3 \
    -o /tmp/ncu_all/${tag}_${w}_all python tools/ncu_workload.py $w > gpurun_out/${tag}_${w}_ncu.log 2>&1
  echo "$w ncu rc=$?"; tail -1 gpurun_out/${tag}_${w}_ncu.log
  python tools/summarize_ncu.py --full /tmp/ncu_all/${tag}_${w}_all.ncu-rep \
    --title "$tag $w: --set full, warm launch of every kernel" > gpurun_out/${tag}_${w}_all.md
  ncu -i /tmp/ncu_all/${tag}_${w}_all.ncu-rep --page raw --csv > gpurun_out/${tag}_${w}_all_raw.csv 2>/dev/null
  gzip -f gpurun_out/${tag}_${w}_all_raw.csv
done
ls -la gpurun_out | tail -12
