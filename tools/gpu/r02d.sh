timeout 900 python -m pytest tests/test_gpu_units.py -x -q > gpurun_out/r02d_units.log 2>&1; echo units rc=$?
tail -3 gpurun_out/r02d_units.log
timeout 300 python tools/unit_probe.py 2,5 10 > gpurun_out/r02d_probe.jsonl 2>&1; echo probe rc=$?
cut -c1-700 gpurun_out/r02d_probe.jsonl
for v in "" _m1 _noidx _m1noidx; do
  PBSM_LIB_NAME=libpbsm$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d_ncu$v.csv python tools/one_join.py 2 4 units > /dev/null 2>&1; echo "== variant $v rc=$?"
  python tools/ncu_kernels.py gpurun_out/r02d_ncu$v.csv 1
done
