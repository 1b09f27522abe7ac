for v in "" _h0 _hi _noidx; do
  PBSM_LIB_NAME=libpbsm$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_ncu$v.csv python tools/one_join.py 2 3 units > /dev/null 2>&1; echo "== variant $v rc=$?"
  python tools/ncu_kernels.py gpurun_out/r02e_ncu$v.csv 1 | grep -E "k_ubin|k_ujoin"
done
python tools/one_join.py 2 3 units > gpurun_out/r02e_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ujoin|k_ularge|k_ubin|k_umap_write" -s 6 -c 5 -o gpurun_out/r02e_full python tools/one_join.py 2 3 units > gpurun_out/r02e_full.log 2>&1; echo full rc=$?
tail -3 gpurun_out/r02e_full.log
