for g in 1 2 4 32; do echo -n "pg$g "; PBSM_LIB_NAME=libpbsm_pg$g.so timeout 300 python tools/bin_probe.py 2; done 2>&1 | tee gpurun_out/r02q_bin.txt
