CFGS="4" bash tools/gpu/variants.sh r02v base binpf
for v in base binpf; do echo -n "$v "; PBSM_LIB_NAME=libpbsm_$v.so timeout 300 python tools/bin_probe.py 2; done
