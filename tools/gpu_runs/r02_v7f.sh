cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in n0 s01 s02 s04 s08 s10 s20; do echo "== $v"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 148 444; done; done
