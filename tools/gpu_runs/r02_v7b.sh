cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in m0 m1 m2 m3; do echo "== $v"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 148 256 444; done; done
