cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in pf2 pf0 pf1 pf4; do echo "== $v"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 148 256 444; done; done
