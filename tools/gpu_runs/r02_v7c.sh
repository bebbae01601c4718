cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in k3F k01 k02 k04 k08 k10 k20; do echo -n "$v "; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 256 | tail -1; done; done
