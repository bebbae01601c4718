cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
GATEWAVE_B200_LIB=variants/lib_noprof.so timeout 600 python -m pytest tests/test_gpu_v5.py -x -q 2>&1 | tail -1
for rep in 1 2 3; do for v in prof noprof; do echo "== $v"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 148 256 444; done; done
GATEWAVE_B200_LIB=variants/lib_prof.so timeout 300 python tools/phase_profile.py 256 2>&1 | tail -3
