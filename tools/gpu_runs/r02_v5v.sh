cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
GATEWAVE_B200_LIB=variants/lib_pb3.so timeout 600 python -m pytest tests/test_gpu_v5.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for rep in 1 2; do for v in base pb3; do echo "== $v"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 148 256 444; done; done
