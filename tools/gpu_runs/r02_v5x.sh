cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
GATEWAVE_B200_LIB=variants/lib_pb3.so timeout 900 python -m pytest tests/test_gpu_v5.py tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_margin.py tests/test_gpu_edges.py -q 2>&1 | tail -3
for rep in 1 2; do for v in base pb3; do echo "== $v"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 148 256 300 444; done; done
