cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
GATEWAVE_B200_LIB=variants/lib_pb3.so timeout 600 python -m pytest tests/test_gpu_v5.py tests/test_gpu_parity.py -q -x 2>&1 | grep -E "FAIL|Error|assert|^E " | head -30
