cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_v5.py tests/test_gpu_parity.py tests/test_gpu_margin.py -x -q 2>&1 | tail -1
for rep in 1 2; do timeout 300 python tools/br_time.py 148 256 444; done
for rep in 1 2; do timeout 300 python tools/c2_time.py 2>/dev/null | tail -1; done
