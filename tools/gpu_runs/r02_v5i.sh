# paired split inverse at GC=1/2: parity through the variant library + same-box A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
GATEWAVE_B200_LIB=variants/lib_pair3.so timeout 600 python -m pytest tests/test_gpu_v5.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for rep in 1 2; do for v in base pair2 pair3; do echo "== $v"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 148 256 444; done; done
