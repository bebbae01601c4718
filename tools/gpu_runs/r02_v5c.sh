# v5 split inverse (I4): parity + same-box A/B against the two-warp inverse
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_v5.py tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_margin.py -x -q -s 2>&1 | grep -v "^$" | tail -22
for rep in 1 2; do for v in i4on i4off; do echo "== $v"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 148 256 444; done; done
timeout 300 python tools/phase_profile.py 148
