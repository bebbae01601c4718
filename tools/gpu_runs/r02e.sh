mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_runtime.py -x -q > gpurun_out/r02e_tests.txt 2>&1
for rep in 1 2; do
for lib in paper_2306_11006_b200/libgatewave_b200.so variants/lib_noxhoist.so; do
  echo "== $lib"; GATEWAVE_B200_LIB=$lib timeout 300 python tools/br_time.py 148 256 444 592
done
echo "== unfused k_lin"; GATEWAVE_BR_UNFUSED=1 timeout 300 python tools/br_time.py 148 256 444 592
done > gpurun_out/r02e_ab.txt 2>&1
