# A/B: loader back-off (no stagger); bench with config-2 wall runs; ncu of GC=2 (no stagger)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in base sl100 sl400 sl1000; do echo "== $v"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 148 256 444; done; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/v5f_bench.json 2> gpurun_out/v5f_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate_v5 -s 1 -c 1 -o gpurun_out/v5f_br256 -f python tools/br_once.py 256 > gpurun_out/v5f_ncu256.log 2>&1
