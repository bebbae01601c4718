# validation of the cleaned v5 (paired inverse at every GC): GPU suite, bench, launch list, ncu, GC sweep, N=2 flow on one GPU
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/v5l_pytest.txt
timeout 900 python bench.py > gpurun_out/v5l_bench.json 2> gpurun_out/v5l_bench.err
timeout 300 python tools/br_time.py 1 64 148 256 296 444 592 1776 > gpurun_out/v5l_gcsweep.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v5l_launches.csv python bench.py --steps 2 --warmup 1 --no-netlist --no-cpu-baseline > gpurun_out/v5l_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate_v5 -s 3 -c 1 -o gpurun_out/v5l_bench_br -f python bench.py --steps 1 --warmup 3 --no-netlist --no-cpu-baseline > gpurun_out/v5l_ncu_full.log 2>&1
timeout 900 python bench.py --gpus 2 --backend gloo --same-device --sharded config3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v5l_bench2.json 2> gpurun_out/v5l_bench2.err
