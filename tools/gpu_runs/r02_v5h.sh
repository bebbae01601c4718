# final-state check of v5 (RED, no stagger): full GPU suite, bench with CPU baseline, launch list, ncu of the bench kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/v5h_pytest.txt
timeout 900 python bench.py > gpurun_out/v5h_bench.json 2> gpurun_out/v5h_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v5h_launches.csv python bench.py --steps 2 --warmup 1 --no-netlist --no-cpu-baseline > gpurun_out/v5h_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate_v5 -s 3 -c 1 -o gpurun_out/v5h_bench_br -f python bench.py --steps 1 --warmup 3 --no-netlist --no-cpu-baseline > gpurun_out/v5h_ncu_full.log 2>&1
