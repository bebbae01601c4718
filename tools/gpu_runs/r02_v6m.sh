# the whole GPU suite with exact mode (split-key v3) forced, and the final ncu of the bench kernel with source
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
GATEWAVE_BR_EXACT=1 timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/v6m_pytest_exact.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate_v5 -s 3 -c 1 -o gpurun_out/v6m_bench_br -f python bench.py --steps 1 --warmup 3 --no-netlist --no-cpu-baseline > gpurun_out/v6m_ncu.log 2>&1
