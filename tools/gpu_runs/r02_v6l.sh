cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_netlists.py -q -k "config2" 2>&1 | tail -2 > gpurun_out/v6l_pytest.txt
timeout 1200 python bench.py > gpurun_out/v6l_bench.json 2> gpurun_out/v6l_bench.err
