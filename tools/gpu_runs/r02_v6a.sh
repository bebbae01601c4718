cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/v6a_bench.json 2> gpurun_out/v6a_bench.err
