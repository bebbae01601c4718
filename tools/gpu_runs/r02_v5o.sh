cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v5o_smoke.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/v5o_bench.json 2> gpurun_out/v5o_bench.err
