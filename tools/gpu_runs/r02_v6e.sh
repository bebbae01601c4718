# validation after the wire-store cache: GPU suite, bench, configs 2/3/5 twice (cached store on the second run)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/v6e_pytest.txt
timeout 900 python bench.py > gpurun_out/v6e_bench.json 2> gpurun_out/v6e_bench.err
for c in 2 3 5; do timeout 900 python tools/netlist_run.py --config $c --repeats 2 > gpurun_out/v6e_config$c.json 2> gpurun_out/v6e_config$c.err; done
