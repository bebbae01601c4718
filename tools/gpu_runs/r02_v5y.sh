# validation after the barrier / ordering changes: GPU suite, smoke, bench, GC sweep, configs 2 and 3
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/v5y_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v5y_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/v5y_bench.json 2> gpurun_out/v5y_bench.err
timeout 300 python tools/br_time.py 1 64 148 256 296 444 1776 > gpurun_out/v5y_gcsweep.txt 2>&1
for c in 2 3; do timeout 900 python tools/netlist_run.py --config $c --repeats 1 > gpurun_out/v5y_config$c.json 2> gpurun_out/v5y_config$c.err; done
