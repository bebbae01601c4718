# validation of MSPLIT: GPU suite, smoke, bench, GC sweep, config 2-5 netlists
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/v6d_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v6d_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/v6d_bench.json 2> gpurun_out/v6d_bench.err
timeout 300 python tools/br_time.py 1 64 148 256 296 444 1776 > gpurun_out/v6d_gcsweep.txt 2>&1
for c in 2 3 5 4; do timeout 1500 python tools/netlist_run.py --config $c --repeats 1 > gpurun_out/v6d_config$c.json 2> gpurun_out/v6d_config$c.err; done
