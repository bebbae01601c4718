# configs 2-5 through runtime.evaluate on one B200 with the final v5 kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 2 3 5 4; do timeout 1500 python tools/netlist_run.py --config $c --repeats 1 > gpurun_out/v5r_config$c.json 2> gpurun_out/v5r_config$c.err; done
