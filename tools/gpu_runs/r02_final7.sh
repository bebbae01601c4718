# GPU suite + smoke after gw_wires_attach started rejecting non-device / foreign-GPU pointers.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( time timeout 1800 python -m pytest tests -m gpu -q ) > gpurun_out/r02z_pytest_gpu.txt 2>&1
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > gpurun_out/r02z_smoke.txt 2>&1
tail -1 gpurun_out/r02z_pytest_gpu.txt; tail -1 gpurun_out/r02z_smoke.txt
