# Round-2 validation on one B200 after the conversion / L2 warm-up / host-path changes.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( time timeout 1800 python -m pytest tests -m gpu -q ) > gpurun_out/r02y_pytest_gpu.txt 2>&1
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > gpurun_out/r02y_smoke.txt 2>&1
( time timeout 900 python bench.py > gpurun_out/r02y_bench.json ) 2> gpurun_out/r02y_bench.err
timeout 300 python tools/e2e_breakdown.py > gpurun_out/r02y_e2e_breakdown.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02y_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-netlist --no-cpu-netlists > /dev/null 2>&1
tail -1 gpurun_out/r02y_pytest_gpu.txt; cat gpurun_out/r02y_smoke.txt | tail -1
