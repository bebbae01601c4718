# Round-2 final validation on one B200 (after the conversion, L2 warm-up, keyswitch and loader-hint changes).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( time timeout 1800 python -m pytest tests -m gpu -q ) > gpurun_out/r02x_pytest_gpu.txt 2>&1
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > gpurun_out/r02x_smoke.txt 2>&1
( time timeout 900 python bench.py > gpurun_out/r02x_bench.json ) 2> gpurun_out/r02x_bench.err
( time timeout 900 python bench.py --impl reference > gpurun_out/r02x_ref.json ) 2> gpurun_out/r02x_ref.err
timeout 300 python tools/e2e_breakdown.py > gpurun_out/r02x_e2e_breakdown.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02x_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-netlist --no-cpu-netlists > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_blind_rotate_v5 -s 3 -c 1 -o gpurun_out/r02x_bench_br python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-netlist --no-cpu-netlists > /dev/null 2>&1
for c in 3 5; do timeout 900 python tools/netlist_run.py --config $c --repeats 2 > gpurun_out/r02x_netlist_config$c.json 2>/dev/null; done
timeout 1200 python tools/netlist_run.py --config 4 --repeats 1 > gpurun_out/r02x_netlist_config4.json 2>/dev/null
tail -1 gpurun_out/r02x_pytest_gpu.txt; tail -1 gpurun_out/r02x_smoke.txt
