# Round-2 evidence run: reference suite through seams 1-3, config 2/3 netlists (wall vs device),
# ncu launch list + full capture of the bench's dominant kernel (traffic).
mkdir -p gpurun_out
for seam in 1 2; do timeout 1500 tools/ref_suite/run.sh run $seam > gpurun_out/r02f_refsuite$seam.txt 2>&1; done
GW_SEAM=3 PYTHONPATH=baseline/_ref:tools/ref_suite:. timeout 900 python -m pytest baseline/_ref/_tests/test_cli.py -p gw_seam -q -p no:cacheprovider > gpurun_out/r02f_refsuite3_cli.txt 2>&1
timeout 1200 python tools/netlist_run.py --config 2 --vectors 20 > gpurun_out/r02f_config2.json 2> gpurun_out/r02f_config2.err
timeout 1200 python tools/netlist_run.py --config 3 --repeats 2 > gpurun_out/r02f_config3.json 2> gpurun_out/r02f_config3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-netlist > gpurun_out/r02f_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate_v3 -s 3 -c 1 -o gpurun_out/r02f_bench_br -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-netlist > gpurun_out/r02f_ncu.log 2>&1
