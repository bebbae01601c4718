# Bench line with the roofline on SURVEY §8(d)'s W_alg, reference arm, launch list of the same command.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( time timeout 900 python bench.py > gpurun_out/r02y_bench.json ) 2> gpurun_out/r02y_bench.err
( time timeout 900 python bench.py --impl reference > gpurun_out/r02y_ref.json ) 2> gpurun_out/r02y_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02y_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-netlist --no-cpu-netlists > /dev/null 2>&1
tail -c 400 gpurun_out/r02y_bench.json
