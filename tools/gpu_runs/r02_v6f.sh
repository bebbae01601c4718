# final-kernel ncu captures at 1 / 2 / 3 gates per SM + phase cycles + bench launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for g in 148 256 444; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate_v5 -s 1 -c 1 -o gpurun_out/v6f_br$g -f python tools/br_once.py $g > gpurun_out/v6f_ncu$g.log 2>&1
done
for g in 148 256 444; do timeout 300 python tools/phase_profile.py $g; done > gpurun_out/v6f_phases.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v6f_launches.csv python bench.py --steps 2 --warmup 1 --no-netlist --no-cpu-baseline > gpurun_out/v6f_ncu_bench.log 2>&1
