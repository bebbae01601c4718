# v5: phase profile + ncu full captures at 1 / 2 / 3 gates per SM
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for g in 148 256 444; do timeout 300 python tools/phase_profile.py $g; done > gpurun_out/v5b_phases.txt 2>&1
for g in 148 256 444; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate_v5 -s 1 -c 1 -o gpurun_out/v5b_br$g -f python tools/br_once.py $g > gpurun_out/v5b_ncu$g.log 2>&1
done
