cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate_v5 -s 1 -c 1 -o gpurun_out/v6b_br148 -f python tools/br_once.py 148 > gpurun_out/v6b_ncu148.log 2>&1
timeout 300 python tools/phase_profile.py 148 > gpurun_out/v6b_phases.txt 2>&1
