cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_keyswitch_tc -s 1 -c 1 -o gpurun_out/ks_cold python tools/ks_once.py > gpurun_out/ks_ncu.log 2>&1
ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_keyswitch_tc -s 1 -c 1 -o gpurun_out/ks_warm python tools/ks_once.py >> gpurun_out/ks_ncu.log 2>&1
tail -3 gpurun_out/ks_ncu.log
