cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2 3; do for w in 0 1; do echo -n "warm=$w "; GATEWAVE_KS_L2WARM=$w timeout 300 python tools/c2_time.py 2>/dev/null | tail -1; done; done
