# v5w (eight warps, one gate per SM): parity, A/B against four-warp v5 at one gate per SM, config 2 latency
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_v5.py tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_margin.py -x -q 2>&1 | tail -3
for rep in 1 2; do for w in 1 0; do echo "== v5w=$w"; GATEWAVE_BR_V5W=$w timeout 300 python tools/br_time.py 1 64 148; done; done
GATEWAVE_BR_PROFILE=1 timeout 300 python tools/phase_profile.py 148
for w in 1 0; do echo "== v5w=$w"; GATEWAVE_BR_V5W=$w timeout 300 python tools/eval_breakdown.py 2>&1 | tail -2; done
