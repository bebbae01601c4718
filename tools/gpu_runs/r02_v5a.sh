# v5 (single key image) first GPU check: parity, margin, timing vs v3 (exact mode)
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_margin.py -x -q -s 2>&1 | tail -25
echo "== v5 default"
timeout 300 python tools/br_time.py 148 256 296 444 1776
for gc in 1 2 3; do echo "== v5 GC=$gc"; GATEWAVE_BR_GC=$gc timeout 300 python tools/br_time.py $((148*gc)); done
echo "== v3 exact"
GATEWAVE_BR_EXACT=1 timeout 300 python tools/br_time.py 148 256 444 1776
