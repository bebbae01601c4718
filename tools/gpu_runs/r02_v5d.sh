# full GPU suite + bench + ncu of the GC=1 and GC=2 v5 kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/v5d_pytest.txt
timeout 600 python bench.py > gpurun_out/v5d_bench.json 2> gpurun_out/v5d_bench.err
for g in 148 256; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate_v5 -s 1 -c 1 -o gpurun_out/v5d_br$g -f python tools/br_once.py $g > gpurun_out/v5d_ncu$g.log 2>&1
done
