# Round-2 re-validation on one B200 after the container was re-created (fresh in-tree build).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( time timeout 1800 python -m pytest tests -m gpu -q ) > gpurun_out/r02x_pytest_gpu.txt 2>&1
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > gpurun_out/r02x_smoke.txt 2>&1
( time timeout 900 python bench.py > gpurun_out/r02x_bench.json ) 2> gpurun_out/r02x_bench.err
( time timeout 900 python bench.py --impl reference > gpurun_out/r02x_ref.json ) 2> gpurun_out/r02x_ref.err
tail -1 gpurun_out/r02x_pytest_gpu.txt; tail -1 gpurun_out/r02x_smoke.txt
