mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/r02b_pytest_gpu.txt 2>&1
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/r02b_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02b_ref.json 2> gpurun_out/r02b_ref.err
