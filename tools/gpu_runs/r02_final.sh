# Round-2 final validation on one B200: GPU suite, smoke, both bench arms (timed), clocks.
mkdir -p gpurun_out
( time timeout 1800 python -m pytest tests -m gpu -q -s ) > gpurun_out/r02z_pytest_gpu.txt 2>&1
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/r02z_smoke.txt 2>&1
( time timeout 900 python bench.py > gpurun_out/r02z_bench.json ) 2> gpurun_out/r02z_bench.err
( time timeout 900 python bench.py --impl reference > gpurun_out/r02z_ref.json ) 2> gpurun_out/r02z_ref.err
