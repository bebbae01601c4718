mkdir -p gpurun_out
# N > 1 bench flow on one GPU: 2 ranks, gloo, both on GPU 0, config 3 sharded with the host-staged exchange
timeout 1200 python bench.py --gpus 2 --backend gloo --same-device --sharded config3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_bench2.json 2> gpurun_out/r02i_bench2.err
# single-GPU digest of config 3 for comparison (sharded flag at N = 1 runs it locally)
timeout 1200 python bench.py --sharded config3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_bench1.json 2> gpurun_out/r02i_bench1.err
