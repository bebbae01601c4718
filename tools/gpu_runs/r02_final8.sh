# N = 2 bench flow on one GPU (test-only gloo / same-device flags) after moving the communicator
# teardown before the JSON line: the line must be the last stdout line, digest identical to N = 1.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --same-device --sharded config3 --no-cpu-baseline > gpurun_out/r02n2_stdout.txt 2> gpurun_out/r02n2_stderr.txt
echo "rc=$?"; tail -c 300 gpurun_out/r02n2_stdout.txt; echo; tail -3 gpurun_out/r02n2_stderr.txt
