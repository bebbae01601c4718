# where the config-2 wall time goes inside bench.py (evaluate trace)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
GATEWAVE_EVAL_TRACE=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/v5m_bench.json 2> gpurun_out/v5m_bench.err
grep "\[evaluate\]" gpurun_out/v5m_bench.err | tail -12
