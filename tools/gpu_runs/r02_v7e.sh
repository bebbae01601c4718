cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_v5.py tests/test_gpu_parity.py tests/test_gpu_margin.py tests/test_gpu_netlists.py tests/test_gpu_runtime.py tests/test_gpu_api.py -x -q 2>&1 | tail -1
for rep in 1 2; do timeout 300 python tools/br_time.py 148 256 444; done
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --no-cpu-netlists --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; a=d['app_latency_config2']
print('value %.0f e2e %.0f ms/step %.4f br %.4f ks %.4f wide %.0f c2 %.1f ms' % (d['value'], d['e2e']['value'], d['ms_per_step'], r['per_launch_ms'], r['keyswitch_ms_per_launch'], d['throughput_wide_level']['gates_per_s'], 1e3*a['combined_netlist']['app_latency_s']))"
done
