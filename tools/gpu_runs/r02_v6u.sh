cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for w in 0 1; do echo -n "warm=$w "; GATEWAVE_KS_L2WARM=$w timeout 300 python tools/c2_time.py 2>/dev/null | tail -1; done; done
for rep in 1 2; do for w in 0 1; do
  GATEWAVE_KS_L2WARM=$w timeout 600 python bench.py --no-cpu-baseline --no-netlist --no-cpu-netlists --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('warm=$w value %.0f e2e %.0f ms/step %.4f br %.4f ks %.4f wide %.0f' % (d['value'], d['e2e']['value'], d['ms_per_step'], r['per_launch_ms'], r['keyswitch_ms_per_launch'], d['throughput_wide_level']['gates_per_s']))"
done; done
