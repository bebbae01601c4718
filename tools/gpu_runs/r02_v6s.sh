cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
GATEWAVE_B200_LIB=variants/lib_st2.so timeout 1200 python -m pytest tests/test_gpu_keyswitch.py tests/test_gpu_large_batch.py -x -q 2>&1 | tail -2
for rep in 1 2 3; do for v in st4 st2; do
  GATEWAVE_KS_MT2=0 GATEWAVE_B200_LIB=variants/lib_$v.so timeout 600 python bench.py --no-cpu-baseline --no-netlist --no-cpu-netlists --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$v value %.0f e2e %.0f ms/step %.4f br %.4f ks %.4f' % (d['value'], d['e2e']['value'], d['ms_per_step'], r['per_launch_ms'], r['keyswitch_ms_per_launch']))"
done; done
