cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in pf2 pf0; do echo "== $v"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 600 python bench.py --no-netlist --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['ms_per_step'])"; done; done
