# A/B: stagger, split inverse at GC 2/3, loader back-off; evaluate() host breakdown
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in base nost nost_i4 sl100 sl400; do echo "== $v"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 148 256 444; done; done
timeout 300 python tools/eval_breakdown.py
