# Same-box A/B of ptxas --register-usage-level (v5 kernel SASS: levels 0-4 / 5 (default) / 6-10 give three schedules).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2 3; do for v in base rul0 rul6; do echo "== $v rep $rep"; GATEWAVE_B200_LIB=variants/lib_$v.so timeout 300 python tools/br_time.py 148 256 444; done; done > gpurun_out/r02_rul_ab.txt 2>&1
tail -5 gpurun_out/r02_rul_ab.txt
