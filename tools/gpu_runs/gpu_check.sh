#!/bin/bash
# One gpurun call: build check, GPU tests, bench (both arms), ncu launch list + full capture.
# usage: tools/gpu_runs/gpu_check.sh TAG [tests|bench|ncu ...]
set -x
TAG=${1:-run}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
for what in "$@"; do
case $what in
tests) timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1 ;;
smoke) timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/${TAG}_smoke.txt 2>&1 ;;
bench) timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err ;;
benchq) timeout 600 python bench.py --no-cpu-baseline --no-netlist > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err ;;
ref) timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err ;;
launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-netlist > gpurun_out/${TAG}_launches.log 2>&1 ;;
ncu) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate -s 1 -c 1 -o gpurun_out/${TAG}_br -f python tools/br_once.py 256 > gpurun_out/${TAG}_ncu.log 2>&1 ;;
ncu4) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate -s 1 -c 1 -o gpurun_out/${TAG}_br592 -f python tools/br_once.py 592; timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate -s 1 -c 1 -o gpurun_out/${TAG}_br444 -f python tools/br_once.py 444 > gpurun_out/${TAG}_ncu4.log 2>&1 ;;
ncuks) timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_keyswitch_tc -s 1 -c 1 -o gpurun_out/${TAG}_ks -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-netlist > gpurun_out/${TAG}_ncuks.log 2>&1 ;;
phase) for g in 128 256 296 592; do timeout 300 python tools/phase_profile.py $g; done > gpurun_out/${TAG}_phase.txt 2>&1 ;;
phase2) for g in 256 592; do GATEWAVE_BR_KERNEL=v2 timeout 300 python tools/phase_profile.py $g; done > gpurun_out/${TAG}_phase2.txt 2>&1 ;;
brtime) timeout 300 python tools/br_time.py > gpurun_out/${TAG}_brtime.txt 2>&1 ;;
gcq) for gc in 1 2 4; do echo "GC=$gc"; GATEWAVE_BR_GC=$gc timeout 300 python tools/br_time.py 148 256 592 2368; done > gpurun_out/${TAG}_gcq.txt 2>&1 ;;
ab) for v in $(ls variants/*.so); do for gc in ${ABGC:-2 4}; do echo "$v GC=$gc"; GATEWAVE_B200_LIB=$v GATEWAVE_BR_GC=$gc timeout 300 python tools/br_time.py 256 2368; done; done > gpurun_out/${TAG}_ab.txt 2>&1 ;;
refsuite) for seam in 1 2; do timeout 1500 tools/ref_suite/run.sh run $seam > gpurun_out/${TAG}_refsuite$seam.txt 2>&1; done ;;  # stage first: tools/ref_suite/run.sh stage
gcsweep) for gc in 1 2 3 4; do echo "GC=$gc"; GATEWAVE_BR_GC=$gc timeout 300 python tools/br_time.py 148 256 444 592 1184 2368; done > gpurun_out/${TAG}_gcsweep.txt 2>&1 ;;
esac
done
ls -la gpurun_out
