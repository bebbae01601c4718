# the reference's own 142-test suite through seams 1/2/3 with v5 as the default kernel; bench; phase profile
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{ for seam in 1 2; do echo "## seam $seam"; timeout 900 bash tools/ref_suite/run.sh run $seam 2>&1 | tail -8; done
  echo "## seam 3 (CLI)"; timeout 600 bash tools/ref_suite/run.sh run 3 -k cli 2>&1 | tail -5; } > gpurun_out/v5n_refsuite.txt
timeout 900 python bench.py > gpurun_out/v5n_bench.json 2> gpurun_out/v5n_bench.err
for g in 148 256 444; do timeout 300 python tools/phase_profile.py $g; done > gpurun_out/v5n_phases.txt 2>&1
