# The reference's own test-suite through seams 1, 2 and 3 on the final build (stage it first here:
# tools/ref_suite/run.sh stage).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for seam in 1 2 3; do echo "## seam $seam"; ( time timeout 1500 tools/ref_suite/run.sh run $seam ) 2>&1 | tail -8; done > gpurun_out/r02_refsuite_final9.txt 2>&1
grep -E "passed|failed" gpurun_out/r02_refsuite_final9.txt
