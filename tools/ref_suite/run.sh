#!/bin/bash
# Run the reference's own test-suite through this engine (tools/ref_suite/gw_seam.py).
#   here:        tools/ref_suite/run.sh stage     (copies the suite next to the reference
#                install in baseline/_ref, git-ignored like it; nothing enters the repo)
#   on the GPU:  tools/ref_suite/run.sh run [SEAM] [pytest args...]
set -e
cd "$(dirname "$0")/../.."
case "$1" in
stage) rm -rf baseline/_ref/_tests && cp -r /root/reference/pkg/tests baseline/_ref/_tests && ls baseline/_ref/_tests ;;
run) seam=${2:-1}; shift; shift || true
     GW_SEAM=$seam PYTHONPATH=baseline/_ref:tools/ref_suite:. python -m pytest baseline/_ref/_tests -p gw_seam -q -p no:cacheprovider "$@" ;;
esac
