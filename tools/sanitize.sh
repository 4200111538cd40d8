#!/bin/bash
# compute-sanitizer over the smoke run and the small-mesh GPU parity tests
# (SURVEY §5): memcheck, racecheck, synccheck, initcheck.  Logs to gpurun_out/.
#   tools/sanitize.sh [pytest -k expression]
set -u
mkdir -p gpurun_out
K=${1:-"lane or operators or ax_dssum_config1 or deterministic or generic or graph_replay"}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/sanitize_${tool}_smoke.log 2>&1
  echo "$tool smoke rc=$?"
  timeout 2400 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$K" \
    > gpurun_out/sanitize_${tool}_parity.log 2>&1
  echo "$tool parity rc=$?"
done
