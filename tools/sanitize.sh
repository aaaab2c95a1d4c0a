#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_small.py, and the
# reference's unit suite against the drop-in headers -> gpurun_out/sanitize_*.log
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_small.py \
    > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_${tool}.log
done
timeout 600 tests/_bin/msc3d_ref_unit_tests > gpurun_out/ref_unit_suite.log 2>&1
echo "exit $?" >> gpurun_out/ref_unit_suite.log
