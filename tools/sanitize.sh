#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the
# small profile workload (under gpurun, 1 GPU).
TAG=${1:-r2}
mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 50 --error-exitcode 9 \
    python tools/profile_workload.py small > gpurun_out/sanitize_${t}_$TAG.log 2>&1
  echo "$t rc=$?"
done
