#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel path (run on the GPU box).
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_workload.py 2>&1 | tail -3
  echo "rc=${PIPESTATUS[0]}"
done
