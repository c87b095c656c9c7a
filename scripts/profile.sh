#!/bin/bash
# Run on the GPU box (via gpurun): launch list + one full ncu capture of each probe kernel.
# Usage: scripts/profile.sh <tag> [bench args...]
set -u
TAG=${1:-r1}; shift || true
# --no-graph: ncu does not attribute kernels replayed inside the prepared CUDA graph; the kernels
# and their launch configuration are the same.
ARGS=${*:-"--steps 3 --warmup 3 --no-cpu --no-e2e --no-graph"}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:'count_kernel|pushdown|selection_result|dense_chunks|peer_exchange' \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py $ARGS > gpurun_out/launches_${TAG}.out 2>&1
for K in count_kernel pushdown_sel_kernel dense_chunks_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:${K} -s 3 -c 1 \
      -o gpurun_out/prof_${TAG}_${K} -f python bench.py $ARGS > gpurun_out/prof_${TAG}_${K}.out 2>&1
done
# the count kernel through the interpreter instead of the fast path (fast path vs interpreter)
SEL_FAST=0 ncu --set full --clock-control none --import-source on -k regex:count_kernel -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_count_interp -f python bench.py $ARGS > gpurun_out/prof_${TAG}_count_interp.out 2>&1
SEL_PUSHDOWN_PATH=single ncu --set full --clock-control none --import-source on -k regex:'pushdown_kernel' -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_pushdown_kernel -f python bench.py $ARGS > gpurun_out/prof_${TAG}_pushdown_kernel.out 2>&1
ls -la gpurun_out | grep $TAG
