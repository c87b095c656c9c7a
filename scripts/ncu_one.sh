#!/bin/bash
# One full ncu capture of a kernel: scripts/ncu_one.sh <tag> <kernel-regex> [bench args]
TAG=$1; K=$2; shift 2
ARGS=${*:-"--steps 2 --warmup 3 --no-cpu --no-e2e"}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:${K} -s 3 -c 1 \
    -o gpurun_out/prof_${TAG} -f python bench.py $ARGS > gpurun_out/prof_${TAG}.out 2>&1
tail -3 gpurun_out/prof_${TAG}.out
