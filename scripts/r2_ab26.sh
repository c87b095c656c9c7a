#!/bin/bash
# count-in-step decomposition at 75M and 600M rows; ncu of the batch count
mkdir -p gpurun_out/r2j
for n in 75000000 600000000; do timeout 300 python scripts/count_in_step.py $n >> gpurun_out/r2j/count_in_step.jsonl 2>>gpurun_out/r2j/count_in_step.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:count_batch -s 2 -c 1 -o gpurun_out/r2j/prof_batch -f python scripts/batch_bench.py > gpurun_out/r2j/prof_batch.out 2>&1
