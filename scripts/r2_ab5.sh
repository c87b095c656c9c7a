#!/bin/bash
# interleaved step A/B (pre-round-2 HEAD vs current) + ncu of the keeping count on C4: base vs nomask
mkdir -p gpurun_out/r2g
timeout 1200 python scripts/ab_step.py 4 75000000,600000000 head=$PWD/build_exp/libsel_head.so cur=- > gpurun_out/r2g/ab_step.jsonl 2>&1
ARGS="--config c4 --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph --no-read-peak --no-configs"
timeout 600 ncu --set full --clock-control none -k regex:count_kernel -s 3 -c 1 -o gpurun_out/r2g/c4_keep_base -f python bench.py $ARGS > gpurun_out/r2g/ncu_base.out 2>&1
SEL_LIB=$PWD/build_exp/libsel_nomask.so timeout 600 ncu --set full --clock-control none -k regex:count_kernel -s 3 -c 1 -o gpurun_out/r2g/c4_keep_nomask -f python bench.py $ARGS > gpurun_out/r2g/ncu_nomask.out 2>&1
