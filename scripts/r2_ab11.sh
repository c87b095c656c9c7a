#!/bin/bash
# push-down with one flush site (5x smaller kernel, 40-52 B spills) vs the unrolled block loop
mkdir -p gpurun_out/r2o
timeout 1500 python scripts/ab_step.py 4 75000000,600000000 prev=$PWD/build_exp/libsel_prev.so one=- > gpurun_out/r2o/ab_step.jsonl 2>&1
for cfg in c3 c5 c6 c4; do
  for v in base prev base prev; do
    lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v " >> gpurun_out/r2o/count_variants.txt
    env $lib timeout 300 python scripts/count_variants.py $cfg 30 >> gpurun_out/r2o/count_variants.txt 2>&1
  done
done
