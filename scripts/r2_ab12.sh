#!/bin/bash
# lane-0 fence (vs all-thread fence) and the whole-chunk copy kernel's grid (1 or 2 CTAs per SM vs
# the push-down's 8): the empty launch at 75M / 600M rows, and the dense case (coded_dense.py)
mkdir -p gpurun_out/r2r
timeout 2000 python scripts/ab_step.py 4 75000000,600000000 prev=$PWD/build_exp/libsel_prev.so fence=$PWD/build_exp/libsel_fence.so dg2=$PWD/build_exp/libsel_dg2.so dg1=$PWD/build_exp/libsel_dg1.so adapt=$PWD/build_exp/libsel_adapt.so > gpurun_out/r2r/ab_step.jsonl 2>&1
for v in fence dg2 dg1; do
  echo "== $v" >> gpurun_out/r2r/coded_dense.txt
  SEL_LIB=$PWD/build_exp/libsel_$v.so timeout 600 python scripts/coded_dense.py >> gpurun_out/r2r/coded_dense.txt 2>&1
done
