#!/bin/bash
# small-shard knobs: 1-chunk push-down blocks below 150M rows; count fast path at 4 CTAs/SM
mkdir -p gpurun_out/r2u
timeout 1500 python scripts/ab_step.py 4 37500000,75000000,600000000 base=- bc1=$PWD/build_exp/libsel_bc1.so m4=$PWD/build_exp/libsel_m4.so > gpurun_out/r2u/ab_step.jsonl 2>&1
