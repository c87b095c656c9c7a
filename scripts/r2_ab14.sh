#!/bin/bash
# feasibility of a fused small-shard Execute: the push-down at 4 CTAs/SM (32 warps, <= 64 regs;
# pd4) and with 16 gathers in flight (pd4g16) vs 8 CTAs/SM; the keep overhead vs table size;
# batch parity with the column prefetch
mkdir -p gpurun_out/r2u
timeout 1500 python scripts/ab_step.py 4 75000000 base=- pd4=$PWD/build_exp/libsel_pd4.so pd4g16=$PWD/build_exp/libsel_pd4g16.so > gpurun_out/r2u/ab_step.jsonl 2>&1
timeout 600 python scripts/keep_cost.py 75000000 150000000 300000000 600000000 > gpurun_out/r2u/keep_cost.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_batch.py -q > gpurun_out/r2u/pytest_batch.log 2>&1; echo rc=$? >> gpurun_out/r2u/pytest_batch.log
