#!/bin/bash
# 1-chunk push-down blocks below 150M rows as the default: GPU suite; A/B against 2 near the threshold
mkdir -p gpurun_out/r2v
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2v/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2v/pytest_gpu.log
timeout 1500 python scripts/ab_step.py 4 75000000,112500000,144000000 bc1=- bc2=$PWD/build_exp/libsel_bc2.so > gpurun_out/r2v/ab_step.jsonl 2>&1
