#!/bin/bash
# new epoch/hyperblock parity tests; sanitizer over every kernel path; push-down block size 2 vs 4
mkdir -p gpurun_out/r2l
timeout 900 python -m pytest tests/test_gpu_selection_epochs.py -x -q > gpurun_out/r2l/pytest_epochs.log 2>&1; echo "rc=$?" >> gpurun_out/r2l/pytest_epochs.log
bash scripts/sanitize.sh > gpurun_out/r2l/sanitizer.txt 2>&1
timeout 1200 python scripts/ab_step.py 4 75000000,600000000 bc2=$PWD/build_exp/libsel_bc2.so bc4=- > gpurun_out/r2l/ab_step_bc.jsonl 2>&1
