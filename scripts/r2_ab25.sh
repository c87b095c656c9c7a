#!/bin/bash
# sel_ctx_set_option parity; streaming (.cs) output stores of the push-down vs write-back
mkdir -p gpurun_out/r2i
timeout 1200 python -m pytest tests/test_gpu_options.py tests/test_gpu_prepared.py -x -q > gpurun_out/r2i/pytest_options.log 2>&1; echo "rc=$?" >> gpurun_out/r2i/pytest_options.log
timeout 1500 python scripts/ab_step.py 4 75000000,600000000 base=- cs=$PWD/build_exp/libsel_cs.so > gpurun_out/r2i/ab_step.jsonl 2>&1
