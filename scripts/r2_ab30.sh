#!/bin/bash
# keeping count: mask / code-bit lines written by TMA bulk stores from shared memory (A/B)
mkdir -p gpurun_out/r2p2
SEL_LIB=$PWD/build_exp/libsel_mbulk.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prepared.py -x -q > gpurun_out/r2p2/pytest_mbulk.log 2>&1; echo "rc=$?" >> gpurun_out/r2p2/pytest_mbulk.log
timeout 1500 python scripts/ab_step.py 4 75000000,300000000,600000000 base=- mbulk=$PWD/build_exp/libsel_mbulk.so mbulk2=$PWD/build_exp/libsel_mbulk2.so > gpurun_out/r2p2/ab_step.jsonl 2>&1
