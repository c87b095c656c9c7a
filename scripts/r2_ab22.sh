#!/bin/bash
# keeping count's local total from its hyperblock scan (no pass over the per-CTA partials)
mkdir -p gpurun_out/r2ff
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2ff/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2ff/pytest_gpu.log
timeout 1500 python scripts/ab_step.py 4 75000000,600000000 base=$PWD/build_exp/libsel_base.so scantotal=- > gpurun_out/r2ff/ab_step.jsonl 2>&1
