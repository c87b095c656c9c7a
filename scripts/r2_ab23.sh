#!/bin/bash
# async prepared execute (returns at the count) + the whole-chunk copy forked beside the push-down
mkdir -p gpurun_out/r2g
timeout 900 python -m pytest tests/test_gpu_prepared.py -x -q > gpurun_out/r2g/pytest_prepared.log 2>&1; echo "rc=$?" >> gpurun_out/r2g/pytest_prepared.log
timeout 1200 python scripts/ab_step.py 4 75000000,600000000 base=- fork=$PWD/build_exp/libsel_fork.so > gpurun_out/r2g/ab_step.jsonl 2>&1
timeout 300 python bench.py --rows 75000000 --steps 50 --no-e2e --no-cpu --no-read-peak --no-configs --peers1 > gpurun_out/r2g/strong_75M.json 2>gpurun_out/r2g/strong_75M.err
timeout 600 python bench.py --no-e2e --no-cpu --no-configs > gpurun_out/r2g/bench_c2.json 2> gpurun_out/r2g/bench_c2.err
timeout 600 python bench.py --no-e2e --no-cpu --no-configs --blocking > gpurun_out/r2g/bench_c2_blocking.json 2> gpurun_out/r2g/bench_c2_blocking.err
