#!/bin/bash
# one-compare batch leaves + finish fences + load_w1 refactor: GPU suite, batch A/B vs the previous build, step A/B
mkdir -p gpurun_out/r2s2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2s2/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2s2/pytest_gpu.log
for r in 1 2 3; do
  for v in prev cur; do
    lib=""; [ "$v" != cur ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v " >> gpurun_out/r2s2/batch_ab.txt
    env $lib timeout 300 python scripts/batch_bench.py 2>&1 | tail -1 | cut -c1-60 >> gpurun_out/r2s2/batch_ab.txt
  done
done
timeout 1200 python scripts/ab_step.py 3 75000000,600000000 prev=$PWD/build_exp/libsel_prev.so cur=- > gpurun_out/r2s2/ab_step.jsonl 2>&1
