#!/bin/bash
# fraction of the selection's stores given evict_last (0.5 / 0.75 vs 1.0); bench line of the final build
mkdir -p gpurun_out/r2t
timeout 1500 python scripts/ab_step.py 3 75000000,300000000,600000000 base=- f05=$PWD/build_exp/libsel_f05.so f075=$PWD/build_exp/libsel_f075.so > gpurun_out/r2t/ab_step.jsonl 2>&1
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/r2t/bench.json 2> gpurun_out/r2t/bench.err
