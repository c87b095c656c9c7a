#!/bin/bash
# 1-chunk push-down blocks at every size (C2 shapes) vs 4 from 150M rows; C5 / C3 (sparse) likewise
mkdir -p gpurun_out/r2w
timeout 1500 python scripts/ab_step.py 3 150000000,300000000,600000000 cur=- bc1all=$PWD/build_exp/libsel_bc1all.so > gpurun_out/r2w/ab_step.jsonl 2>&1
for v in cur bc1all; do
  lib=""; [ "$v" != cur ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
  for c in c3 c5 c4; do
    echo -n "$v $c " >> gpurun_out/r2w/configs.txt
    env $lib timeout 400 python bench.py --config $c --steps 30 --no-e2e --no-cpu --no-read-peak --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['latency_ms']['pushdown_kernels'], d['latency_ms']['count_kernel'])" >> gpurun_out/r2w/configs.txt
  done
done
