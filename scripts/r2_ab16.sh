#!/bin/bash
# consumed selection lines discarded from L2 (no write-back of dead masks) vs demoted to normal
mkdir -p gpurun_out/r2w
timeout 1500 python scripts/ab_step.py 4 300000000,600000000 base=- disc=$PWD/build_exp/libsel_disc.so > gpurun_out/r2w/ab_step.jsonl 2>&1
for v in base disc; do
  lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
  echo "== $v" >> gpurun_out/r2w/c5.txt
  env $lib timeout 300 python bench.py --config c5 --steps 30 --no-e2e --no-cpu --no-read-peak --no-configs >> gpurun_out/r2w/c5.txt 2>/dev/null
done
