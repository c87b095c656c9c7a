#!/bin/bash
# L2 bulk prefetch of each warp's next chunk for the keeping count (SEL_PREFETCH=1) vs off (default
# for selection-only keeps): the keep work sits between a chunk's last use and the next loads
mkdir -p gpurun_out/r2y
for cfg in c3 c2 c4 c5 c0; do
  for pf in default 1 default 1; do
    env=""; [ "$pf" != default ] && env="SEL_PREFETCH=$pf"
    echo -n "$pf " >> gpurun_out/r2y/count_variants.txt
    env $env timeout 300 python scripts/count_variants.py $cfg 30 >> gpurun_out/r2y/count_variants.txt 2>&1
  done
done
