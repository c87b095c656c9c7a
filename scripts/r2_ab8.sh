#!/bin/bash
# mask store as 16-byte warp-major stores of 4 chunks (v4, timing only) vs the per-chunk store / none
mkdir -p gpurun_out/r2j
for cfg in c4 c5 c2; do
  for v in base nomask v4 base; do
    lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v " >> gpurun_out/r2j/count_variants.txt
    env $lib timeout 300 python scripts/count_variants.py $cfg 30 >> gpurun_out/r2j/count_variants.txt 2>&1
  done
done
