#!/bin/bash
bash scripts/r2_verify.sh r2f
for cfg in c5 c2 c4; do
  for v in base nomask; do
    lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v " >> gpurun_out/r2f/count_variants.txt
    env $lib timeout 300 python scripts/count_variants.py $cfg 30 >> gpurun_out/r2f/count_variants.txt 2>&1
  done
done
