#!/bin/bash
# Round 2 A/B 2: what the keeping count's ~9 % over the plain count is (timing-only variants:
# nomask = no mask store, nocnt = no chunk count / superblock atomic, nostore = neither).
mkdir -p gpurun_out/r2d
for cfg in c5 c2; do
  for v in base nomask nocnt nostore; do
    lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v " >> gpurun_out/r2d/count_variants.txt
    env $lib timeout 300 python scripts/count_variants.py $cfg 30 >> gpurun_out/r2d/count_variants.txt 2>&1
  done
done
