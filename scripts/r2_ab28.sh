#!/bin/bash
# batch count variants: next-chunk L2 prefetch (with / without the later-columns prefetch), 4 CTAs/SM
mkdir -p gpurun_out/${OUT:-r2m}
for r in 1 2 3; do
  for v in ${VARIANTS:-cur pfn b4}; do
    lib=""; [ "$v" != cur ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v " >> gpurun_out/${OUT:-r2m}/batch_ab.txt
    env $lib timeout 300 python scripts/batch_bench.py 2>&1 | tail -1 | cut -c1-60 >> gpurun_out/${OUT:-r2m}/batch_ab.txt
  done
done
