#!/bin/bash
# two grid-strided chunks per count iteration (pair): keep work overlapped with the next loads
mkdir -p gpurun_out/r2aa
for cfg in c3 c2 c4 c5 c0; do
  for v in base pair base pair; do
    lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v " >> gpurun_out/r2aa/count_variants.txt
    env $lib timeout 300 python scripts/count_variants.py $cfg 30 >> gpurun_out/r2aa/count_variants.txt 2>&1
  done
done
timeout 1500 python scripts/ab_step.py 3 75000000,600000000 base=- pair=$PWD/build_exp/libsel_pair.so > gpurun_out/r2aa/ab_step.jsonl 2>&1
SEL_LIB=$PWD/build_exp/libsel_pair.so timeout 1200 python -m pytest tests -m gpu -x -q -k "fastpath or parity or fullsize" > gpurun_out/r2aa/pytest_pair.log 2>&1; echo "rc=$?" >> gpurun_out/r2aa/pytest_pair.log
