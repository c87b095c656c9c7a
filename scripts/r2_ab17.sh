#!/bin/bash
# compacted code bits (wc): parity of every coded path on the compact build, then step A/B
mkdir -p gpurun_out/r2x
SEL_LIB=$PWD/build_exp/libsel_wc.so timeout 1500 python -m pytest tests -m gpu -x -q -k "coded or fastpath or parity or prepared or fullsize or epochs or peers" > gpurun_out/r2x/pytest_wc.log 2>&1; echo "rc=$?" >> gpurun_out/r2x/pytest_wc.log
timeout 1500 python scripts/ab_step.py 4 75000000,300000000,600000000 base=- wc=$PWD/build_exp/libsel_wc.so > gpurun_out/r2x/ab_step.jsonl 2>&1
for v in base wc; do
  lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
  echo -n "$v " >> gpurun_out/r2x/count_variants.txt
  env $lib timeout 300 python scripts/count_variants.py c2 30 >> gpurun_out/r2x/count_variants.txt 2>&1
done
