#!/bin/bash
# batch count: L2 prefetch of the chunk's other columns (bpf) vs none; then the default bench line
mkdir -p gpurun_out/r2t
for v in base bpf base bpf; do
  lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
  echo -n "$v " >> gpurun_out/r2t/batch.txt
  env $lib timeout 300 python scripts/batch_bench.py >> gpurun_out/r2t/batch.txt 2>&1
done
bash scripts/r2_final_check.sh
