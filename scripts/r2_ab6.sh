#!/bin/bash
# split library: GPU suite; the mask-store form A/B on the current build; sel_pushdown path crossover
mkdir -p gpurun_out/r2h
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2h/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2h/pytest_gpu.log
for cfg in c4 c2 c5; do
  for v in base plainst noclob; do
    lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v " >> gpurun_out/r2h/count_variants.txt
    env $lib timeout 300 python scripts/count_variants.py $cfg 30 >> gpurun_out/r2h/count_variants.txt 2>&1
  done
done
timeout 900 python scripts/pushdown_paths.py > gpurun_out/r2h/pushdown_paths.jsonl 2>&1
