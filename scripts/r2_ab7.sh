#!/bin/bash
# dynamic count tail: GPU suite, interleaved step A/B vs the grid-strided tail, count variants;
# the mask-store form A/B (plainst / noclob; built from the previous source, store code unchanged)
mkdir -p gpurun_out/r2i
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2i/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2i/pytest_gpu.log
timeout 1200 python scripts/ab_step.py 4 75000000,600000000 nodyn=$PWD/build_exp/libsel_nodyn.so dyn=- > gpurun_out/r2i/ab_step.jsonl 2>&1
for cfg in c4 c2 c5; do
  for v in base nodyn plainst noclob; do
    lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v " >> gpurun_out/r2i/count_variants.txt
    env $lib timeout 300 python scripts/count_variants.py $cfg 30 >> gpurun_out/r2i/count_variants.txt 2>&1
  done
done
