#!/bin/bash
# batch count: SWAR byte-point leaves and 4-byte point leaves; parity + A/B vs HEAD's library
mkdir -p gpurun_out/r2k
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/r2k/pytest_batch.log 2>&1; echo "rc=$?" >> gpurun_out/r2k/pytest_batch.log
for r in 1 2 3; do
  for v in base new; do
    lib=""; [ "$v" = base ] && lib="SEL_LIB=$PWD/build_exp/libsel_base.so"
    echo -n "$v " >> gpurun_out/r2k/batch_ab.txt
    env $lib timeout 300 python scripts/batch_bench.py 2>&1 | tail -1 >> gpurun_out/r2k/batch_ab.txt
  done
done
