#!/bin/bash
# batch count at 4 CTAs/SM: parity + timing; sanitizers over every path (incl. the async Execute)
mkdir -p gpurun_out/r2o
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_prepared.py tests/test_gpu_options.py -x -q > gpurun_out/r2o/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2o/pytest.log
for r in 1 2; do timeout 300 python scripts/batch_bench.py 2>&1 | tail -1 >> gpurun_out/r2o/batch.txt; done
bash scripts/sanitize.sh > gpurun_out/r2o/sanitizer.txt 2>&1
