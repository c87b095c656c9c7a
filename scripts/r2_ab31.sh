#!/bin/bash
# whole-table parity incl. the async bench step; ncu of the final batch count
mkdir -p gpurun_out/r2r
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_options.py -x -q > gpurun_out/r2r/pytest_fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/r2r/pytest_fullsize.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:count_batch -s 2 -c 1 -o gpurun_out/r2r/prof_batch -f python scripts/batch_bench.py > gpurun_out/r2r/prof_batch.out 2>&1
