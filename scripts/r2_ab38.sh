#!/bin/bash
# cross-stream ordering after an async Execute: GPU suite + step check
mkdir -p gpurun_out/r2y
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2y/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2y/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu --no-configs > gpurun_out/r2y/bench.json 2> gpurun_out/r2y/bench.err
timeout 300 python bench.py --rows 75000000 --steps 50 --no-e2e --no-cpu --no-read-peak --no-configs --peers1 > gpurun_out/r2y/strong_75M.json 2>gpurun_out/r2y/strong_75M.err
