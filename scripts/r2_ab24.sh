#!/bin/bash
# async prepared execute: GPU suite; device-side launch list of one Execute at 75M rows (warm L2)
mkdir -p gpurun_out/r2h
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2h/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2h/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2h/launches_75M.csv python scripts/step_breakdown.py 75000000 > gpurun_out/r2h/ncu_75M.log 2>&1
