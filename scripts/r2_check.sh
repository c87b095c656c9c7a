#!/bin/bash
# Round-2 re-verification of HEAD on a B200: GPU suite, default bench line, the 75M-row shard step,
# the count kernel's issue-rate counters (fast path and interpreter).
mkdir -p gpurun_out/r2a
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2a/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2a/bench_default.json 2> gpurun_out/r2a/bench_default.err
timeout 300 python bench.py --rows 75000000 --steps 50 --no-e2e --no-cpu --no-read-peak --no-configs --peers1 > gpurun_out/r2a/strong_75M.json 2>gpurun_out/r2a/strong_75M.err
M=smsp__issue_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio
ARGS="--steps 2 --warmup 3 --no-cpu --no-e2e --no-graph --no-read-peak --no-configs"
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:'count_kernel|pushdown_sel_kernel' -c 6 python bench.py $ARGS > gpurun_out/r2a/ncu_issue_fast.csv 2>&1
SEL_FAST=0 timeout 600 ncu --metrics $M --clock-control none --csv -k regex:'count_kernel' -c 3 python bench.py $ARGS > gpurun_out/r2a/ncu_issue_interp.csv 2>&1
ls -la gpurun_out/r2a
