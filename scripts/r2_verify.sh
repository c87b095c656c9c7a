#!/bin/bash
# GPU suite + the measurements a kernel/host change must not regress: overhead probe, default
# bench line (C2), and the 75M-row shard step. Usage: scripts/r2_verify.sh <tag> [pytest args]
TAG=${1:-r2v}; shift || true
mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest tests -m gpu -x -q ${*:-} > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/pytest_gpu.log
tail -3 gpurun_out/$TAG/pytest_gpu.log
timeout 300 python scripts/overhead_probe.py 60000 75000000 600000000 > gpurun_out/$TAG/overhead.jsonl 2>&1
timeout 300 python bench.py --rows 75000000 --steps 50 --no-e2e --no-cpu --no-read-peak --no-configs --peers1 > gpurun_out/$TAG/strong_75M.json 2>gpurun_out/$TAG/strong_75M.err
timeout 600 python bench.py --no-e2e --no-cpu --no-configs > gpurun_out/$TAG/bench_c2.json 2> gpurun_out/$TAG/bench_c2.err
