#!/bin/bash
# ncu of the 8-GPU shard size (75M rows, 1-chunk push-down blocks): launch list + full captures
bash scripts/profile.sh r2q75 --rows 75000000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-graph --no-configs --no-read-peak
python scripts/summarize_profiles.py r2q75 c2_75M > gpurun_out/r2q75_summary.json 2>&1
mkdir -p gpurun_out/r2q75_profiles
cp -r profiles/r2q75/* gpurun_out/r2q75_profiles/
rm -f gpurun_out/*.ncu-rep
