#!/bin/bash
# final build: round measurement set + launch list of the default bench (library kernels)
bash scripts/round_measure.sh
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:'count_kernel|pushdown|selection_result|dense_chunks|peer_exchange' \
    --log-file gpurun_out/meas/launches_final.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-graph --no-configs > gpurun_out/meas/launches_final.out 2>&1
