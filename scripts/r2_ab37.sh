#!/bin/bash
# push-down block size by density below 150M rows (dyn) vs 1-chunk blocks always (bc1fixed):
# GPU suite on dyn; per-config shard-size bench lines under both
mkdir -p gpurun_out/r2x2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2x2/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2x2/pytest_gpu.log
for r in 1 2; do
for spec in "c2 75000000" "c5 125000000" "c4 60000000" "c3 37500000" "c6 60000000" "c0 75000000" "c2 144000000"; do
  set -- $spec
  for v in bc1fixed dyn; do
    lib=""; [ "$v" != dyn ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v $1 $2 " >> gpurun_out/r2x2/configs.txt
    env $lib timeout 400 python bench.py --config $1 --rows $2 --steps 40 --no-e2e --no-cpu --no-read-peak --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['latency_ms']['pushdown_kernels'], d['latency_ms']['count_kernel'])" >> gpurun_out/r2x2/configs.txt
  done
done
done
