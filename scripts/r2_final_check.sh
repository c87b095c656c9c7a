#!/bin/bash
# What the driver runs at round end, on this build: smoke, the default bench line (timed), the
# reference arm, and a 2-rank same-device run of the N>1 bench path.
mkdir -p gpurun_out/r2s
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2s/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r2s/smoke.txt
( time timeout 900 python bench.py > gpurun_out/r2s/bench.json 2> gpurun_out/r2s/bench.err ) 2> gpurun_out/r2s/bench_time.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2s/bench_ref.json 2> gpurun_out/r2s/bench_ref.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --same-device > gpurun_out/r2s/bench_2rank.json 2> gpurun_out/r2s/bench_2rank.err
