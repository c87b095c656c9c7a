#!/bin/bash
# the final build: GPU suite, smoke, default bench line, reference arm, 10-minute random stress
mkdir -p gpurun_out/${OUT:-r2z}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${OUT:-r2z}/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${OUT:-r2z}/pytest_gpu.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${OUT:-r2z}/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/${OUT:-r2z}/smoke.txt
( time timeout 900 python bench.py > gpurun_out/${OUT:-r2z}/bench.json 2> gpurun_out/${OUT:-r2z}/bench.err ) 2> gpurun_out/${OUT:-r2z}/bench_time.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${OUT:-r2z}/bench_ref.json 2> gpurun_out/${OUT:-r2z}/bench_ref.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --same-device > gpurun_out/${OUT:-r2z}/bench_2rank.json 2> gpurun_out/${OUT:-r2z}/bench_2rank.err
SECONDS_BUDGET=${STRESS_S:-600} timeout 900 python scripts/stress.py > gpurun_out/${OUT:-r2z}/stress.txt 2>&1; echo "rc=$?" >> gpurun_out/${OUT:-r2z}/stress.txt
