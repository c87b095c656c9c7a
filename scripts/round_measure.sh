# Round-end measurement set: default bench line, every config, the standalone
# push-down paths, and the strong-scaling shard sizes with a one-rank peer exchange.
mkdir -p gpurun_out/meas
timeout 600 python bench.py > gpurun_out/meas/bench_default.json 2> gpurun_out/meas/bench_default.err
for c in c0 c1 c3 c4 c5 c6; do
  timeout 400 python bench.py --config $c --steps 50 --no-e2e --no-read-peak > gpurun_out/meas/bench_$c.json 2> gpurun_out/meas/bench_$c.err
done
timeout 600 python scripts/pushdown_paths.py > gpurun_out/meas/pushdown_paths.jsonl 2>&1
for r in 600000000 300000000 150000000 75000000; do
  timeout 300 python bench.py --rows $r --steps 50 --no-e2e --no-cpu --no-read-peak --peers1 > gpurun_out/meas/strong_$r.json 2>/dev/null
done
ls -la gpurun_out/meas
