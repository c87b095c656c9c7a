mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
for cfg in c2 c3 c4 c5; do
 for f in 0 1; do
  SEL_FAST=$f timeout 300 python bench.py --config $cfg --steps 20 --no-cpu --no-e2e --no-read-peak > gpurun_out/ab_${cfg}_fast$f.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_${cfg}_fast$f.json')); print('$cfg fast=$f', d['ms_per_step'], d['latency_ms']['count_kernel'], d['latency_ms']['pushdown_kernels'], d['latency_ms']['count_probe']['median'])"
 done
done
