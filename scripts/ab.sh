#!/bin/bash
# A/B timing of library variants (build_exp/libsel_<tag>.so, see _build.py) on bench configs.
# Usage (GPU box): scripts/ab.sh "c2 c4" base gb16 ...   (base = the in-tree libsel.so)
CFGS=$1; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in $CFGS; do
  for v in "$@"; do
    lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    env $lib timeout 300 python bench.py --steps 20 --warmup 5 --config $cfg --no-e2e --no-cpu 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $v', d['ms_per_step'], d['latency_ms']['count_kernel'], d['latency_ms']['pushdown_kernels'])" 2>&1 | tail -1
  done
done
