#!/bin/bash
# Round 2 A/B 1: fixed per-call costs (overhead_probe) and count-kernel variants
# (quad = masks stored without the row-major transposition, timing only; minb4/minb2 = fast-path
# register bound 64 / 128).
mkdir -p gpurun_out/r2b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b/build.log 2>&1
timeout 300 python scripts/overhead_probe.py 60000 6000000 75000000 600000000 > gpurun_out/r2b/overhead.jsonl 2>&1
for cfg in c2 c5 c4; do
  for v in base quad minb4 minb2; do
    lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v " >> gpurun_out/r2b/count_variants.txt
    env $lib timeout 300 python scripts/count_variants.py $cfg 30 >> gpurun_out/r2b/count_variants.txt 2>&1
  done
done
ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.max --clock-control none --csv -k regex:'count_kernel|pushdown|prefix|dense' -c 80 \
  python scripts/overhead_probe.py 75000000 > gpurun_out/r2b/ncu_75M.csv 2>&1
