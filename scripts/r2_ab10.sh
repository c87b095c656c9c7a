#!/bin/bash
# push-down helpers not inlined (i-cache: 25 % no-instruction stalls) vs inlined; block size 2 vs 4
# at 150M / 300M rows
mkdir -p gpurun_out/r2n
timeout 1500 python scripts/ab_step.py 4 75000000,600000000 noinl=$PWD/build_exp/libsel_noinl.so base=- > gpurun_out/r2n/ab_step_noinl.jsonl 2>&1
for cfg in c3 c5 c6; do
  for v in base noinl base noinl; do
    lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v " >> gpurun_out/r2n/count_variants.txt
    env $lib timeout 300 python scripts/count_variants.py $cfg 30 >> gpurun_out/r2n/count_variants.txt 2>&1
  done
done
timeout 1500 python scripts/ab_step.py 3 150000000,300000000 bc2=$PWD/build_exp/libsel_bc2.so base=- > gpurun_out/r2n/ab_step_bc.jsonl 2>&1
SEL_LIB=$PWD/build_exp/libsel_noinl.so timeout 600 ncu --set full --clock-control none -k regex:pushdown_sel_kernel -s 3 -c 1 -o gpurun_out/r2n/pd_noinl -f python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph --no-read-peak --no-configs > gpurun_out/r2n/ncu.out 2>&1
ncu -i gpurun_out/r2n/pd_noinl.ncu-rep --page raw --csv > gpurun_out/r2n/pd_noinl_raw.csv 2>&1
ncu -i gpurun_out/r2n/pd_noinl.ncu-rep --page source --csv > gpurun_out/r2n/pd_noinl_src.csv 2>&1
rm -f gpurun_out/r2n/*.ncu-rep
