#!/bin/bash
# the count's partial tail chunk evaluated first (tailfirst = in-tree) vs last (base); timing markers
mkdir -p gpurun_out/r2ee
SEL_LIB=$PWD/build_exp/libsel_dbg.so python scripts/step_breakdown.py 75000000 > gpurun_out/r2ee/dbg_75M.txt 2>&1
SEL_LIB=$PWD/build_exp/libsel_dbg.so python scripts/step_breakdown.py 600000000 > gpurun_out/r2ee/dbg_600M.txt 2>&1
timeout 1500 python scripts/ab_step.py 4 75000000,150000000,600000000 base=$PWD/build_exp/libsel_base.so tailfirst=- > gpurun_out/r2ee/ab_step.jsonl 2>&1
