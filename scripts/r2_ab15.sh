#!/bin/bash
# the coded column's bits stored with normal priority (wplain) / evict_first (wfirst) vs evict_last
mkdir -p gpurun_out/r2v
timeout 1500 python scripts/ab_step.py 4 300000000,600000000 base=- wplain=$PWD/build_exp/libsel_wplain.so wfirst=$PWD/build_exp/libsel_wfirst.so > gpurun_out/r2v/ab_step.jsonl 2>&1
