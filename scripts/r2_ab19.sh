#!/bin/bash
# keeping-count L2 prefetch vs table size (C2 shapes): where does it stop paying?
mkdir -p gpurun_out/r2z
timeout 2000 python scripts/ab_step.py 4 37500000,75000000,150000000,300000000 off=- pf=-@SEL_PREFETCH=1 > gpurun_out/r2z/ab_step.jsonl 2>&1
