#!/bin/bash
# ncu profile of the default bench step (launch list + full captures) summarised on the box, the
# reports deleted (gpurun copies back <= 64 MiB), then the round measurement set.
bash scripts/profile.sh r2p
python scripts/summarize_profiles.py r2p c2 > gpurun_out/r2p_summary.json 2>&1
mkdir -p gpurun_out/r2p_profiles
cp -r profiles/r2p/* gpurun_out/r2p_profiles/
cp profiles/ncu_traffic.json gpurun_out/r2p_profiles/ncu_traffic.json
for K in count_kernel pushdown_sel_kernel; do
  ncu -i gpurun_out/prof_r2p_${K}.ncu-rep --page details > gpurun_out/r2p_profiles/details_${K}.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
bash scripts/round_measure.sh
du -sh gpurun_out
