#!/bin/bash
# ncu profile of the default bench step (launch list + full captures) summarised on the box, the
# reports deleted (gpurun copies back <= 64 MiB), then the round measurement set.
bash scripts/profile.sh r2q
python scripts/summarize_profiles.py r2q c2 > gpurun_out/r2q_summary.json 2>&1
mkdir -p gpurun_out/r2q_profiles
cp -r profiles/r2q/* gpurun_out/r2q_profiles/
cp profiles/ncu_traffic.json gpurun_out/r2q_profiles/ncu_traffic.json
for K in count_kernel pushdown_sel_kernel; do
  ncu -i gpurun_out/prof_r2q_${K}.ncu-rep --page details > gpurun_out/r2q_profiles/details_${K}.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
bash scripts/round_measure.sh
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/meas/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/meas/pytest_gpu.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/meas/smoke.txt 2>&1
du -sh gpurun_out
