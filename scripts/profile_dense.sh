# Run on the GPU box (via gpurun): launch list of bench.py c5 and full ncu captures of the
# push-down kernels at config 5 s = 1 (every chunk full: dense_chunks_kernel does the work).
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1k_c5.csv python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/launches_r1k_c5.out 2>&1
SWEEP_LAYOUTS=scattered SWEEP_S=1.0 SWEEP_EAGER=1 ncu --set full --clock-control none --import-source on -k regex:dense_chunks_kernel -s 2 -c 1 -o gpurun_out/prof_r1k_c5_dense_chunks_kernel -f python scripts/sweep_bench.py > gpurun_out/prof_dense.out 2>&1
SWEEP_LAYOUTS=scattered SWEEP_S=1.0 SWEEP_EAGER=1 ncu --set full --clock-control none --import-source on -k regex:pushdown_sel_kernel -s 2 -c 1 -o gpurun_out/prof_r1k_c5_pushdown_sel_kernel -f python scripts/sweep_bench.py > gpurun_out/prof_pd.out 2>&1
python scripts/summarize_profiles.py r1k_c5 c5_sweep_s1 > gpurun_out/summ.txt 2>&1
rm -f gpurun_out/*.ncu-rep
mkdir -p gpurun_out/prof_copy && cp -r profiles/r1k_c5 profiles/ncu_traffic.json gpurun_out/prof_copy/
