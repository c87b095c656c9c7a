"""Summarise an .ncu-rep: key metrics + top stall reasons + hottest source lines."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = {h[i]: (v[i], u[i]) for i in range(len(h))}
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum", "lts__t_sectors_op_atom.sum",
        "smsp__inst_executed.sum"]
for k in keys:
    if k in d: print(f"{k:60s} {d[k][0]} {d[k][1]}")
stalls = [(k, d[k][0]) for k in h if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio")]
def f(x):
    try: return float(x)
    except: return 0.0
stalls = sorted(stalls, key=lambda kv: -f(kv[1]))[:8]
print("top stalls (cycles per issued instr):")
for k, val in stalls: print(f"   {k.replace('smsp__average_warp_latency_issue_stalled_','')[:-6]:30s} {val}")
