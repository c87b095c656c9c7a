"""Summarise a round's ncu captures (gpurun_out/) into profiles/<tag>/ (tracked):
  launches.csv        the launch list of `bench.py` filtered to libsel's kernels (+ per-kernel share)
  ncu_<kernel>.txt     key metrics, DRAM traffic, stall totals and the hottest SASS lines
and update profiles/ncu_traffic.json (dram read+write bytes per launch, read by bench.py).

    python scripts/summarize_profiles.py r1 [config]
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUR = ("count_kernel", "pushdown_kernel", "pushdown_sel_kernel", "selection_result_kernel",
       "dense_chunks_kernel", "superblock_prefix_kernel")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second"]


def kname(full):
    for k in OUR:
        if k in full and not (k == "pushdown_kernel" and "pushdown_sel_kernel" in full):
            return k
    return None


def launches(tag, out_dir):
    src = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    if not os.path.exists(src):
        return None
    text = open(src).read()
    text = text[text.index('"ID"'):] if '"ID"' in text else text
    rows = list(csv.DictReader(io.StringIO(text)))
    mine = [r for r in rows if kname(r.get("Kernel Name", ""))]
    with open(os.path.join(out_dir, "launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "block", "gpu__time_duration.sum", "unit"])
        for r in mine:
            w.writerow([r["ID"], kname(r["Kernel Name"]), r.get("Grid Size", ""), r.get("Block Size", ""),
                        r["Metric Value"], r["Metric Unit"]])
    tot = {}
    for r in mine:
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] in ("nsecond", "ns"):
            v /= 1000.0
        elif r["Metric Unit"] in ("msecond", "ms"):
            v *= 1000.0
        tot[kname(r["Kernel Name"])] = tot.get(kname(r["Kernel Name"]), 0.0) + v
    return {"all_launches": len(rows), "libsel_launches": len(mine), "us_by_kernel": tot}


def summarize(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    lines = [f"kernel: {d.get('Kernel Name', ('?',))[0]}"]
    for k in KEYS:
        if k in d:
            lines.append(f"{k:60s} {d[k][0]} {d[k][1]}")
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(sass)))
    if len(srows) > 2:
        sh = srows[1]
        ix = {k: i for i, k in enumerate(sh)}
        data = srows[2:]
        agg = {}
        for r in data:
            for k in sh:
                if k.startswith("stall_") and "(Not" not in k:
                    try:
                        agg[k] = agg.get(k, 0) + int(r[ix[k]] or 0)
                    except ValueError:
                        pass
        tot = sum(agg.values()) or 1
        lines.append("stall samples (share of all warp-state samples):")
        for k, val in sorted(agg.items(), key=lambda kv: -kv[1])[:8]:
            lines.append(f"   {k:28s} {val:8d}  {100.0 * val / tot:5.1f}%")
        lines.append("hottest SASS (samples, long-scoreboard, instruction):")
        top = sorted(data, key=lambda r: -int(r[ix['# Samples']] or 0))[:15]
        for r in top:
            lines.append(f"   {r[ix['# Samples']]:>7} lsb={r[ix['stall_long_sb']]:>6}  {r[ix['Source']].strip()[:100]}")
    open(out, "w").write("\n".join(lines) + "\n")

    def num(k):
        try:
            val, unit = d[k]
            x = float(val.replace(",", ""))
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
        except Exception:
            return None
    r, w = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    return int(r + w) if r is not None and w is not None else None


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    config = sys.argv[2] if len(sys.argv) > 2 else "c2"
    out_dir = os.path.join(ROOT, "profiles", tag)
    os.makedirs(out_dir, exist_ok=True)
    info = launches(tag, out_dir) or {}
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    traffic.setdefault(config, {})
    for k in OUR:
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}_{k}.ncu-rep")
        if os.path.exists(rep):
            t = summarize(rep, os.path.join(out_dir, f"ncu_{k}.txt"))
            if t:
                traffic[config][k] = t
    traffic[config]["_source"] = f"profiles/{tag}/ncu_*.txt (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch)"
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    json.dump(info, open(os.path.join(out_dir, "launches_summary.json"), "w"), indent=1)
    print(json.dumps(info, indent=1))
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
