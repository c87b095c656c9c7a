#!/usr/bin/env python
"""bench.py — the exact-selectivity probe on B200 (BASELINE.json metric: "selectivity-probe latency
(ms) and scanned GB/s vs HBM peak at 1/2/4/8 B200").

One step = one pass of the whole hot path over the worked example R of the
paper (BASELINE.json configs[1]): 600M rows, predicate
`A = 2 AND B < 2001 AND B > 1000 AND (C = 1 OR C = 4)` (Listing 3.1):
  a2-a5  sel_count   -> the exact count (100,200,000), all-reduced over ranks when N > 1
  a6-a7  sel_pushdown -> ascending row ids + projected A, C, D, offsets over ranks
Rows are sharded contiguously over ranks (strong scaling: the global table is fixed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|...]
Under torchrun (N > 1) every rank runs its shard; rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "selectivity-probe latency (ms) and scanned GB/s vs HBM peak at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c0", "c1", "c2", "c3", "c4", "c5", "c6"])
    ap.add_argument("--rows", type=int, default=0, help="override global rows (testing only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-read-peak", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time table.execute() per step instead of the prepared (graph) execute")
    ap.add_argument("--blocking", action="store_true",
                    help="time the blocking prepared Execute (returns after the materialisation) "
                         "instead of sel_prepared_execute_async (returns at the count; the "
                         "materialisation completes in stream order inside the timed region)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the other configs' probes (c3, c5) measured beside c2")
    ap.add_argument("--no-xchg-ab", action="store_true",
                    help="N > 1: skip timing the other exchange mechanism")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--ref-rows", type=int, default=60_000_000,
                    help="--impl reference: rows of the workload each oracle step runs on")
    ap.add_argument("--cpu-rows", type=int, default=0,
                    help="rows of the CPU oracle baseline (0: the whole table)")
    ap.add_argument("--comm1", action="store_true",
                    help="testing: give the N=1 context a one-rank NCCL communicator (the N>1 "
                         "collectives on the step's critical path, without peers)")
    ap.add_argument("--same-device", action="store_true",
                    help="testing: every rank on cuda:0 (torch.distributed over gloo; the ranks "
                         "time-slice one GPU, so timings are meaningless) to exercise the N > 1 "
                         "path on a one-GPU box")
    ap.add_argument("--xchg", default=os.environ.get("SEL_XCHG", "peers"), choices=["peers", "nccl"],
                    help="N > 1: the cross-rank exchange — the library's own over peer memory "
                         "(NCCL on every rank if any rank cannot map the others) or NCCL")
    ap.add_argument("--peers1", action="store_true",
                    help="testing: give the N=1 context a one-rank peer exchange (the N>1 "
                         "exchange on the step's critical path)")
    return ap.parse_args()


# ---- workloads ---------------------------------------------------------------------------------

def workload(name, rows):
    """(global rows, generator(row_start, row_count, device) -> Table, program AST, projection,
    description). BASELINE.json configs: c1..c5; the bench line is c2. c6 (NEXT(3))
    also needs key sets: see key_sets()."""
    from selgen import configs
    if name == "c6":
        n = rows or configs.ssb_sizes(80)["lineorder"]
        node, _ = configs.q2_probes(80)["q2.1"]
        return (n, lambda s, c, d: configs.gen_lineorder_q2(n, 80, s, c, device=d), node, [0, 1, 3],
                "SSB SF-80 lineorder, Q2.1 semijoin probe: lo_partkey IN {p_category = 12} AND "
                "lo_suppkey IN {s_region = 1} (PAPER.md:719-729), push-down of orderdate, partkey, revenue")
    if name == "c0":   # SURVEY §8d optional context: TPC-H SF-50 orders
        n = rows or 75_000_000
        return (n, lambda s, c, d: configs.gen_orders(n, s, c, device=d),
                configs.orders_probes()["q5_orderdate"], [0, 1],
                "TPC-H SF-50 orders (75M rows), Q5's o_orderdate one-year range (PAPER.md:698-699; "
                "15.2% of orders, PAPER.md:646), push-down of o_orderkey, o_custkey")
    if name == "c2":
        n = rows or configs.C2_ROWS
        return (n, lambda s, c, d: configs.gen_c2(n, s, c, device=d),
                configs.c2_probes()["listing"], configs.C2_PROJECT,
                "worked example R (PAPER.md:55-64): 600M rows, Listing 3.1 COUNT + push-down of A,C,D")
    if name in ("c1", "c3"):
        n = rows or (60_000 if name == "c1" else 300_000_000)
        cols = ["l_orderkey", "l_discount", "l_extendedprice", "l_returnflag", "l_shipdate", "l_shipmode"]
        def gen(s, c, d):
            return configs.gen_lineitem(n, s, c, device=d, columns=cols)
        probes = configs.lineitem_probes(gen(0, 16, "cpu"))
        if name == "c1":
            return n, gen, probes["listing1"], [0], "TPC-H SF-0.01 lineitem, Listing 1.1 mapped"
        return n, gen, probes["q10"], [0, 2, 1], "TPC-H SF-50 lineitem, Q10-style predicate"
    if name == "c4":
        n = rows or 480_000_000
        return (n, lambda s, c, d: configs.gen_lineorder(n, s, c, device=d),
                configs.lineorder_probes()["q1.1"], [3], "SSB SF-80 lineorder, Q1.1 predicate")
    n = rows or configs.C5_ROWS
    return (n, lambda s, c, d: configs.gen_sweep(n, s, c, device=d),
            configs.sweep_probe(configs.sweep_threshold(n, 0.01)), [1],
            "1e9-row sweep, x < 0.01 N")


def key_sets(name):
    """The IN_BITMAP key sets of a workload ([(uint64 words, nbits)], ids = positions), or []."""
    if name != "c6":
        return []
    from selgen import configs
    return configs.q2_probes(80)["q2.1"][1]


def const_columns(prog, types):
    """Columns the program pins to one value (a conjunction with a single-point leaf on them):
    the push-down fills those projections instead of reading them."""
    import paper_1806_08384_b200 as sel
    plan = sel.program_plan(prog, types)
    if plan["path"] != 1:
        return set()
    return {L["col"] for L in plan["leaves"]
            if "bitmap" not in L and len(L["lo"]) == 1 and L["span"] == [0]}


def coded_columns(prog, types, proj):
    """Projected columns pinned to two values by a fast-path 1-byte leaf: the keeping count keeps
    one code bit per row for them and the push-down never reads them."""
    import os as _os
    import paper_1806_08384_b200 as sel
    if _os.environ.get("SEL_CODED", "1") == "0":
        return set()
    plan = sel.program_plan(prog, types)
    for L, kind in zip(plan["leaves"], plan.get("fast") or []):
        pts = sum(sp + 1 for sp in L["span"])
        two_points = (kind == 4 and pts == 2) or (kind == 2 and L["span"] == [0, 0])
        if two_points and L["col"] in proj:
            return {L["col"]}
    return set()


def algo_bytes(table, prog_cols, proj, local_count, pushdown_path=0, consts=(), coded=()):
    """Algorithmic bytes.
    step  = what COUNT + push-down must move once (e.g. C2: 5.4 GB scan + 0.40 GB of D
            read + 1.303 GB written = 7.10 GB): rows x distinct predicate widths + selected x
            non-predicate projected widths + selected x (4 + projected widths) + 8 B count.
            Implementation-independent: the same figure divides both arms' step times.
    count kernel = rows x distinct predicate widths + 8 B.
    push-down kernel, by the path it took:
      single pass (0): the count scan + selected x non-predicate projected widths + writes;
      from a kept selection (1): the selection (rows/8 + 2 B per 1024 rows) + selected x all
                       projected widths + writes — it evaluates nothing, so no predicate column
                       is charged; columns pinned to a constant (`consts`) are filled, not read."""
    w = [c.width for c in table.columns]
    n = table.n_rows
    scan = n * sum(w[c] for c in prog_cols)
    count_b = scan + 8
    write = local_count * (4 + sum(w[c] for c in proj))
    single = scan + local_count * sum(w[c] for c in set(proj) if c not in prog_cols) + write
    if pushdown_path == 1:
        selection = n // 8 + 2 * ((n + 1023) // 1024)
        push_b = (selection + len(coded) * (n // 8)
                  + local_count * sum(w[c] for c in proj if c not in consts and c not in coded) + write)
    else:
        push_b = single
    return count_b, push_b, single + 8


def prog_columns(node):
    from selgen.program import Cmp, Between, In, InSet, And, Or, Not
    if isinstance(node, (Cmp, Between, In, InSet)):
        return {node.col}
    if isinstance(node, (And, Or)):
        return prog_columns(node.l) | prog_columns(node.r)
    if isinstance(node, Not):
        return prog_columns(node.x)
    return set()


# ---- clocks ----------------------------------------------------------------------------------------

class ClockSampler:
    """NVML sampling of SM clock and throttle reasons DURING the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.0002)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 1.0:   # sampling before the region
                time.sleep(0.0005)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self._t.join()

    def mark(self):
        """End of the timed region: samples after this cover the same steps' second pass (the
        per-kernel timing pass), which keeps the GPU under the same load."""
        self.n_timed = len(self.samples)

    def summary(self):
        xs = self.samples
        nt = getattr(self, "n_timed", len(xs))
        med = statistics.median(xs) if xs else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(xs), "samples_timed_region": nt,
                "sm_mhz_timed_region": statistics.median(xs[:nt]) if nt else None,
                "sm_mhz_min": min(xs) if xs else None,
                "window": "the timed steps and the same steps' per-kernel timing pass right after"}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(kernel, config, applies=True):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu capture
    (captured at N = 1 on the full table: null for other launch shapes)."""
    if not applies:
        return None
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(config, {}).get(kernel)
    except Exception:
        return None


# ---- the oracle as baseline / reference arm ------------------------------------------------------

def cpu_baseline(host_cols, table_like, prog, proj, prog_cols, nthreads, bitmaps=None):
    """The oracle as it stands (SURVEY §8(d) CPU protocol), outside any timed GPU region:
    all_cores     — count (oracle_count_mt) + push-down (oracle_pushdown_mt) on `nthreads`;
    single_thread — count (oracle_count) + push-down (oracle_pushdown) on one thread.
    Both over the rows given; each records its seconds, GB/s of the step's algorithmic bytes and
    rows/s. Returns (all_cores, single_thread, count)."""
    import oracle
    types = table_like.types
    rows = len(host_cols[0]) if host_cols else 0

    def leg(threads):
        t0 = time.perf_counter()
        if threads > 1:
            cnt = oracle.count_mt(host_cols, types, prog, threads, bitmaps=bitmaps)
            t1 = time.perf_counter()
            c2, _, _ = oracle.pushdown_mt(host_cols, types, prog, proj=proj, bitmaps=bitmaps,
                                          nthreads=threads)
        else:
            cnt = oracle.count(host_cols, types, prog, bitmaps=bitmaps)
            t1 = time.perf_counter()
            c2, _, _ = oracle.pushdown(host_cols, types, prog, proj=proj, bitmaps=bitmaps)
        t2 = time.perf_counter()
        assert c2 == cnt
        _, _, step_b = algo_bytes(table_like, prog_cols, proj, cnt, 0)
        return {"threads": threads, "rows": rows, "count_s": round(t1 - t0, 3),
                "pushdown_s": round(t2 - t1, 3), "step_s": round(t2 - t0, 3),
                "gbs": round(step_b / (t2 - t0) / 1e9, 3),
                "rows_per_s": round(rows / (t2 - t0))}, cnt

    allc, cnt = leg(nthreads)
    single, _ = leg(1)
    return allc, single, cnt


def cpu_model():
    """The host CPU model (each CPU record states the model and the thread count)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on the host cores, on a bounded sample."""
    import numpy as np
    import oracle
    from selgen import encode
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n, gen, node, proj, desc = workload(args.config, args.rows)
    bms = key_sets(args.config)
    sample = min(n, args.ref_rows)
    T = gen(0, sample, "cpu")
    cols = [c.numpy() for c in T.columns]
    prog = encode(node, T.types)
    pc = prog_columns(node)
    nthreads = os.cpu_count() or 1
    w = [c.width for c in T.columns]
    def step():
        t0 = time.perf_counter()
        cnt = oracle.count_mt(cols, T.types, prog, nthreads, bitmaps=bms)
        c2, ids, outs = oracle.pushdown_mt(cols, T.types, prog, proj=proj, bitmaps=bms,
                                           nthreads=nthreads)
        return time.perf_counter() - t0, cnt
    for _ in range(args.warmup):
        step()
    times = []
    cnt = 0
    for _ in range(args.steps):
        dt, cnt = step()
        times.append(dt)
    cb, pb, total = algo_bytes(T, pc, proj, cnt, 0)
    ms = 1000 * sum(times) / len(times)
    value = total / (ms / 1000) / 1e9
    line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32/u8 compare, u64 count", "data": "synthetic",
            "config": {"workload": f"{args.config}: {desc}", "global_rows": n,
                       "sample_rows": sample},
            "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": nthreads,
                             "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"first {sample} of {n} rows of the workload per step; count (oracle_count_mt) and push-down (oracle_pushdown_mt) on {nthreads} threads"},
            "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)


# ---- our arm ---------------------------------------------------------------------------------------

def _max_over_ranks(vals, world, dev):
    """Element-wise max over ranks of a list of floats (the device-time rule)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=_red_dev(dev))
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t]


def time_prepared(prep, steps, world, dev, wait=False):
    """ms per prepared-Execute replay: CUDA events around `steps` replays on the current stream,
    barrier + synchronize on both sides, max over ranks. wait=False: each replay returns at its
    count (sel_prepared_execute_async), the materialisation finishing in stream order."""
    import torch
    import torch.distributed as dist
    for _ in range(3):
        prep.run()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        prep.run(wait=wait)
    b.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    return _max_over_ranks([a.elapsed_time(b) / steps], world, dev)[0]


def measure_exchange_ab(args, sel, sdist, T, names, proj_names, prog, n, s, local_count, world,
                        dev, main_xchg):
    """N > 1: the same prepared Execute over the other exchange mechanism (a second context), so
    that one run measures both the library's peer-memory exchange and north_star's NCCL
    collectives."""
    other = "nccl" if main_xchg.startswith("peers") else "peers"
    ctx2 = sel.Context(dev)
    try:
        got = sdist.setup_exchange(ctx2, other)
    except Exception as ex:  # noqa: BLE001 - e.g. NCCL refuses two ranks on one GPU (--same-device)
        ctx2.close()
        return {"requested": other, "error": f"{type(ex).__name__}: {ex}"[:300]}
    t2 = sel.Table(ctx2, names, T.types, [c.data for c in T.columns], row_offset=s, global_rows=n)
    prep = t2.prepare_execute(prog, project=proj_names, max_size=n, capacity=max(local_count, 1))
    ms = time_prepared(prep, args.steps, world, dev, wait=args.blocking)
    c = prep.run()
    prep.release()
    t2.release()
    if got.startswith("peers"):
        ctx2.drop_peers()
    import torch.distributed as dist
    dist.barrier()
    ctx2.close()
    return {"requested": other, "exchange": got, "ms_per_step": round(ms, 4), "count": c,
            "steps": args.steps}


def measure_configs(names_, args, sel, sdist, world, rank, dev, hbm):
    """Other BASELINE.json configs in the same run: for each, the count probe's
    latency through the public call (host clock, >= 50 warm reps, max over ranks per rep), the
    count kernel's time (the library's CUDA events, median of 20) and roofline against the
    measured peak, and the prepared Execute step of bench.workload's probe and projection."""
    import torch
    from selgen import encode
    out = {}
    for name in names_:
        n, gen, node, proj, desc = workload(name, 0)
        s, e = sdist.shard_range(n, world, rank)
        T = gen(s, e - s, dev)
        torch.cuda.synchronize()
        ctx = sel.Context(dev)
        xchg = sdist.setup_exchange(ctx, args.xchg) if world > 1 else None
        names = [c.name for c in T.columns]
        t = sel.Table(ctx, names, T.types, [c.data for c in T.columns], row_offset=s, global_rows=n)
        prog = encode(node, T.types)
        pc = prog_columns(node)
        for _ in range(5):
            cnt = t.count(prog)
        lat = []
        for _ in range(max(50, args.steps)):
            t0 = time.perf_counter()
            t.count(prog)
            lat.append(1000 * (time.perf_counter() - t0))
        lat = _max_over_ranks(lat, world, dev)
        ctx.enable_timing(True)
        kms = []
        for _ in range(20):
            t.count(prog)
            kms.append(ctx.last_kernel_ms())
        ctx.enable_timing(False)
        k_ms = _max_over_ranks([statistics.median(kms)], world, dev)[0]
        cb = (e - s) * sum(T.columns[c].width for c in pc) + 8
        gbs = cb / (k_ms / 1000) / 1e9
        local = t.pushdown(prog, capacity=0).local_count
        prep = t.prepare_execute(prog, project=[names[j] for j in proj], max_size=n,
                                 capacity=max(local, 1))
        step_ms = time_prepared(prep, args.steps, world, dev, wait=args.blocking)
        prep.release()
        xs = sorted(lat)
        out[name] = {
            "workload": desc, "global_rows": n, "rows_per_gpu": e - s, "selected": cnt,
            "count_probe_ms": {"min": round(xs[0], 4), "median": round(statistics.median(xs), 4),
                               "p99": round(xs[min(len(xs) - 1, int(0.99 * len(xs)))], 4),
                               "reps": len(xs), "clock": "host, around Table.count (sel_count)"},
            "count_kernel": {"bound": "hbm", "ms": round(k_ms, 4),
                             "algorithmic_bytes_per_launch": int(cb),
                             "achieved": round(gbs, 2), "peak": hbm, "unit": "GB/s",
                             "frac": round(gbs / hbm, 4)},
            "execute_step_ms": round(step_ms, 4),
            "exchange": xchg}
        if name == "c3":
            out[name]["vs_paper_30ms"] = ("the paper's GPU probe overhead was a flat 18-28 ms "
                                          "(PAPER.md:430, 446); this probe's median is "
                                          f"{statistics.median(xs):.3f} ms")
        t.release()
        if world > 1 and xchg and xchg.startswith("peers"):
            ctx.drop_peers()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        ctx.close()
        del T, t
        torch.cuda.empty_cache()
    return out


_GLOO = False


def _red_dev(dev):
    """Device of the small tensors reduced over torch.distributed (CPU under --same-device/gloo)."""
    return "cpu" if _GLOO else dev


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1806_08384_b200 as sel
    from selgen import encode

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world
    global _GLOO
    if args.same_device:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if args.same_device:
            _GLOO = True
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    from paper_1806_08384_b200 import dist as sdist
    n, gen, node, proj, desc = workload(args.config, args.rows)
    s, e = sdist.shard_range(n, world, rank)
    T = gen(s, e - s, dev)
    torch.cuda.synchronize()
    ctx = sel.Context(dev)
    xchg = None
    if world > 1:
        xchg = sdist.setup_exchange(ctx, args.xchg)
    elif args.comm1:
        ctx.set_comm(1, 0, sel.Context.new_unique_id())
        xchg = "nccl (one rank)"
    elif args.peers1:
        ctx.set_peers(1, 0, [ctx.peer_handle()])
        xchg = "peers (one rank)"
    bms = key_sets(args.config)   # NEXT(3) key sets (c6), registered once like the table
    bm_dev = []
    for words, nbits in bms:
        bm_dev.append(torch.from_numpy(words.view(np.int64).copy()).to(dev))
        assert ctx.register_bitmap(bm_dev[-1], nbits) == len(bm_dev) - 1
    names = [c.name for c in T.columns]
    table = sel.Table(ctx, names, T.types, [c.data for c in T.columns], row_offset=s, global_rows=n)
    prog = encode(node, T.types)
    pc = prog_columns(node)
    proj_names = [names[j] for j in proj]
    stream = torch.cuda.current_stream(dev)

    # exact-size outputs from a first count (Algorithm 1: count, then materialise)
    probe = table.pushdown(prog, project=proj_names)
    local_count = probe.local_count
    global_count = probe.count
    cap = max(local_count, 1)
    out_ids = torch.empty(cap, dtype=torch.int32, device=dev)
    out_cols = [torch.empty(cap, dtype=c.data.dtype, device=dev) for c in (T.columns[j] for j in proj)]

    count_ms, push_ms, count_lat, push_lat, ready_lat = [], [], [], [], []

    # Algorithm 1's Execute(compound, isSPD=true, maxSize) with PUSH_DOWN_MAX_SELECTIVITY = 1.0
    # (the paper's push-down experiments): count (keeping the selection and the
    # projected predicate columns) -> device-side gate -> materialise. Prepared once (validated,
    # captured into a CUDA graph: include/sel.h sel_prepare_execute), one replay + sync per step.
    prepared = None if args.no_graph else table.prepare_execute(
        prog, project=proj_names, max_size=n, capacity=local_count, out=(out_ids, out_cols))

    class _R:
        pass

    def step(record, wait=True):
        t0 = time.perf_counter()
        if prepared is not None:
            c = prepared.run(wait=wait)
            r = _R()
            r.count, r.materialized = c, prepared.materialized
        else:
            r = table.execute(prog, project=proj_names, max_size=n, capacity=local_count,
                              out=(out_ids, out_cols))
        t1 = time.perf_counter()
        if record == "latency":
            count_lat.append(1000 * (t1 - t0))
        elif record == "ready":
            ready_lat.append(1000 * (t1 - t0))
        elif record == "kernels":
            k1, k2 = ctx.last_times()
            count_ms.append(k1); push_ms.append(k2)
        return r.count, r

    # The timed steps run without the library's per-kernel timing events (event-record nodes in
    # the graph cost ~20 us per step: scripts/step_overhead.py); the per-kernel times come from a
    # second pass of the same steps with timing on.
    ctx.enable_timing(False)
    for _ in range(max(args.warmup, 3)):
        c, r = step(None)
        assert c == global_count and r.materialized
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step("ready", wait=args.blocking)
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark()
        if world > 1:
            dist.barrier()
        dev_ms = ev0.elapsed_time(ev1)
        for _ in range(max(args.steps, 20)):   # the blocking Execute's latency, call to return
            step("latency")
        ctx.enable_timing(True)
        for _ in range(3):
            step(None)
        for _ in range(max(args.steps, 20)):
            step("kernels")
        ctx.enable_timing(False)
    pd_path = ctx.last_pushdown_path()
    consts = const_columns(prog, T.types)
    coded = coded_columns(prog, T.types, proj) if pd_path == 1 else set()
    cb, pb, step_b = algo_bytes(T, pc, proj, local_count, pd_path, consts, coded)
    my_bytes = step_b
    t = torch.tensor([dev_ms, my_bytes, cb, pb, statistics.median(count_ms), statistics.median(push_ms)],
                     dtype=torch.float64, device=_red_dev(dev))
    if world > 1:
        tmax = t.clone(); dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone(); dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    else:
        tmax = tsum = t
    total_ms = float(tmax[0])
    ms_per_step = total_ms / args.steps
    agg_bytes = float(tsum[1])
    value_gbs = agg_bytes / (ms_per_step / 1000) / 1e9

    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs")
    peak_note = "MEASURED_PEAKS.json hbm_gbs (copy, read+write)"
    if not hbm:
        hbm, peak_note = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    push_k = statistics.median(push_ms)
    count_k = statistics.median(count_ms)
    push_gbs = pb / (push_k / 1000) / 1e9
    count_gbs = cb / (count_k / 1000) / 1e9

    # ---- probe latency: host clock around the public call, >= 50 warm reps ----
    def _stats(xs):
        xs = sorted(xs)
        return {"min": round(xs[0], 4), "median": round(statistics.median(xs), 4),
                "p99": round(xs[min(len(xs) - 1, int(0.99 * len(xs)))], 4), "reps": len(xs)}
    ctx.enable_timing(False)
    for _ in range(5):
        table.count(prog)
    count_probe = []
    for _ in range(max(50, args.steps)):
        t0 = time.perf_counter()
        table.count(prog)
        count_probe.append(1000 * (time.perf_counter() - t0))
    count_probe_stats = _stats(count_probe)

    # ---- read-only streaming reference measured in this run (SURVEY §8(d) peak iii) ----
    read_peak = None
    if world == 1 and not args.no_read_peak:
        buf = torch.ones(1 << 31, dtype=torch.float32, device=dev)   # 8 GiB
        for _ in range(3):
            buf.sum()
        ra, rb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ra.record()
        for _ in range(5):
            buf.sum()
        rb.record()
        torch.cuda.synchronize()
        read_peak = round(5 * buf.numel() * 4 / (ra.elapsed_time(rb) / 1000) / 1e9, 1)
        del buf
        torch.cuda.empty_cache()

    # ---- e2e: the same step through the public API from pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        # End to end through the public API from pinned host memory, pipelined across steps:
        # step i+1's inputs stream in (copy engine H2D) while step i probes and step i's results
        # stream out (D2H) — PCIe is full duplex. Every step still copies all its inputs in and
        # its results out inside the timed region; device inputs/outputs are double-buffered.
        host = [c.data.cpu().pin_memory() for c in T.columns]
        bufs = [[c.data for c in T.columns], [torch.empty_like(c.data) for c in T.columns]]
        tabs = [table, sel.Table(ctx, names, T.types, bufs[1], row_offset=s, global_rows=n)]
        outs = [(out_ids, out_cols), (torch.empty_like(out_ids), [torch.empty_like(o) for o in out_cols])]
        h_ids = torch.empty(cap, dtype=torch.int32).pin_memory()
        h_cols = [torch.empty(cap, dtype=o.dtype).pin_memory() for o in out_cols]
        h2d = sum(h.numel() * h.element_size() for h in host)
        d2h = cap * 4 + sum(h.numel() * h.element_size() for h in h_cols) + 8
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev = lambda: torch.cuda.Event()
        in_ready, out_ready, out_free = [ev(), ev()], [ev(), ev()], [ev(), ev()]

        def h2d_into(b):
            with torch.cuda.stream(s_in):
                for d, h in zip(bufs[b], host):
                    d.copy_(h, non_blocking=True)
                in_ready[b].record(s_in)

        def run(steps):
            counts = []
            h2d_into(0)
            for i in range(steps):
                b = i % 2
                stream.wait_event(in_ready[b])
                if i + 1 < steps:
                    h2d_into(1 - b)                          # overlaps this step's probe
                if i >= 2:
                    stream.wait_event(out_free[b])
                r = tabs[b].execute(prog, project=proj_names, max_size=n, capacity=local_count,
                                    out=outs[b])
                counts.append(r.count)
                out_ready[b].record(stream)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(out_ready[b])
                    h_ids.copy_(outs[b][0], non_blocking=True)
                    for h, o in zip(h_cols, outs[b][1]):
                        h.copy_(o, non_blocking=True)
                    out_free[b].record(s_out)
            return counts

        run(2)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(s_in)
        counts = run(args.e2e_steps)
        s_out.synchronize()
        eb.record(s_out)
        torch.cuda.synchronize()
        assert all(c == global_count for c in counts)
        e_ms = torch.tensor([ea.elapsed_time(eb)], dtype=torch.float64, device=_red_dev(dev))
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e_step = float(e_ms[0]) / args.e2e_steps
        e2e = {"value": round(agg_bytes / (e_step / 1000) / 1e9, 3), "unit": "GB/s",
               "ms_per_step": round(e_step, 3), "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": args.e2e_steps,
               "mode": "pipelined across steps (H2D of step i+1 || probe + D2H of step i), pinned host memory"
                       + ("; key sets resident (registered once)" if bms else "")}
        tabs[1].release()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        nrows = T.n_rows if not args.cpu_rows else min(T.n_rows, args.cpu_rows)
        host_cols = [c.data[:nrows].cpu().numpy().view(
            {1: np.int32, 2: np.int64, 3: np.float32, 4: np.int32, 5: np.uint8, 6: np.uint16,
             7: np.uint32}[c.ctype]) for c in T.columns]
        nthreads = os.cpu_count() or 1
        sample_table = type("S", (), {})()
        sample_table.columns, sample_table.n_rows, sample_table.types = T.columns, nrows, T.types
        allc, single, cnt = cpu_baseline(host_cols, sample_table, prog, proj, pc, nthreads,
                                         bitmaps=bms)
        what = "the whole table" if nrows == T.n_rows else f"the first {nrows} of {n} rows"
        cpu = {"value": allc["gbs"], "unit": "GB/s", "cores": nthreads, "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": f"{what}: count (oracle_count_mt) + push-down (oracle_pushdown_mt) on "
                         f"{nthreads} threads, {allc['step_s']} s; single_thread: oracle_count + "
                         f"oracle_pushdown on 1 thread, {single['step_s']} s",
               "all_cores": allc, "single_thread": single}
        del host_cols

    push_name = "pushdown_sel_kernel" if pd_path == 1 else "pushdown_kernel"
    # Sector-granular minimum of the push-down: a gather must move every 32-byte
    # sector holding a selected row; counted exactly from this run's row ids (outside the timed
    # region). For the single pass the predicate columns are scanned densely anyway.
    ids64 = (out_ids[:local_count].to(torch.int64) & 0xFFFFFFFF) - s
    w_all = [c.width for c in T.columns]
    def sectors(width):
        if local_count == 0:
            return 0
        return int(torch.unique_consecutive(ids64 // (32 // width)).numel())
    write_b = local_count * (4 + sum(w_all[j] for j in proj))
    def lines(width):      # 128-byte lines holding a selected row: the DRAM fetch granularity of
        if local_count == 0:   # scattered gathers measured by ncu (~90-128 B per gathered value)
            return 0
        return int(torch.unique_consecutive(ids64 // (128 // width)).numel())
    if pd_path == 1:
        # projected predicate columns whose values the count kept (SEL_KEEP_VALUES=1, within
        # 8 B/row) are copied contiguously from their slots: count x width, not sectors
        kept, budget = set(), 8
        if os.environ.get("SEL_KEEP_VALUES", "0") == "1":
            for j in proj:
                if j in pc and j not in kept and j not in consts and w_all[j] <= budget:
                    kept.add(j)
                    budget -= w_all[j]
        pb_sector = (T.n_rows // 8 + 2 * ((T.n_rows + 1023) // 1024)
                     + len(coded) * (T.n_rows // 8)
                     + sum(local_count * w_all[j] for j in kept)
                     + sum(32 * sectors(w_all[j]) for j in set(proj)
                           if j not in kept and j not in consts and j not in coded)
                     + write_b)
        pb_line = (T.n_rows // 8 + 2 * ((T.n_rows + 1023) // 1024)
                   + len(coded) * (T.n_rows // 8)
                   + sum(local_count * w_all[j] for j in kept)
                   + sum(128 * lines(w_all[j]) for j in set(proj)
                         if j not in kept and j not in consts and j not in coded)
                   + write_b)
    else:
        pb_sector = (T.n_rows * sum(w_all[j] for j in pc)
                     + sum(32 * sectors(w_all[j]) for j in set(proj) if j not in pc) + write_b)
        pb_line = (T.n_rows * sum(w_all[j] for j in pc)
                   + sum(128 * lines(w_all[j]) for j in set(proj) if j not in pc) + write_b)
    roof_count = {"bound": "hbm", "achieved": round(count_gbs, 2), "peak": hbm, "unit": "GB/s",
                  "frac": round(count_gbs / hbm, 4), "traffic": ncu_traffic("count_kernel", args.config, world == 1 and not args.rows),
                  "kernel": "count_kernel", "ms": round(count_k, 4),
                  "algorithmic_bytes_per_launch": int(cb), "peak_source": peak_note}
    push_sector_gbs = pb_sector / (push_k / 1000) / 1e9
    roof_push = {"bound": "hbm", "achieved": round(push_gbs, 2), "peak": hbm, "unit": "GB/s",
                 "frac": round(push_gbs / hbm, 4), "traffic": ncu_traffic(push_name, args.config, world == 1 and not args.rows),
                 "kernel": push_name, "ms": round(push_k, 4),
                 "algorithmic_bytes_per_launch": int(pb), "peak_source": peak_note,
                 "sector_bytes_per_launch": int(pb_sector),
                 "achieved_sector": round(push_sector_gbs, 2),
                 "frac_sector": round(push_sector_gbs / hbm, 4),
                 # the DRAM-granularity floor: every 128-byte line holding a selected row of a
                 # gathered column is fetched whole (ncu: ~90-128 B per scattered 4-byte gather)
                 "line_bytes_per_launch": int(pb_line),
                 "achieved_line": round(pb_line / (push_k / 1000) / 1e9, 2),
                 "frac_line": round(pb_line / (push_k / 1000) / 1e9 / hbm, 4)}
    for r in (roof_count, roof_push):
        r["ms_source"] = ("median of the library's CUDA events around the kernel on its stream, "
                          "over a second pass of the same steps right after the timed region "
                          "(events inside the timed graph would add ~20 us per step)")
    for r in (roof_count, roof_push):   # the same achieved rate against SURVEY §8(d)'s other peaks
        r["frac_nominal_8tbs"] = round(r["achieved"] / 8000.0, 4)
        if read_peak:
            r["frac_read_stream"] = round(r["achieved"] / read_peak, 4)
    roof_dom = roof_push if push_k >= count_k else roof_count
    exchange_ab = None
    if world > 1 and not args.no_xchg_ab:
        exchange_ab = measure_exchange_ab(args, sel, sdist, T, names, proj_names, prog, n, s,
                                          local_count, world, dev, xchg or "")
    other_configs = None
    if args.config == "c2" and not args.rows and not args.no_configs:
        other_configs = measure_configs(["c3", "c5"], args, sel, sdist, world, rank, dev, hbm)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value_gbs, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32/u8 compare, u64 count", "data": "synthetic",
            "config": {"workload": f"{args.config}: {desc}", "global_rows": n,
                       "rows_per_gpu": e - s, "selected": global_count,
                       "parallelism": f"row-shard x{world}",
                       "exchange": xchg,
                       "l2": "inputs larger than L2 (no flush needed)",
                       "step": ("sel_execute = count (keeping the selection) -> device-side gate -> "
                                "materialise" + (", per table.execute()" if prepared is None else
                                                 ", prepared once and replayed as a CUDA graph") +
                                ("" if args.blocking or prepared is None else
                                 "; each step returns when its count is on the host "
                                 "(sel_prepared_execute_async), its materialisation completing "
                                 "in stream order before the next step's count starts"))},
            "rows_per_s": round(n / (ms_per_step / 1000)),
            "step_frac_aggregate_hbm": round(value_gbs / (world * hbm), 4),
            "latency_ms": {"execute_median": round(statistics.median(count_lat), 4),
                           "execute_min": round(min(count_lat), 4),
                           "execute_p99": _stats(count_lat)["p99"],
                           "execute_clock": "host, blocking sel_prepared_execute, call to return",
                           "count_ready": _stats(ready_lat) if ready_lat else None,
                           "count_ready_clock": ("host, each timed step's call to return (at its "
                                                 "count unless --blocking)"),
                           "count_probe": count_probe_stats,
                           "count_kernel": round(count_k, 4), "pushdown_kernels": round(push_k, 4)},
            "roofline": roof_dom,
            "read_stream_gbs": read_peak,
            "read_stream_note": "torch float32 sum over 8 GiB, this run (SURVEY 8(d) peak iii)",
            "roofline_kernels": {"count_kernel": roof_count, push_name: roof_push},
            "pushdown_path": pd_path,
            "clocks": clk.summary(),
            "e2e": e2e,
            # per step: the count and the push-down; on the selection path also the whole-chunk
            # copy (>= 8 Mi local rows) and, when NCCL carries the exchange, the 1-CTA kernel that
            # finishes the result words after its all-gather (else the count's last CTA does;
            # DESIGN.md §5)
            "gpu_launches": ((2 + int((e - s) >= (8 << 20)
                                      and os.environ.get("SEL_DENSE_SPLIT", "1") != "0")
                              + int(bool(xchg) and str(xchg).startswith("nccl")))
                             if pd_path == 1 else 2) * args.steps,
            "cpu_baseline": cpu,
            "exchange_ab": exchange_ab,
            "other_configs": other_configs,
        }
        emit(line)
    if prepared is not None:
        prepared.release()
    table.release()
    if world > 1:
        if ctx.nranks > 1 and xchg and xchg.startswith("peers"):
            ctx.drop_peers()          # every rank unmaps before any rank frees its buffer
        dist.barrier()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


_JSON_FD = None


def emit(line):
    """The bench line, alone on the real stdout (native libraries such as NCCL print banners to
    fd 1; main() points fd 1 at stderr for the run)."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
