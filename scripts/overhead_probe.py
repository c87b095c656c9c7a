"""Fixed per-call cost of the probe (outside the scan): C2-shaped tables of several sizes, host
clock around each call (median of 300) and device time of back-to-back asynchronous counts.
One JSON line per size; a torch launch+sync round trip for reference.

    python scripts/overhead_probe.py [rows ...]
"""
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08384_b200 as sel  # noqa: E402
from selgen import configs, encode  # noqa: E402


def host_ms(fn, reps=300):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    return {"min": round(ts[0], 4), "median": round(statistics.median(ts), 4),
            "p99": round(ts[int(0.99 * (len(ts) - 1))], 4)}


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [60_000, 6_000_000, 75_000_000]
    dev = torch.device("cuda:0")
    x = torch.zeros(1, device=dev)

    def torch_rt():
        x.add_(1)
        torch.cuda.synchronize()
    print(json.dumps({"torch_launch_sync_ms": host_ms(torch_rt)}), flush=True)
    ctx = sel.Context(dev)
    for n in sizes:
        T = configs.gen_c2(n, device=dev)
        t = sel.Table(ctx, ["A", "B", "C", "D"], T.types, [c.data for c in T.columns])
        prog = encode(configs.c2_probes()["listing"], T.types)
        rec = {"rows": n}
        rec["count"] = host_ms(lambda: t.count(prog))
        rec["count_keep"] = host_ms(lambda: t.count(prog, keep_selection=True))
        q = t.prepare_execute(prog, project=["A", "C", "D"], max_size=n)
        rec["prepared_execute"] = host_ms(q.run)
        out = torch.zeros(1, dtype=torch.int64, device=dev)
        for _ in range(20):
            t.count_async(prog, out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(300):
            t.count_async(prog, out)
        b.record()
        torch.cuda.synchronize()
        rec["count_async_device_ms"] = round(a.elapsed_time(b) / 300, 4)
        ctx.enable_timing(True)
        q.run()
        for _ in range(50):
            q.run()
        rec["kernels_ms"] = [round(v, 4) for v in ctx.last_times()]
        ctx.enable_timing(False)
        q.release()
        print(json.dumps(rec), flush=True)
        t.release()
        del T
        torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
