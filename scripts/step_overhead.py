"""Fixed per-step overhead of a prepared Execute (graph launch + sync): C2-shaped tables of several
sizes, timing events on and off, CUDA-event time over 200 back-to-back steps. One JSON line per
size."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08384_b200 as sel  # noqa: E402
from selgen import configs, encode  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    ctx = sel.Context(dev)
    for n in [60_000, 6_000_000, 75_000_000]:
        T = configs.gen_c2(n, device=dev)
        t = sel.Table(ctx, ["A", "B", "C", "D"], T.types, [c.data for c in T.columns])
        prog = encode(configs.c2_probes()["listing"], T.types)
        rec = {"rows": n}
        for timing in (True, False):
            ctx.enable_timing(timing)
            q = t.prepare_execute(prog, project=["A", "C", "D"], max_size=n)
            for _ in range(20):
                q.run()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            t0 = time.perf_counter()
            for _ in range(200):
                q.run()
            b.record()
            torch.cuda.synchronize()
            rec[f"timing{int(timing)}_ms"] = round(a.elapsed_time(b) / 200, 4)
            rec[f"timing{int(timing)}_host_ms"] = round((time.perf_counter() - t0) / 200 * 1000, 4)
            if timing:
                rec["kernels_ms"] = [round(x, 4) for x in ctx.last_times()]
            q.release()
        print(json.dumps(rec), flush=True)
        t.release()
    ctx.close()


if __name__ == "__main__":
    main()
