"""BASELINE.json config 5: the selectivity sweep 1e-6 .. 1.0 on the 1e9-row table, count vs
push-down compaction cost, scattered (x = (a i + b) mod N) and clustered (x = i)
layouts. Per selectivity: the Execute step (count keeping the selection -> materialise ids + y),
the kernel times, and the closed-form count check (count(x < t) = t). One JSON line per point.
Env: ROWS, SWEEP_LAYOUTS="scattered,clustered", SWEEP_S="1e-6,...,1.0", SWEEP_EAGER=1 (execute()
calls instead of the prepared graph, for ncu: scripts/profile.sh notes why)."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08384_b200 as sel  # noqa: E402
from selgen import configs, encode  # noqa: E402


class _Eager:
    """The prepared execute's run()/release() through plain execute() calls."""

    def __init__(self, t, prog, n, out):
        self.t, self.prog, self.n, self.out = t, prog, n, out

    def run(self):
        return self.t.execute(self.prog, project=["y"], max_size=self.n, capacity=self.n,
                              out=self.out).count

    def release(self):
        pass


def main():
    dev = torch.device("cuda:0")
    n = int(os.environ.get("ROWS", configs.C5_ROWS))
    ctx = sel.Context(dev)
    layouts = os.environ.get("SWEEP_LAYOUTS", "scattered,clustered").split(",")
    sels = [float(x) for x in os.environ.get("SWEEP_S", "1e-6,1e-5,1e-4,1e-3,1e-2,0.1,0.5,1.0").split(",")]
    eager = os.environ.get("SWEEP_EAGER") == "1"
    for layout in layouts:
        T = configs.gen_sweep(n, device=dev, layout=layout)
        t = sel.Table(ctx, ["x", "y"], T.types, [c.data for c in T.columns])
        out_ids = torch.empty(n, dtype=torch.int32, device=dev)
        out_y = torch.empty(n, dtype=torch.int32, device=dev)
        for s in sels:
            thr = configs.sweep_threshold(n, s)
            prog = encode(configs.sweep_probe(thr), T.types)
            if eager:
                q = _Eager(t, prog, n, (out_ids, [out_y]))
            else:
                q = t.prepare_execute(prog, project=["y"], max_size=n, capacity=n,
                                      out=(out_ids, [out_y]))
            for _ in range(3):
                q.run()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                c = q.run()
            b.record()
            torch.cuda.synchronize()
            step = a.elapsed_time(b) / 10
            ctx.enable_timing(True)
            ks = []
            for _ in range(5):
                q.run()
                ks.append(ctx.last_times())
            ctx.enable_timing(False)
            q.release()
            cm = statistics.median(k[0] for k in ks)
            pm = statistics.median(k[1] for k in ks)
            assert c == thr, (layout, s, c, thr)
            print(json.dumps({"layout": layout, "selectivity": s, "selected": c,
                              "step_ms": round(step, 4), "count_ms": round(cm, 4),
                              "pushdown_ms": round(pm, 4),
                              "count_gbs": round(4 * n / cm / 1e6, 1)}), flush=True)
        t.release()
        del T
        torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
