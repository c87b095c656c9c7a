"""Kernel times of the count probe variants on one workload (DESIGN.md §5 A/B): plain count,
count keeping the selection, count keeping the selection + projected predicate values, and the
push-down from the kept selection. Environment knobs (SEL_FAST, SEL_PREFETCH, SEL_CTAS_PER_SM, ...)
apply. Usage: python scripts/count_variants.py c2 [reps]"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1806_08384_b200 as sel  # noqa: E402
from selgen import encode  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    dev = torch.device("cuda:0")
    n, gen, node, proj, desc = bench.workload(cfg, 0)
    T = gen(0, n, dev)
    ctx = sel.Context(dev)
    names = [c.name for c in T.columns]
    t = sel.Table(ctx, names, T.types, [c.data for c in T.columns])
    prog = encode(node, T.types)
    pn = [names[j] for j in proj]
    ctx.enable_timing(True)
    out = {"config": cfg, "env": {k: v for k, v in os.environ.items() if k.startswith("SEL_")}}
    def med(f):
        xs = []
        for i in range(reps + 3):
            f()
            if i >= 3:
                xs.append(ctx.last_times())
        return [round(statistics.median(x[j] for x in xs), 4) for j in (0, 1)]
    out["plain_count_ms"] = med(lambda: t.count(prog))[0]
    out["keep_sel_count_ms"] = med(lambda: t.count(prog, keep_selection=True))[0]
    out["keep_vals_count_ms"] = med(lambda: t.count(prog, keep_selection=True, keep_columns=pn))[0]
    cnt = t.count(prog)
    o = (torch.empty(max(cnt, 1), dtype=torch.int32, device=dev),
         [torch.empty(max(cnt, 1), dtype=T.columns[j].data.dtype, device=dev) for j in proj])
    def pd():
        t.count(prog, keep_selection=True, keep_columns=pn)
        t.pushdown(prog, project=pn, capacity=cnt, out=o)
    out["pushdown_from_kept_vals_ms"] = med(pd)[1]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
