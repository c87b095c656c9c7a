"""Coded projection at dense selections: 600M rows, x = i (INT32), z in {1, 4}
(DICT8) on every row; Execute(x < t AND z IN (1, 4)) projecting z and x, selectivity t / N.
Median execute() time over 20 calls; run with SEL_DENSE_SPLIT=0 and =1 to compare the
whole-chunk copy against staging every row. One JSON line per selectivity."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08384_b200 as sel  # noqa: E402
from paper_1806_08384_b200 import col  # noqa: E402

N = int(os.environ.get("ROWS", 600_000_000))
ctx = sel.Context()
dev = ctx.device
g = torch.Generator(device=dev).manual_seed(7)
x = torch.arange(N, dtype=torch.int32, device=dev)
z = (torch.randint(0, 2, (N,), device=dev, generator=g, dtype=torch.uint8) * 3 + 1)
t = sel.Table.from_tensors(ctx, {"x": x, "z": z})
for s in (0.1, 0.5, 1.0):
    pred = (col("x") < int(s * N)) & col("z").isin([1, 4])
    r = t.execute(pred, project=["z", "x"], max_size=N)
    assert r.count == int(s * N)
    zz = r.columns["z"]
    ok = bool(torch.equal(zz[:1_000_000].to(torch.uint8), z[:1_000_000]))
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        t.execute(pred, project=["z", "x"], max_size=N)
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps({"rows": N, "s": s, "dense_split": os.environ.get("SEL_DENSE_SPLIT", "1"),
                      "coded": os.environ.get("SEL_CODED", "1"), "z_prefix_ok": ok,
                      "execute_ms_median": round(statistics.median(ts), 4)}), flush=True)
