"""NEXT(4) baselines beside the exact probe: on the worked example's 600M-row R,
the exact count, the block-sampled count estimate and the equi-depth histogram estimate, with
their times (host clock around the blocking calls). One JSON line."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08384_b200 as sel  # noqa: E402
from selgen import configs, encode  # noqa: E402
from selgen.program import Cmp  # noqa: E402


def timed(f, reps=5):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = f()
    return r, (time.perf_counter() - t0) / reps * 1000


def main():
    dev = torch.device("cuda:0")
    T = configs.gen_c2(device=dev)
    ctx = sel.Context(dev)
    t = sel.Table(ctx, ["A", "B", "C", "D"], T.types, [c.data for c in T.columns])
    out = {}
    prog = encode(configs.c2_probes()["listing"], T.types)
    out["listing_exact"], out["listing_exact_ms"] = timed(lambda: t.count(prog))
    for stride in (16, 256):
        (c, rows, est), ms = timed(lambda s=stride: t.count_sampled(prog, s, 0))
        out[f"listing_sampled_1_in_{stride}"] = round(est)
        out[f"listing_sampled_1_in_{stride}_ms"] = round(ms, 3)
    x = 1500
    eq = encode(Cmp("=", 1, x), T.types)
    out["B_eq_exact"], out["B_eq_exact_ms"] = timed(lambda: t.count(eq))
    for stride, B in ((1, 256), (16, 256), (256, 64)):
        h, ms = timed(lambda s=stride, b=B: t.histogram("B", buckets=b, stride=s), reps=3)
        out[f"B_eq_equidepth_{B}b_1_in_{stride}"] = round(sel.equi_depth_estimate(h, x))
        out[f"B_eq_equidepth_{B}b_1_in_{stride}_build_ms"] = round(ms, 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
