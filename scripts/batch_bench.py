"""Kernel time of sel_count_batch (NEXT(2)) on the worked example: the four leaves of Listing 3.1
and their conjunction in one scan, vs five separate counts. Prints one JSON line."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08384_b200 as sel  # noqa: E402
from selgen import configs, encode  # noqa: E402
from selgen.program import Cmp, In, And  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    T = configs.gen_c2(device=dev)
    ctx = sel.Context(dev)
    t = sel.Table(ctx, ["A", "B", "C", "D"], T.types, [c.data for c in T.columns])
    leaves = [Cmp("=", 0, 2), Cmp("<", 1, 2001), Cmp(">", 1, 1000), In(2, (1, 4))]
    progs = [encode(x, T.types) for x in leaves] + [encode(configs.c2_probes()["listing"], T.types)]
    ctx.enable_timing(True)
    def med(f, reps=20):
        xs = []
        for i in range(reps + 3):
            f()
            if i >= 3:
                xs.append(ctx.last_kernel_ms())
        return statistics.median(xs)
    batch = med(lambda: t.count_batch(progs))
    singles = [med(lambda p=p: t.count(p)) for p in progs]
    n = T.n_rows
    print(json.dumps({"batch_ms": round(batch, 4), "batch_gbs": round(n * 9 / batch / 1e6, 1),
                      "singles_ms": [round(x, 4) for x in singles], "singles_sum_ms": round(sum(singles), 4),
                      "counts": t.count_batch(progs)}))


if __name__ == "__main__":
    main()
