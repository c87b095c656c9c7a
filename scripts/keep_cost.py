"""Kernel time of the plain count vs the count keeping the selection on C2-shaped tables of
several sizes (the keep overhead vs size). One JSON line per size."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08384_b200 as sel  # noqa: E402
from selgen import configs, encode  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    ctx = sel.Context(dev)
    ctx.enable_timing(True)
    for n in [int(x) for x in (sys.argv[1:] or ["75000000", "150000000", "600000000"])]:
        T = configs.gen_c2(n, device=dev)
        t = sel.Table(ctx, ["A", "B", "C", "D"], T.types, [c.data for c in T.columns])
        prog = encode(configs.c2_probes()["listing"], T.types)

        def med(f, reps=30):
            xs = []
            for i in range(reps + 3):
                f()
                if i >= 3:
                    xs.append(ctx.last_times()[0])
            return round(statistics.median(xs), 4)
        rec = {"rows": n, "plain_ms": med(lambda: t.count(prog)),
               "keep_ms": med(lambda: t.count(prog, keep_selection=True))}
        print(json.dumps(rec), flush=True)
        t.release()
        del T
        torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
