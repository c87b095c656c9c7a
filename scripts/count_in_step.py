"""Why the keeping count inside an Execute is slower than alone: the count
kernel's time (library CUDA events) at one C2-shaped size under each condition — plain count,
keeping count, the count of an Execute (keeping the selection and C's code bits, finishing the
result words), the same with coded projections off, and the plain/keeping count right after a
256 MB device write (dirty L2 lines, like the previous Execute's output). One JSON line."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08384_b200 as sel  # noqa: E402
from selgen import configs, encode  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 75_000_000
    dev = torch.device("cuda:0")
    ctx = sel.Context(dev)
    T = configs.gen_c2(n, device=dev)
    t = sel.Table(ctx, ["A", "B", "C", "D"], T.types, [c.data for c in T.columns])
    prog = encode(configs.c2_probes()["listing"], T.types)
    junk = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    ctx.enable_timing(True)

    def med(f, dirty=False, idx=0, reps=30):
        xs = []
        for i in range(reps + 3):
            if dirty:
                junk.fill_(i)
            f()
            if i >= 3:
                xs.append(ctx.last_times()[idx])
        return round(statistics.median(xs), 4)

    ex = lambda: t.execute(prog, project=["A", "C", "D"], max_size=n)
    rec = {"rows": n,
           "plain": med(lambda: t.count(prog)),
           "keep": med(lambda: t.count(prog, keep_selection=True)),
           "execute_count": med(ex),
           "execute_pushdown": med(ex, idx=1),
           "plain_after_write": med(lambda: t.count(prog), dirty=True),
           "keep_after_write": med(lambda: t.count(prog, keep_selection=True), dirty=True),
           "execute_count_after_write": med(ex, dirty=True)}
    rec["keep_after_pushdown"] = med(lambda: (t.pushdown(prog, project=["A", "C", "D"], capacity=n),
                                              t.count(prog, keep_selection=True)))
    rec["execute_gated_count"] = med(lambda: t.execute(prog, project=["A", "C", "D"], max_size=0,
                                                       capacity=1))
    ctx.set_option("dense_split", 0)
    rec["execute_count_no_dense"] = med(ex)
    ctx.set_option("dense_split", 1)
    ctx.set_option("coded", 0)
    rec["execute_count_uncoded"] = med(ex)
    rec["execute_pushdown_uncoded"] = med(ex, idx=1)
    print(json.dumps(rec), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
