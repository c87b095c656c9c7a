"""Crossover of sel_pushdown's two paths without a kept selection: the single pass
(evaluate + decoupled look-back, mode 0) vs two passes (keeping count, then materialise from the
selection, mode 2), end of call to end of call (host clock, blocking calls), on the worked
example's table and Listing 3.1 at several sizes. Prints one JSON line per size."""
import json
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1806_08384_b200 as sel  # noqa: E402
from selgen import configs, encode  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    ctx = sel.Context(dev)
    sizes = [int(x) for x in (sys.argv[1:] or
             ["60000", "240000", "1020000", "2040000", "4200000", "8400000", "16800000", "67200000", "600000000"])]
    for n in sizes:
        T = configs.gen_c2(n, device=dev)
        t = sel.Table(ctx, ["A", "B", "C", "D"], T.types, [c.data for c in T.columns])
        prog = encode(configs.c2_probes()["listing"], T.types)
        cnt = t.count(prog)
        out = (torch.empty(max(cnt, 1), dtype=torch.int32, device=dev),
               [torch.empty(max(cnt, 1), dtype=c.data.dtype, device=dev) for c in
                (T.columns[j] for j in configs.C2_PROJECT)])
        other = encode(configs.c2_probes()["between_in"], T.types)
        rec = {"rows": n, "selected": cnt}
        for mode in (0, 2):
            ctx.set_pushdown_path(mode)
            ts = []
            for i in range(25):
                t.count(other, keep_selection=True)  # drop the kept selection
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r = t.pushdown(prog, project=["A", "C", "D"], capacity=cnt, out=out)
                ts.append(1000 * (time.perf_counter() - t0))
                assert r.count == cnt and ctx.last_pushdown_path() == mode
            rec[f"mode{mode}_ms"] = round(statistics.median(ts[5:]), 4)
        ctx.set_pushdown_path(-1)
        print(json.dumps(rec), flush=True)
        t.release()
        del T, out
        torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
