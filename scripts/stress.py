"""Randomised GPU-vs-oracle stress (not part of the suite): random tables (types, sizes up to 2M
rows, boundary-heavy values) x random programs (interpreter trees and fast-path conjunctions) x
every path (count, execute, push-down modes 0/1/2 with coded/constant projections, prepared
execute, sampled and batch counts), for SECONDS seconds. Prints a summary; exits 1 on the first
mismatch with the case."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
import paper_1806_08384_b200 as sel  # noqa: E402
from selgen.program import random_program, encode, INT32, INT64, FLOAT32, DATE32, DICT8, DICT16, DICT32  # noqa: E402
from helpers import random_table  # noqa: E402
from test_gpu_fastpath import fast_conjunction, TYPES as FT  # noqa: E402

VIEW = {INT32: np.int32, INT64: np.int64, FLOAT32: np.float32, DATE32: np.int32, DICT8: np.uint8,
        DICT16: np.int16, DICT32: np.int32}


def main():
    secs = float(os.environ.get("SECONDS_BUDGET", "240"))
    dev = torch.device("cuda:0")
    ctx = sel.Context(dev)
    rng = np.random.default_rng(int(os.environ.get("SEED", "7")))
    t0, cases = time.time(), 0
    while time.time() - t0 < secs:
        fast = rng.random() < 0.5
        types = FT if fast else [list(VIEW)[int(i)] for i in rng.integers(0, 7, int(rng.integers(1, 5)))]
        n = int(rng.choice([1, 1023, 1025, 4097, 65537, 300_001, 2_000_003]))
        cols, pools = random_table(rng, types, n)
        tens = [torch.from_numpy(np.ascontiguousarray(c).view(VIEW[t]).copy()).to(dev) for c, t in zip(cols, types)]
        t = sel.Table(ctx, [f"c{i}" for i in range(len(types))], types, tens)
        for _ in range(4):
            node = fast_conjunction(rng, pools) if fast else random_program(rng, types, pools, max_depth=3)
            prog = encode(node, types)
            proj = sorted(set(int(x) for x in rng.integers(0, len(types), 2)))
            wc, wids, wcols = oracle.pushdown(cols, types, prog, proj=proj)
            def check(tag, r):
                if r.count != wc or not np.array_equal(r.rowids.cpu().numpy().view(np.uint32), wids):
                    raise AssertionError((tag, n, types, node, r.count, wc))
                for j, c in enumerate(proj):
                    got = r.columns[c].cpu().numpy().view(wcols[j].dtype)
                    if not np.array_equal(got, wcols[j]):
                        raise AssertionError((tag, "col", c, n, types, node))
            assert t.count(prog) == wc, ("count", n, types, node)
            check("execute", t.execute(prog, project=proj, max_size=n))
            for mode in (0, 2, -1):
                ctx.set_pushdown_path(mode)
                t.count(encode(random_program(rng, types, pools, max_depth=1), types), keep_selection=True)
                check(f"pushdown{mode}", t.pushdown(prog, project=proj, capacity=max(wc, 1)))
            ctx.set_pushdown_path(-1)
            check("pushdown-kept", t.pushdown(prog, project=proj, capacity=max(wc, 1)))
            q = t.prepare_execute(prog, project=proj, max_size=n)
            q.run()
            check("prepared", q.result())
            assert q.run(wait=False) == wc, ("prepared-async", n, types, node)
            torch.cuda.synchronize()
            check("prepared-async", q.result())
            q.release()
            b = t.count_batch([prog, encode(random_program(rng, types, pools, max_depth=2), types)])
            assert b[0] == wc, ("batch", n, types, node)
            cases += 1
        t.release()
    print(f"stress ok: {cases} cases in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
