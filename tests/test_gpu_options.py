"""Every tuning switch of sel_ctx_set_option (include/sel.h) against the CPU oracle: none of them
may change a result (counts, ascending row ids and gathered values are unique), only
which kernel variant or launch shape produces it. Each non-default setting runs, on a fresh
context, random programs on a ragged table through every materialisation path, the worked
example (C2's coded projection) through Execute and a prepared Execute, and a
clustered table large enough for the whole-chunk copy (>= 8 Mi rows)."""

import numpy as np
import pytest

import oracle
import paper_1806_08384_b200 as sel
from selgen import configs
from selgen.program import Cmp, And, encode, random_program, INT32, INT64, FLOAT32, DICT8, DICT16

from helpers import random_table
from test_gpu_parity import check_parity, register

pytestmark = pytest.mark.gpu

SETTINGS = [("fast", 0), ("coded", 0), ("dense_split", 0), ("keep_values", 1), ("prefetch", 1),
            ("prefetch", 0), ("count_warps", 8), ("ctas_per_sm", 1), ("ctas_per_sm", 2),
            ("two_pass_min_rows", 0), ("graph_comm", 0)]


def _execute_parity(t, cols, types, prog, proj):
    want_c, want_ids, want_cols = oracle.pushdown(cols, types, prog, proj=proj)
    for r in (t.execute(prog, project=proj, max_size=t.local_rows), None):
        if r is None:
            q = t.prepare_execute(prog, project=proj, max_size=t.local_rows)
            assert q.run() == want_c
            r = q.result()
        assert r.count == want_c and r.materialized
        np.testing.assert_array_equal(r.rowids.cpu().numpy().view(np.uint32), want_ids)
        for j, c in enumerate(proj):
            np.testing.assert_array_equal(r.columns[c].cpu().numpy().view(want_cols[j].dtype),
                                          want_cols[j])
    q.release()


@pytest.mark.parametrize("name,value", SETTINGS)
def test_option_keeps_results(cuda_device, name, value):
    ctx = sel.Context(cuda_device)
    try:
        ctx.set_option(name, value)
        rng = np.random.default_rng(abs(hash((name, value))) % (1 << 32))
        types = [INT32, DICT8, INT64, FLOAT32, DICT16]
        cols, pools = random_table(rng, types, 70_001)
        t = register(ctx, cols, types)
        for _ in range(12):
            check_parity(t, cols, types, random_program(rng, types, pools, max_depth=4),
                         proj=[0, 1, 2, 3, 4])
        t.release()
        T = configs.gen_c2(600_000)
        c2 = [c.numpy() for c in T.columns]
        t2 = register(ctx, c2, T.types)
        _execute_parity(t2, c2, T.types, encode(configs.c2_probes()["listing"], T.types),
                        configs.C2_PROJECT)
        t2.release()
        n = 9 * (1 << 20) + 333
        x = np.arange(n, dtype=np.int32)
        y = (np.arange(n) % 3).astype(np.uint8)
        t3 = register(ctx, [x, y], [INT32, DICT8])
        for node in (Cmp("<", 0, 6_000_000), And(Cmp(">=", 0, 1000), Cmp("<", 1, 2))):
            _execute_parity(t3, [x, y], [INT32, DICT8], encode(node, [INT32, DICT8]), [0, 1])
        t3.release()
    finally:
        ctx.close()


def test_option_errors(cuda_device):
    ctx = sel.Context(cuda_device)
    try:
        for name, value in [("nope", 1), ("fast", 2), ("prefetch", 3), ("count_warps", 4),
                            ("ctas_per_sm", -1), ("two_pass_min_rows", -5)]:
            with pytest.raises(sel.SelError) as e:
                ctx.set_option(name, value)
            assert e.value.status == 1, (name, value)
        ctx.set_pushdown_path(0)                 # forced single pass: the threshold is ignored
        ctx.set_option("two_pass_min_rows", 0)
        ctx.set_pushdown_path(-1)
    finally:
        ctx.close()
