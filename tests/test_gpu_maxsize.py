"""Maximum sizes (row ids are uint32, tables of >= 2^32 rows are rejected):
a single-GPU table of 2^32 - 1 rows (a 1-byte column, 4 GB) and a shard whose global row ids end
at 2^32 - 2. Expected values are closed forms (the positions are planted), so no oracle pass over
4 billion rows is needed; counts above 2^31 check the 64-bit count path."""

import numpy as np
import pytest
import torch

import oracle
import paper_1806_08384_b200 as sel
from selgen.program import Cmp, Not, And, encode, DICT8, INT32

pytestmark = pytest.mark.gpu

N_MAX = (1 << 32) - 1
PLANTED = [0, 1023, 1024, (1 << 31) - 1, 1 << 31, (1 << 32) - 1025, (1 << 32) - 1024, N_MAX - 1]


@pytest.fixture(scope="module")
def ctx(cuda_device):
    c = sel.Context(cuda_device)
    yield c
    c.close()


def test_table_of_2_pow_32_minus_1_rows(ctx):
    dev = ctx.device
    x = torch.zeros(N_MAX, dtype=torch.uint8, device=dev)
    x[torch.tensor(PLANTED, dtype=torch.int64, device=dev)] = 7
    t = sel.Table(ctx, ["x"], [DICT8], [x])
    hit = encode(Cmp("=", 0, 7), [DICT8])
    miss = encode(Not(Cmp("=", 0, 7)), [DICT8])
    assert t.count(hit) == len(PLANTED)
    assert t.count(miss) == N_MAX - len(PLANTED)              # > 2^31: the 64-bit count
    want = np.array(PLANTED, dtype=np.uint32)
    for mode in (-1, 0, 2):                                   # automatic, single pass, two passes
        ctx.set_pushdown_path(mode)
        try:
            res = t.pushdown(hit, project=["x"], capacity=len(PLANTED))
        finally:
            ctx.set_pushdown_path(-1)
        assert res.count == len(PLANTED)
        np.testing.assert_array_equal(res.rowids.cpu().numpy().view(np.uint32), want)
        assert bool((res.columns["x"] == 7).all())
    r = t.execute(hit, project=["x"], max_size=len(PLANTED))
    assert r.materialized
    np.testing.assert_array_equal(r.rowids.cpu().numpy().view(np.uint32), want)
    # a huge selection against a small capacity: exact count, first rows written, gated execute
    res = t.pushdown(miss, project=["x"], capacity=4)
    assert res.count == N_MAX - len(PLANTED) and res.gated
    np.testing.assert_array_equal(res.rowids[:4].cpu().numpy().view(np.uint32), [1, 2, 3, 4])
    g = t.execute(miss, project=["x"], max_size=1000, capacity=4)
    assert not g.materialized and g.count == N_MAX - len(PLANTED)
    # the block sample covers the last (ragged) chunk
    nchunks = (N_MAX + 1023) // 1024
    cnt, rows, _ = t.count_sampled(hit, nchunks - 1, 0)
    assert rows == 1024 + (N_MAX - (nchunks - 1) * 1024)      # chunks 0 and nchunks-1
    assert cnt == sum(1 for p in PLANTED if p < 1024 or p >= (nchunks - 1) * 1024)
    t.release()
    del x
    torch.cuda.empty_cache()
    with pytest.raises(sel.SelError):
        sel.Table(ctx, ["x"], [DICT8], [torch.zeros(16, dtype=torch.uint8, device=dev)],
                  global_rows=1 << 32)


def test_shard_ending_at_the_last_row_id(ctx):
    """A rank's shard whose global ids run up to 2^32 - 2 (global N = 2^32 - 1)."""
    rng = np.random.default_rng(32)
    n = 5000
    off = N_MAX - n
    v = rng.integers(-5, 5, n).astype(np.int32)
    t = sel.Table(ctx, ["v"], [INT32], [torch.from_numpy(v).to(ctx.device)], row_offset=off,
                  global_rows=N_MAX)
    for node in [Cmp(">", 0, 2), And(Cmp(">=", 0, -5), Cmp("<", 0, 0)), Cmp("=", 0, 4)]:
        prog = encode(node, [INT32])
        want_c, want_ids, _ = oracle.pushdown([v], [INT32], prog, row_offset=off)
        for mode in (0, 2):
            ctx.set_pushdown_path(mode)
            try:
                res = t.pushdown(prog, project=["v"])
            finally:
                ctx.set_pushdown_path(-1)
            assert res.count == want_c
            got = res.rowids.cpu().numpy().view(np.uint32)
            np.testing.assert_array_equal(got, want_ids)
            assert int(got.max()) <= N_MAX - 1
    t.release()
