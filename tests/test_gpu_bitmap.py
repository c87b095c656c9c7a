"""GPU parity of IN_BITMAP leaves: `col IN <registered key set>` evaluated
in the sm_100a kernels vs the CPU oracle, element by element, under AND/OR/NOT with every other
leaf kind, on ragged sizes, through count, every push-down path and execute; plus the registry's
error behaviour (include/sel.h sel_bitmap_register / sel_bitmap_release)."""

import numpy as np
import pytest
import torch

import oracle
import paper_1806_08384_b200 as sel
from selgen.program import (Cmp, Between, InSet, And, Or, Not, encode, random_program, INT32,
                            INT64, FLOAT32, DATE32, DICT8, DICT16, DICT32)

from helpers import random_table, random_bitmaps, make_bitmap
from test_gpu_parity import register

pytestmark = pytest.mark.gpu

SIZES = [1, 1023, 1025, 8192 + 17, 70001]


@pytest.fixture(scope="module")
def bctx(cuda_device):
    c = sel.Context(cuda_device)
    yield c
    c.close()


def upload(ctx, bitmaps):
    """Register the key sets in order on a context without other sets: ids = positions."""
    ids = []
    for words, nbits in bitmaps:
        w = torch.from_numpy(words.view(np.int64).copy()).to(ctx.device)
        ids.append(ctx.register_bitmap(w, nbits))
    return ids


def release(ctx, ids):
    for i in ids:
        ctx.release_bitmap(i)


def _table(rng, types, n):
    cols, pools = random_table(rng, types, n)
    for c, t in enumerate(types):   # small non-negative values so that the key sets hit rows
        if t != FLOAT32 and n:
            small = rng.integers(0, 256 if t == DICT8 else 1100, n)
            cols[c] = np.where(rng.random(n) < 0.5, small.astype(cols[c].dtype), cols[c])
    return cols, pools


def parity(table, cols, types, node, bms, proj):
    prog = encode(node, types)
    want_count, want_ids, want_cols = oracle.pushdown(cols, types, prog, proj=proj, bitmaps=bms)
    assert table.count(prog) == want_count, node
    for mode in ("kept", "sel", "single"):
        if mode == "kept":
            assert table.count(prog, keep_selection=True, keep_columns=proj) == want_count
        elif mode == "sel":
            assert table.count(prog, keep_selection=True) == want_count
        else:
            table.count(encode(Cmp("=", 0, 0) if types[0] != FLOAT32 else Cmp("=", 0, 0.0), types),
                        keep_selection=True)   # replace the kept selection by another program's
        res = table.pushdown(prog, project=proj, capacity=want_count)
        assert res.count == want_count, (mode, node)
        np.testing.assert_array_equal(res.rowids.cpu().numpy().view(np.uint32), want_ids,
                                      err_msg=f"{mode} {node}")
        for j, c in enumerate(proj):
            got = res.columns[c].cpu().numpy().view(want_cols[j].dtype)
            np.testing.assert_array_equal(got, want_cols[j], err_msg=f"{mode} col {c}")
    return want_count


@pytest.mark.parametrize("n", SIZES)
def test_bitmap_random_programs_ragged(bctx, n):
    types = [INT32, DICT8, INT64, DICT16, DATE32, DICT32, FLOAT32]
    rng = np.random.default_rng(1000 + n)
    cols, pools = _table(rng, types, n)
    bms = random_bitmaps(rng, pools)
    ids = upload(bctx, bms)
    assert ids == list(range(len(bms)))
    try:
        t = register(bctx, cols, types)
        nonempty = 0
        for trial in range(25):
            node = random_program(rng, types, pools, max_depth=3, n_bitmaps=len(bms))
            proj = sorted({int(x) for x in rng.integers(0, len(types), 2)})
            c = parity(t, cols, types, node, bms, proj)
            nonempty += 0 < c < n
        if n > 1000:
            assert nonempty > 3
        t.release()
    finally:
        release(bctx, ids)


def test_bitmap_boundaries_every_width(bctx):
    """v = nbits-1 / nbits / negative values and NOT on 1-, 2-, 4- and 8-byte columns."""
    n = 5000
    rng = np.random.default_rng(5)
    nbits = 300
    keys = sorted(set(int(k) for k in rng.integers(0, nbits, 120)) | {0, 63, 64, nbits - 1})
    bms = [make_bitmap(keys, nbits)]
    ids = upload(bctx, bms)
    try:
        vals = np.array([-1, 0, 63, 64, nbits - 1, nbits, nbits + 1, 255], dtype=np.int64)
        types = [DICT8, DICT16, INT32, INT64]
        cols = [rng.choice(vals[vals >= 0], n).astype(np.uint8),
                rng.choice(np.r_[vals[vals >= 0], 65535], n).astype(np.uint16),
                rng.choice(np.r_[vals, -2**31], n).astype(np.int32),
                rng.choice(np.r_[vals, -2**63, 2**40], n).astype(np.int64)]
        t = register(bctx, cols, types)
        for c in range(4):
            for node in (InSet(c, ids[0]), Not(InSet(c, ids[0])),
                         And(InSet(c, ids[0]), Cmp(">", c, 0)),
                         Or(Not(InSet(c, ids[0])), Cmp("=", c, 64))):
                parity(t, cols, types, node, bms, [c])
        t.release()
    finally:
        release(bctx, ids)


def test_bitmap_registry_errors(bctx):
    n = 4096
    x = np.arange(n, dtype=np.int32)
    t = register(bctx, [x], [INT32])
    w = torch.zeros(4, dtype=torch.int64, device=bctx.device)
    w[0] = 0b1011
    i = bctx.register_bitmap(w, 256)
    prog = encode(InSet(0, i), [INT32])
    assert t.count(prog) == 3
    with pytest.raises(sel.SelError) as e:          # unregistered id
        t.count(encode(InSet(0, i + 7), [INT32]))
    assert e.value.status == 1
    with pytest.raises(sel.SelError) as e:          # IN_BITMAP leaves are not batched
        t.count_batch([prog, encode(Cmp("<", 0, 5), [INT32])])
    assert e.value.status == 1
    big = torch.zeros(8, dtype=torch.int64, device=bctx.device)
    with pytest.raises(sel.SelError) as e:          # 16-byte alignment
        bctx.register_bitmap(big[1:], 64)
    assert e.value.status == 2
    with pytest.raises(sel.SelError) as e:          # nbits = 0
        bctx.register_bitmap(big, 0)
    assert e.value.status == 1
    # re-registering under a released id uses the new set (no stale kept selection)
    assert t.count(prog, keep_selection=True) == 3
    bctx.release_bitmap(i)
    with pytest.raises(sel.SelError):
        t.count(prog)
    w2 = torch.zeros(4, dtype=torch.int64, device=bctx.device)
    w2[1] = 1                                        # key 64 only
    j = bctx.register_bitmap(w2, 256)
    assert j == i
    r = t.pushdown(prog, capacity=16)
    assert r.count == 1 and r.rowids.cpu().numpy().view(np.uint32).tolist() == [64]
    with pytest.raises(sel.SelError):
        bctx.release_bitmap(j + 100)
    bctx.release_bitmap(j)
    t.release()


def test_bitmap_star_join_semijoin(bctx):
    """The SSB-style use: a fact table's foreign key filtered by the key set
    of a dimension predicate, AND a date range, executed with Algorithm 1's gate."""
    rng = np.random.default_rng(77)
    n, ndim = 3_000_000, 30_000
    custkey = rng.integers(0, ndim, n).astype(np.uint32)        # DICT32 foreign key
    orderdate = rng.integers(19920101, 19981231, n).astype(np.int32)
    revenue = rng.integers(0, 10**7, n).astype(np.int64)
    region = rng.integers(0, 5, ndim)                            # dimension attribute
    bms = [make_bitmap(np.flatnonzero(region == 2), ndim)]
    ids = upload(bctx, bms)
    try:
        types = [DICT32, DATE32, INT64]
        cols = [custkey, orderdate, revenue]
        t = register(bctx, cols, types)
        node = And(InSet(0, ids[0]), Between(1, 19940101, 19941231))
        prog = encode(node, types)
        want = oracle.count(cols, types, prog, bitmaps=bms)
        assert want == int((np.isin(custkey, np.flatnonzero(region == 2)) &
                            (orderdate >= 19940101) & (orderdate <= 19941231)).sum())
        assert t.count(prog) == want
        res = t.execute(prog, project=[0, 2], max_size=want)
        assert res.materialized and res.count == want
        c, ids_w, cols_w = oracle.pushdown(cols, types, prog, proj=[0, 2], bitmaps=bms)
        np.testing.assert_array_equal(res.rowids.cpu().numpy().view(np.uint32), ids_w)
        np.testing.assert_array_equal(res.columns[2].cpu().numpy(), cols_w[1])
        gated = t.execute(prog, project=[0, 2], max_size=want - 1)
        assert not gated.materialized and gated.count == want
        t.release()
    finally:
        release(bctx, ids)


def test_bitmap_staged_and_global_sets_together(bctx):
    """A key set too large for the count kernel's shared memory (2^21 bits = 256 KB, looked up in
    global memory) beside small staged ones, in one program, with kept values competing for the
    same shared memory; also through the block-sampled count."""
    n = 200_000
    rng = np.random.default_rng(21)
    big_n = 1 << 21
    a = rng.integers(0, big_n + 5000, n).astype(np.int32)
    b = rng.integers(0, 70_000, n).astype(np.uint32)
    c = rng.integers(0, 256, n).astype(np.uint8)
    big = make_bitmap(np.flatnonzero(rng.random(big_n) < 0.3), big_n)
    small = make_bitmap(np.flatnonzero(rng.random(70_000) < 0.5), 70_000)
    tiny = make_bitmap(range(0, 256, 3), 256)
    bms = [big, small, tiny]
    ids = upload(bctx, bms)
    assert ids == [0, 1, 2]
    try:
        types = [INT32, DICT32, DICT8]
        cols = [a, b, c]
        t = register(bctx, cols, types)
        for node in (And(InSet(0, 0), InSet(1, 1)),
                     Or(And(InSet(0, 0), Not(InSet(2, 2))), InSet(1, 1)),
                     And(Not(InSet(0, 0)), And(InSet(1, 1), InSet(2, 2)))):
            parity(t, cols, types, node, bms, [0, 1, 2])
            prog = encode(node, types)
            got, rows, _ = t.count_sampled(prog, 3, 1)
            chunk = np.arange(n) // 1024
            keep = (chunk % 3) == 1
            assert rows == int(keep.sum())
            assert got == oracle.count([x[keep] for x in cols], types, prog, bitmaps=bms)
        t.release()
    finally:
        release(bctx, ids)


def test_bitmap_large_staged_set_32_warp_count(bctx):
    """A staged key set large enough (150 KB) that only one CTA fits per SM: the count runs
    32-warp CTAs (pick_count_warps). Plain count, keeping count (kept values yield to the set),
    execute, prepared execute and the block-sampled count all match the oracle; ragged size."""
    n = 1_000_003
    rng = np.random.default_rng(33)
    nb = 1_200_000
    k = rng.integers(0, nb + 1000, n).astype(np.int32)
    s = rng.integers(0, 40_000, n).astype(np.int32)
    v = rng.integers(-10**6, 10**6, n).astype(np.int64)
    bms = [make_bitmap(np.flatnonzero(rng.random(nb) < 0.04), nb),
           make_bitmap(np.flatnonzero(rng.random(40_000) < 0.2), 40_000)]
    ids = upload(bctx, bms)
    assert ids == [0, 1]
    try:
        types = [INT32, INT32, INT64]
        cols = [k, s, v]
        t = register(bctx, cols, types)
        for node in (And(InSet(0, 0), InSet(1, 1)), Or(InSet(0, 0), Not(InSet(1, 1))),
                     And(InSet(0, 0), Cmp(">", 2, 0))):
            parity(t, cols, types, node, bms, [0, 2])
            prog = encode(node, types)
            want_c, want_ids, want_cols = oracle.pushdown(cols, types, prog, proj=[0, 2], bitmaps=bms)
            r = t.execute(prog, project=[0, 2], max_size=n)
            assert r.materialized and r.count == want_c
            np.testing.assert_array_equal(r.rowids.cpu().numpy().view(np.uint32), want_ids)
            np.testing.assert_array_equal(r.columns[2].cpu().numpy(), want_cols[1])
            q = t.prepare_execute(prog, project=[0, 2], max_size=n)
            assert q.run() == want_c
            np.testing.assert_array_equal(q.result().rowids.cpu().numpy().view(np.uint32), want_ids)
            q.release()
            got, rows, _ = t.count_sampled(prog, 5, 2)
            keep = (np.arange(n) // 1024) % 5 == 2
            assert rows == int(keep.sum())
            assert got == oracle.count([x[keep] for x in cols], types, prog, bitmaps=bms)
        t.release()
    finally:
        release(bctx, ids)
