"""GPU parity: libsel's sm_100a kernels (through the C ABI) vs the CPU oracle, element by element,
bit-exact (counts, ascending row-id sets and gathered values are unique).

Sizes span several 1024-row warp chunks and 8192-row CTA tiles plus ragged tails; the full-size
worked example (600M rows, BASELINE.json configs[1]) runs in bench.py's launch configuration and
is checked against the closed form of its tuple multiset."""

import math

import numpy as np
import pytest
import torch

import oracle
import paper_1806_08384_b200 as sel
from selgen import configs
from selgen.program import (Cmp, Between, In, And, Or, Not, Const, F32Bits, encode, encode_raw,
                            random_program, INT32, INT64, FLOAT32, DATE32, DICT8, DICT16, DICT32)

from helpers import random_table

pytestmark = pytest.mark.gpu

_TORCH = {INT32: torch.int32, INT64: torch.int64, FLOAT32: torch.float32, DATE32: torch.int32,
          DICT8: torch.uint8, DICT16: torch.int16, DICT32: torch.int32}


@pytest.fixture(scope="module")
def ctx(cuda_device):
    c = sel.Context(cuda_device)
    yield c
    c.close()


def to_gpu(arr, t, dev):
    a = np.ascontiguousarray(arr)
    view = {INT32: np.int32, INT64: np.int64, FLOAT32: np.float32, DATE32: np.int32,
            DICT8: np.uint8, DICT16: np.int16, DICT32: np.int32}[t]
    return torch.from_numpy(a.view(view).copy()).to(dev)


def register(ctx, cols, types, row_offset=0, global_rows=None):
    names = [f"c{i}" for i in range(len(cols))]
    tens = [to_gpu(c, t, ctx.device) for c, t in zip(cols, types)]
    return sel.Table(ctx, names, types, tens, row_offset=row_offset, global_rows=global_rows)


def _invalidate_selection(table):
    """A keep-selection probe of a constant program drops the context's kept selection."""
    table.count(encode(Const(True), table.types), keep_selection=True)


def check_parity(table, cols, types, node, proj=None, capacity=None, row_offset=0):
    """Count and every materialisation path vs the oracle:
       kept  — count keeping the selection AND the projected predicate columns' values, then
               push-down (Algorithm 1's order; what sel_execute does);
       sel   — count keeping only the selection, push-down gathers every projected column;
       single— no kept selection: single pass (evaluate + decoupled look-back);
       two   — no kept selection: two passes inside the call (keeping count, then materialise)."""
    prog = encode(node, types)
    proj = proj or []
    want_count, want_ids, want_cols = oracle.pushdown(cols, types, prog, proj=proj,
                                                      capacity=capacity, row_offset=row_offset)
    assert table.count(prog) == want_count, node
    cap = want_count if capacity is None else capacity
    n = table.local_rows
    const = sel.program_path(prog, types) == 2
    for mode in ("kept", "sel", "single", "two"):
        if mode == "kept":
            assert table.count(prog, keep_selection=True, keep_columns=proj) == want_count
        elif mode == "sel":
            assert table.count(prog, keep_selection=True) == want_count
        else:
            _invalidate_selection(table)
            table.ctx.set_pushdown_path(0 if mode == "single" else 2)
        try:
            res = table.pushdown(prog, project=proj, capacity=cap)
        finally:
            table.ctx.set_pushdown_path(-1)
        path = table.ctx.last_pushdown_path()
        if n > 0 and want_count > 0:
            # a program folded to a constant never launches the count kernel, so nothing is kept
            want_path = 0 if mode == "single" or const else (2 if mode == "two" else 1)
            assert path == want_path, (mode, path)
        assert res.count == want_count and res.local_count == want_count
        got_ids = res.rowids.cpu().numpy().view(np.uint32)
        np.testing.assert_array_equal(got_ids, want_ids, err_msg=f"{mode} {node}")
        for j, c in enumerate(proj):
            got = res.columns[c].cpu().numpy().view(want_cols[j].dtype)
            np.testing.assert_array_equal(got, want_cols[j], err_msg=f"{mode} col {c}")


def test_worked_example_scaled(ctx):
    n = 6_000_000
    T = configs.gen_c2(n)
    cols = [c.numpy() for c in T.columns]
    t = register(ctx, cols, T.types)
    for node in configs.c2_probes().values():
        check_parity(t, cols, T.types, node, proj=configs.C2_PROJECT)
        assert t.count(encode(node, T.types)) == 1_002_000


SIZES = [1, 3, 4, 5, 31, 1023, 1024, 1025, 4097, 8191, 8192, 8193, 65537, 250_003]


@pytest.mark.parametrize("n", SIZES)
def test_random_programs_ragged_sizes(ctx, n):
    rng = np.random.default_rng(n)
    types = [INT32, DICT8, INT64, FLOAT32, DICT16, DATE32, DICT32]
    cols, pools = random_table(rng, types, n)
    t = register(ctx, cols, types)
    for _ in range(25):
        node = random_program(rng, types, pools, max_depth=4)
        check_parity(t, cols, types, node, proj=[0, 1, 2, 3, 4, 5, 6])


def test_float_nan_signed_zero_subnormal(ctx):
    rng = np.random.default_rng(17)
    types = [FLOAT32, FLOAT32]
    cols, pools = random_table(rng, types, 20_000, with_nan=True)
    t = register(ctx, cols, types)
    for _ in range(60):
        check_parity(t, cols, types, random_program(rng, types, pools, max_depth=4), proj=[0])
    for node in [Cmp("=", 0, 0.0), Not(Cmp("<", 0, 1.0)), Cmp("<", 0, F32Bits(0x7FC00000)),
                 Not(Cmp("=", 0, F32Bits(0x7FC00000))), Cmp(">", 0, 1e-45), Between(0, -0.0, 0.0)]:
        check_parity(t, cols, types, node, proj=[1])


def test_empty_table_and_constants(ctx):
    types = [INT32]
    t = register(ctx, [np.zeros(0, np.int32)], types)
    for node in [Cmp("=", 0, 1), Const(True), Const(False)]:
        assert t.count(encode(node, types)) == 0
        assert t.pushdown(encode(node, types), capacity=10).count == 0
    x = np.arange(-50, 10_000, dtype=np.int32)
    t2 = register(ctx, [x], types)
    for node in [Const(True), Const(False), Or(Cmp("<", 0, 5), Cmp(">=", 0, 5)),
                 And(Cmp("<", 0, 5), Cmp(">=", 0, 5))]:
        check_parity(t2, [x], types, node, proj=[0])


def test_capacity_gate(ctx):
    """Algorithm 1: the exact count is always returned; only the first
    `capacity` ascending rows are written; capacity == count passes (strict '>')."""
    rng = np.random.default_rng(5)
    types = [INT32, DICT8]
    cols, pools = random_table(rng, types, 100_000)
    t = register(ctx, cols, types)
    node = Or(Cmp(">", 0, 0), In(1, (1, 2, 255)))
    prog = encode(node, types)
    full = oracle.count(cols, types, prog)
    for cap in [0, 1, 17, 8191, full // 2, full, full + 100]:
        for path in (1, 0, 2):
            if path == 1:
                t.count(prog, keep_selection=True)
            else:
                _invalidate_selection(t)
                ctx.set_pushdown_path(path)
            sentinel = torch.full((max(cap, 1) + 64,), -7, dtype=torch.int32, device=ctx.device)
            outc = torch.full((max(cap, 1) + 64,), 99, dtype=torch.uint8, device=ctx.device)
            try:
                res = t.pushdown(prog, project=[1], capacity=cap, out=(sentinel, [outc]))
            finally:
                ctx.set_pushdown_path(-1)
            assert ctx.last_pushdown_path() == path
            assert res.count == full and res.local_count == full
            assert res.gated == (full > cap)
            # nothing written past the capacity
            assert (sentinel[cap:].cpu() == -7).all()
            assert (outc[cap:].cpu() == 99).all()
        check_parity(t, cols, types, node, proj=[1], capacity=cap)


def test_shard_loop_offsets(ctx):
    """Register contiguous shards with their global offsets: counts add up, row ids
    are global, and the concatenation equals the unsharded result."""
    n = 300_007
    T = configs.gen_lineitem(n)
    cols = [c.numpy() for c in T.columns]
    probes = configs.lineitem_probes(T)
    cuts = [0, 77_777, 77_778, 200_000, n]
    for name, node in probes.items():
        prog = encode(node, T.types)
        want_c, want_ids, _ = oracle.pushdown(cols, T.types, prog)
        total, ids = 0, []
        for s, e in zip(cuts[:-1], cuts[1:]):
            t = register(ctx, [c[s:e] for c in cols], T.types, row_offset=s, global_rows=n)
            total += t.count(prog)
            ids.append(t.pushdown(prog).rowids.cpu().numpy().view(np.uint32))
        assert total == want_c, name
        np.testing.assert_array_equal(np.concatenate(ids), want_ids)


def test_large_program_block(ctx):
    """A program at the validator's limits (128 instructions, 512 constants) takes the large
    parameter block and the interpreter path."""
    rng = np.random.default_rng(8)
    instrs = [(0x30, 0, 0, 256), (0x30, 1, 256, 256), (0x41, 0, 0, 0)]
    k = 0
    while len(instrs) < 127:
        instrs += [(0x13 if k % 2 else 0x12, k % 2, int(rng.integers(512)), 0), (0x40 if k % 3 else 0x41, 0, 0, 0)]
        k += 1
    instrs.append((0x42, 0, 0, 0))
    consts = [int(v) for v in rng.integers(-3000, 3000, 512)]
    prog = encode_raw(instrs, [c & (2**64 - 1) for c in consts])
    types = [INT32, INT32]
    x = rng.integers(-3000, 3000, 200_000).astype(np.int32)
    y = rng.integers(-3000, 3000, 200_000).astype(np.int32)
    t = register(ctx, [x, y], types)
    want_c, want_ids, _ = oracle.pushdown([x, y], types, prog)
    assert t.count(prog) == want_c
    np.testing.assert_array_equal(t.pushdown(prog).rowids.cpu().numpy().view(np.uint32), want_ids)


def test_program_errors_surface(ctx):
    t = register(ctx, [np.arange(10, dtype=np.int32)], [INT32])
    with pytest.raises(sel.SelError) as e:
        t.count(b"SELP\x02\x00")
    assert e.value.status == 4
    with pytest.raises(sel.SelError) as e:
        t.count(encode_raw([(0x10, 0, 0, 0)], [1 << 40]))
    assert e.value.status == 3


def test_alignment_and_size_checks(ctx):
    x = torch.zeros(100, dtype=torch.int32, device=ctx.device)
    with pytest.raises(sel.SelError) as e:
        sel.Table(ctx, ["x"], [INT32], [x[1:]])
    assert e.value.status == 2
    with pytest.raises(sel.SelError) as e:
        sel.Table(ctx, ["x"], [INT32], [x], global_rows=1 << 32)
    assert e.value.status == 5


def test_nccl_single_rank_comm_and_timing(ctx, cuda_device):
    c = sel.Context(cuda_device)
    c.set_comm(1, 0, sel.Context.new_unique_id())
    c.enable_timing(True)
    T = configs.gen_c2(600_000)
    cols = [x.numpy() for x in T.columns]
    t = register(c, cols, T.types)
    prog = encode(configs.c2_probes()["listing"], T.types)
    assert t.count(prog) == 100_200
    assert c.last_kernel_ms() > 0
    res = t.pushdown(prog, project=[3])
    assert res.count == 100_200 and res.offset == 0
    np.testing.assert_array_equal(res.rowids.cpu().numpy().view(np.uint32),
                                  oracle.pushdown(cols, T.types, prog)[1])
    c.close()


def _closed_form_ids_gpu(T, node, dev):
    """Closed-form ascending row ids of a C2 predicate, computed on the GPU with torch."""
    ta, tb, tc, tm = T.meta["tuples"]
    from helpers import np_mask
    hit = np_mask(node, [ta.astype(np.int32), tb.astype(np.int32), tc.astype(np.uint8)],
                  [INT32, INT32, DICT8], len(ta))
    ends = np.cumsum(tm)
    starts = ends - tm
    a, b, _ = T.meta["affine"]
    parts = []
    for s, e in zip(starts[hit], ends[hit]):
        parts.append(torch.arange(int(s), int(e), dtype=torch.int64, device=dev))
    j = torch.cat(parts)
    return torch.sort((a * j + b) % T.n_total).values, int(tm[hit].sum())


def test_full_size_worked_example(ctx):
    """BASELINE.json configs[1] at full size (600M rows), in bench.py's launch configuration:
    exact count 100,200,000 for all encodings, and the push-down row ids / projected
    columns equal the closed form of the tuple multiset (every one of the 100.2M rows checked)."""
    dev = ctx.device
    T = configs.gen_c2(device=dev)
    t = sel.Table(ctx, ["A", "B", "C", "D"], T.types, [c.data for c in T.columns])
    for node in configs.c2_probes().values():
        assert t.count(encode(node, T.types)) == 100_200_000
    assert t.count(encode(Cmp("=", 0, 2), T.types)) == 120_000_000
    node = configs.c2_probes()["listing"]
    want_ids, want_n = _closed_form_ids_gpu(T, node, dev)
    res = t.execute(encode(node, T.types), project=["A", "C", "D"], max_size=600_000_000,
                    capacity=100_200_000)       # bench.py's step: Execute(isSPD) = count + materialise
    assert res.materialized and ctx.last_pushdown_path() == 1
    assert res.count == want_n == 100_200_000
    got = res.rowids.to(torch.int64) & 0xFFFFFFFF
    assert torch.equal(got, want_ids)
    assert bool((res.columns["A"] == 2).all())
    cc = res.columns["C"]
    assert bool(((cc == 1) | (cc == 4)).all())
    assert torch.equal(res.columns["D"], T.col("D").data[got])
    # a plain sel_pushdown (no kept selection) gives the same bytes: at this size it takes two
    # passes by default (2); forced, the single pass (0)
    for mode, want_path in ((-1, 2), (0, 0)):
        _invalidate_selection(t)
        ctx.set_pushdown_path(mode)
        try:
            res2 = t.pushdown(encode(node, T.types), project=["A", "C", "D"], capacity=want_n)
        finally:
            ctx.set_pushdown_path(-1)
        assert ctx.last_pushdown_path() == want_path
        assert res2.count == want_n
        assert torch.equal(res2.rowids, res.rowids)
        for k in "ACD":
            assert torch.equal(res2.columns[k], res.columns[k])
        del res2
    # the complement partitions the table (count(P) + count(NOT P) = N)
    assert t.count(encode(Not(node), T.types)) == 600_000_000 - 100_200_000


def test_context_destroyed_before_table(cuda_device):
    """A table released (or garbage-collected) after its context was destroyed is safe; probes on
    it report SEL_E_STATE instead of touching freed memory."""
    c = sel.Context(cuda_device)
    t = register(c, [np.arange(100, dtype=np.int32)], [INT32])
    c.close()
    with pytest.raises(sel.SelError) as e:
        t.count(encode(Cmp("<", 0, 5), [INT32]))
    assert e.value.status == 8
    t.release()


def test_execute_gate(ctx):
    """sel_execute = Algorithm 1's Execute(compound, isSPD=true, maxSize):
    count > maxSize "throws" (nothing materialised, buffers untouched); count <= maxSize (strict
    '>', so maxSize == count passes) materialises exactly the oracle's rows and values."""
    n = 600_000
    T = configs.gen_c2(n)
    cols = [c.numpy() for c in T.columns]
    t = register(ctx, cols, T.types)
    node = configs.c2_probes()["listing"]
    prog = encode(node, T.types)
    want_c, want_ids, want_cols = oracle.pushdown(cols, T.types, prog, proj=configs.C2_PROJECT)
    for max_size in (0, want_c - 1):
        ids = torch.full((want_c,), -7, dtype=torch.int32, device=ctx.device)
        outs = [torch.full((want_c,), 5, dtype=d, device=ctx.device) for d in (torch.int32, torch.uint8, torch.int32)]
        r = t.execute(prog, project=configs.C2_PROJECT, max_size=max_size, capacity=want_c, out=(ids, outs))
        assert r.count == want_c and not r.materialized and r.rowids.numel() == 0
        assert bool((ids == -7).all()) and all(bool((o == 5).all()) for o in outs)
    for max_size in (want_c, n):
        r = t.execute(prog, project=configs.C2_PROJECT, max_size=max_size)
        assert r.materialized and r.count == want_c and ctx.last_pushdown_path() == 1
        np.testing.assert_array_equal(r.rowids.cpu().numpy().view(np.uint32), want_ids)
        for j, c in enumerate(configs.C2_PROJECT):
            np.testing.assert_array_equal(r.columns[c].cpu().numpy().view(want_cols[j].dtype), want_cols[j])
    # a selection that matches nothing: count 0 passes any gate (0 > 0 is false), writes nothing
    r = t.execute(encode(Cmp("=", 0, 99), T.types), project=[3], max_size=0, capacity=4)
    assert r.materialized and r.count == 0 and r.rowids.numel() == 0
    # a gated execute still keeps its selection: a push-down of the same program reuses it
    r = t.execute(prog, project=[3], max_size=0, capacity=want_c)
    assert not r.materialized and r.count == want_c
    p = t.pushdown(prog, project=[3], capacity=want_c)
    assert ctx.last_pushdown_path() == 1 and p.count == want_c
    np.testing.assert_array_equal(p.rowids.cpu().numpy().view(np.uint32), want_ids)
    # both kernels of the one-synchronisation execute are timed
    ctx.enable_timing(True)
    try:
        r = t.execute(prog, project=configs.C2_PROJECT, max_size=n)
        c_ms, p_ms = ctx.last_times()
        assert r.materialized and c_ms > 0 and p_ms > 0
    finally:
        ctx.enable_timing(False)


def test_constant_projections(ctx):
    """A conjunction pins a column with a single-value leaf: the push-down fills that projection
    instead of keeping or gathering it. Every type (negative INT32/INT64, FLOAT32 of either sign,
    DICT8/16 codes) through execute, both push-down paths and a prepared execute; x = 0.0 is two
    keys (-0, +0) and must still gather the real bits."""
    n = 300_017
    rng = np.random.default_rng(8)
    a = rng.choice(np.array([-5, 3, 7], dtype=np.int32), n)
    b = rng.choice(np.array([-(2**40), 1, 2**50], dtype=np.int64), n)
    f = rng.choice(np.array([-1.5, 1.5, 0.0, -0.0], dtype=np.float32), n)
    d8 = rng.integers(0, 4, n).astype(np.uint8)
    d16 = rng.choice(np.array([0, 65535], dtype=np.uint16), n)
    cols = [a, b, f, d8, d16]
    types = [INT32, INT64, FLOAT32, DICT8, DICT16]
    t = register(ctx, cols, types)
    progs = [
        And(And(Cmp("=", 0, -5), Cmp("=", 1, -(2**40))), Cmp("=", 2, -1.5)),
        And(And(Cmp("=", 2, 1.5), Cmp("=", 4, 65535)), Cmp("<", 3, 3)),
        And(Cmp("=", 2, 0.0), Cmp("=", 3, 2)),                     # f: -0 and +0 both selected
        And(In(0, (7,)), Between(1, 1, 1)),
    ]
    proj = [0, 1, 2, 3, 4]
    for node in progs:
        plan = sel.program_plan(encode(node, types), types)
        assert plan["path"] == 1
        check_parity(t, cols, types, node, proj=proj)
        prog = encode(node, types)
        want_c, want_ids, want_cols = oracle.pushdown(cols, types, prog, proj=proj)
        for r in (t.execute(prog, project=proj, max_size=n),):
            assert r.materialized and r.count == want_c
            for j in proj:
                np.testing.assert_array_equal(r.columns[j].cpu().numpy().view(want_cols[j].dtype), want_cols[j])
        q = t.prepare_execute(prog, project=proj, max_size=n)
        assert q.run() == want_c
        res = q.result()
        for j in proj:
            np.testing.assert_array_equal(res.columns[j].cpu().numpy().view(want_cols[j].dtype), want_cols[j])
        q.release()
    # x = 0.0 selects both zeros: the projected bits are not a constant
    _, _, wc = oracle.pushdown(cols, types, encode(progs[2], types), proj=[2])
    assert len(set(wc[0].view(np.uint32).tolist())) == 2
    t.release()


def test_selection_chunk_densities(ctx):
    """Kept selections whose per-chunk counts span empty, 1, sector and warp boundaries
    (15/16/17, 31/32/33, 63/64/65), dense and full chunks, and a ragged tail; every
    materialisation path."""
    rng = np.random.default_rng(64)
    ks = [0, 1, 2, 15, 16, 17, 31, 32, 33, 48, 63, 64, 65, 100, 511, 1023, 1024, 0, 64, 7]
    n = 1024 * len(ks) - 300                                     # the last chunk is ragged
    x = np.zeros(n, np.int32)
    for c, k in enumerate(ks):
        lo, hi = 1024 * c, min(n, 1024 * c + 1024)
        pick = rng.choice(hi - lo, size=min(k, hi - lo), replace=False)
        x[lo + pick] = 1
    y = rng.integers(-1000, 1000, n).astype(np.int32)
    types = [INT32, INT32]
    t = register(ctx, [x, y], types)
    for node in [Cmp("=", 0, 1), And(Cmp("=", 0, 1), Cmp(">", 1, 0)), Cmp("=", 0, 0)]:
        check_parity(t, [x, y], types, node, proj=[1, 0])


def test_exactness_1000_random_cases(ctx):
    """SPEC.md acceptance 3 (zero tolerance): 1,000 random tables of <= 10^4 rows with
    random column types and random predicate trees of depth <= 3; the GPU count and the
    materialised row ids and values equal the oracle's."""
    rng = np.random.default_rng(1000)
    all_types = [INT32, INT64, FLOAT32, DATE32, DICT8, DICT16, DICT32]
    for case in range(1000):
        k = int(rng.integers(1, 4))
        types = [all_types[int(i)] for i in rng.integers(0, len(all_types), k)]
        n = int(rng.integers(0, 10_001))
        cols, pools = random_table(rng, types, n)
        t = register(ctx, cols, types)
        node = random_program(rng, types, pools, max_depth=3)
        prog = encode(node, types)
        proj = [int(rng.integers(0, k))]
        want_c, want_ids, want_cols = oracle.pushdown(cols, types, prog, proj=proj)
        assert t.count(prog) == want_c, (case, node)
        res = t.pushdown(prog, project=proj, capacity=want_c)
        assert res.count == want_c, (case, node)
        np.testing.assert_array_equal(res.rowids.cpu().numpy().view(np.uint32), want_ids,
                                      err_msg=f"case {case}")
        got = res.columns[proj[0]].cpu().numpy().view(want_cols[0].dtype)
        np.testing.assert_array_equal(got, want_cols[0], err_msg=f"case {case}")
        t.release()


def test_kept_selection_serves_repeated_pushdowns(ctx):
    """A kept selection is not consumed: any number of push-downs (and executes' own selections)
    materialise the same rows (regression: the superblock sums must survive the prefix scan)."""
    T = configs.gen_c2(600_000)
    cols = [c.numpy() for c in T.columns]
    t = register(ctx, cols, T.types)
    prog = encode(configs.c2_probes()["listing"], T.types)
    want_c, want_ids, want_cols = oracle.pushdown(cols, T.types, prog, proj=[2, 3])
    runs = []
    t.count(prog, keep_selection=True)
    runs += [t.pushdown(prog, project=[2, 3]) for _ in range(3)]
    runs.append(t.execute(prog, project=[2, 3], max_size=600_000))
    runs += [t.pushdown(prog, project=[2, 3]) for _ in range(2)]
    q = t.prepare_execute(prog, project=[2, 3], max_size=600_000)
    q.run()
    runs.append(q.result())
    runs += [t.pushdown(prog, project=[2, 3]) for _ in range(2)]
    for r in runs:
        assert r.count == want_c
        np.testing.assert_array_equal(r.rowids.cpu().numpy().view(np.uint32), want_ids)
        for j, c in enumerate([2, 3]):
            np.testing.assert_array_equal(r.columns[c].cpu().numpy().view(want_cols[j].dtype), want_cols[j])
    q.release()


def test_count_async_and_user_graph_capture(ctx, cuda_device):
    """sel_count_async: no host synchronisation; the count lands in a device word — also when the
    call is captured into the caller's own CUDA graph (torch.cuda.graph) and replayed after the
    column changed in place; constant programs and an empty table; a one-rank peer context."""
    T = configs.gen_c2(600_000)
    cols = [c.numpy().copy() for c in T.columns]
    types = T.types
    for cx in (ctx, None):
        if cx is None:
            cx = sel.Context(cuda_device)
            cx.set_peers(1, 0, [cx.peer_handle()])
        t = register(cx, cols, types)
        prog = encode(configs.c2_probes()["listing"], types)
        out = torch.zeros(4, dtype=torch.int64, device=cx.device)
        s = torch.cuda.Stream(cx.device)
        with torch.cuda.stream(s):
            t.count_async(prog, out[0:1], stream=s)
            t.count_async(encode(Const(True), types), out[1:2], stream=s)
            t.count_async(encode(Const(False), types), out[2:3], stream=s)
        s.synchronize()
        assert out[:3].tolist() == [100_200, 600_000, 0]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            t.count_async(prog, out[3:4], stream=s)
        out[3] = -1
        g.replay()
        torch.cuda.synchronize()
        assert int(out[3]) == 100_200
        t.tensors[0].fill_(2)                                # every row has A = 2 now
        g.replay()
        torch.cuda.synchronize()
        want = oracle.count([np.full(600_000, 2, np.int32)] + cols[1:], types, prog)
        assert int(out[3]) == want
        del g
        t.release()
        if cx is not ctx:
            cx.drop_peers()
            cx.close()
    e = register(ctx, [np.zeros(0, np.int32)], [INT32])
    o = torch.full((1,), -1, dtype=torch.int64, device=ctx.device)
    e.count_async(encode(Cmp("=", 0, 1), [INT32]), o)
    torch.cuda.synchronize()
    assert int(o) == 0


def test_fully_selected_chunks_dense_copy(ctx):
    """Tables of >= 8M rows leave fully selected 1024-row chunks to the whole-chunk copy kernel
    (dense_chunks_kernel) beside the push-down: clustered and dense selections, full chunks next
    to partial and dense-not-full ones and a ragged tail, kept/constant projections, capacity cuts
    inside and at a full chunk; every materialisation path vs the oracle."""
    rng = np.random.default_rng(88)
    n = 12_000_037
    x = np.arange(n, dtype=np.int32)
    y = rng.integers(-(1 << 31), (1 << 31) - 1, n, dtype=np.int64).astype(np.int32)
    z = (np.arange(n) % 7).astype(np.uint8)
    types = [INT32, INT32, DICT8]
    cols = [x, y, z]
    t = register(ctx, cols, types)
    for node in [Cmp("<", 0, 9_000_123), Cmp(">=", 0, 3_000_000),
                 And(Cmp("<", 0, 9_000_123), Cmp(">", 1, 0)),
                 Or(Cmp("<", 0, 2_048_000), Cmp(">", 1, 2_000_000_000)),
                 And(Cmp(">=", 0, 1_000_000), Cmp("=", 2, 3)),
                 # scattered rows first: the full chunks after them land at unaligned positions
                 Or(Cmp(">", 1, 2_000_000_000), Cmp(">=", 0, 6_000_000)),
                 # dense, not full chunks; 8-byte-free mix of widths; the ragged tail dense
                 Cmp(">", 1, -1_500_000_000), Cmp("<", 1, 0),
                 And(Cmp(">=", 0, 11_000_000), Not(Cmp("=", 2, 5)))]:
        check_parity(t, cols, types, node, proj=[1, 2, 0])
    for node, cap in [(Cmp("<", 0, 9_000_123), c) for c in (4_096, 5_000, 1_000_000)] + \
                     [(Cmp(">", 1, -1_500_000_000), c) for c in (4_000, 5_000, 777_777)]:
        # a capacity cut at / inside a full (then a dense) chunk
        prog = encode(node, types)
        want_c, want_ids, _ = oracle.pushdown(cols, types, prog, capacity=cap)
        t.count(prog, keep_selection=True)
        r = t.pushdown(prog, project=[1], capacity=cap)
        assert r.count == want_c and r.gated
        np.testing.assert_array_equal(r.rowids.cpu().numpy().view(np.uint32), want_ids)
        np.testing.assert_array_equal(r.columns[1].cpu().numpy(), y[want_ids])
    t.release()


def test_fully_selected_chunks_coded(ctx):
    """Coded projections (a conjunction pins the projected column to two values: an IN of two
    points on a 1- or 4-byte column; the keeping count keeps one code bit per row) through the
    whole-chunk copy: full chunks take each row's value from its code bit in dense_chunks_kernel,
    partial ones in the push-down's staging; capacity cuts at and inside a full chunk."""
    rng = np.random.default_rng(89)
    n = 12_000_037
    x = np.arange(n, dtype=np.int32)
    z = rng.integers(0, 7, n).astype(np.uint8)
    z[:6_000_000] = rng.choice(np.array([1, 4], np.uint8), 6_000_000)
    w = rng.integers(-(1 << 31), (1 << 31) - 1, n, dtype=np.int64).astype(np.int32)
    w[2_000_000:10_000_000] = rng.choice(np.array([-5, 100_000], np.int32), 8_000_000)
    types = [INT32, DICT8, INT32]
    cols = [x, z, w]
    t = register(ctx, cols, types)
    plan_cases = [(And(Cmp("<", 0, 9_000_123), In(1, (1, 4))), [1, 2, 0]),
                  (And(In(2, (-5, 100_000)), Cmp(">=", 0, 1_000_000)), [2, 1]),
                  (In(1, (4, 1)), [1]),
                  (And(In(1, (1, 4)), In(2, (100_000, -5))), [2, 0, 1])]
    for node, proj in plan_cases:
        check_parity(t, cols, types, node, proj=proj)
    node = And(Cmp("<", 0, 9_000_123), In(1, (1, 4)))
    prog = encode(node, types)
    for cap in (4_096, 5_000, 1_000_000):
        # Algorithm 1's Execute: the keeping count records the code bits of z (projected), and
        # the materialisation writes z from them — through the whole-chunk copy too (ADVICE r1:
        # the capacity cut must be exercised on the CODED path, so assert that it was taken)
        want_c, want_ids, _ = oracle.pushdown(cols, types, prog, capacity=cap)
        r = t.execute(prog, project=[1, 0], max_size=n, capacity=cap)
        flags = ctx.last_pushdown_flags()
        assert flags & sel._native.SEL_PD_CODED and flags & sel._native.SEL_PD_WHOLE_CHUNKS, flags
        assert r.count == want_c and r.materialized and r.local_count > cap
        np.testing.assert_array_equal(r.rowids.cpu().numpy().view(np.uint32), want_ids)
        np.testing.assert_array_equal(r.columns[1].cpu().numpy(), z[want_ids])
        np.testing.assert_array_equal(r.columns[0].cpu().numpy(), x[want_ids])
        # the two passes inside sel_pushdown (no kept selection) take the coded path as well
        _invalidate_selection(t)
        r = t.pushdown(prog, project=[1, 0], capacity=cap)
        assert ctx.last_pushdown_path() == 2 and ctx.last_pushdown_flags() & sel._native.SEL_PD_CODED
        assert r.count == want_c and r.gated
        np.testing.assert_array_equal(r.rowids.cpu().numpy().view(np.uint32), want_ids)
        np.testing.assert_array_equal(r.columns[1].cpu().numpy(), z[want_ids])
        np.testing.assert_array_equal(r.columns[0].cpu().numpy(), x[want_ids])
    t.release()
