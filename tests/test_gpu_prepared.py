"""Prepared executes (include/sel.h sel_prepare_execute / sel_prepared_execute): Algorithm 1's
Execute captured once into a CUDA graph and replayed. Every run must equal a
fresh sel_execute and the oracle — including after the columns change in place, after the
context reallocates its scratch, after the bitmap registry changes, with timing toggled, and on
the non-graph cases (constant programs, empty tables)."""

import numpy as np
import pytest
import torch

import oracle
import paper_1806_08384_b200 as sel
from selgen import configs
from selgen.program import Cmp, InSet, And, Const, encode, random_program, INT32, DICT8, INT64

from helpers import random_table, make_bitmap
from test_gpu_parity import register

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pctx(cuda_device):
    c = sel.Context(cuda_device)
    yield c
    c.close()


def _check(q, cols, types, prog, proj):
    want_c, want_ids, want_cols = oracle.pushdown(cols, types, prog, proj=proj)
    assert q.run() == want_c
    assert q.materialized and q.local_count == want_c
    r = q.result()
    np.testing.assert_array_equal(r.rowids.cpu().numpy().view(np.uint32), want_ids)
    for j, c in enumerate(proj):
        np.testing.assert_array_equal(r.columns[c].cpu().numpy().view(want_cols[j].dtype), want_cols[j])
    return want_c


def test_prepared_parity_and_live_columns(pctx):
    n = 600_000
    T = configs.gen_c2(n)
    cols = [c.numpy().copy() for c in T.columns]
    t = register(pctx, cols, T.types)
    prog = encode(configs.c2_probes()["listing"], T.types)
    proj = configs.C2_PROJECT
    q = t.prepare_execute(prog, project=proj, max_size=n)
    for _ in range(3):
        c = _check(q, cols, T.types, prog, proj)
    assert c == 100_200
    assert pctx.last_pushdown_path() == 1
    # the graph reads the columns' current contents: change B in place, run again
    b = t.tensors[1]
    b[::7] = 1500                                     # inside (1000, 2001)
    cols[1] = b.cpu().numpy().copy()
    c2 = _check(q, cols, T.types, prog, proj)
    assert c2 > c
    # the run left its selection kept: a push-down of the same program reuses it
    p = t.pushdown(prog, project=[3], capacity=c2)
    assert pctx.last_pushdown_path() == 1 and p.count == c2
    # the same table through a fresh execute agrees
    r = t.execute(prog, project=proj, max_size=n)
    np.testing.assert_array_equal(r.rowids.cpu().numpy(), q.result().rowids.cpu().numpy())
    q.release()
    t.release()


def test_prepared_gate_writes_nothing(pctx):
    n = 300_000
    T = configs.gen_c2(n)
    cols = [c.numpy() for c in T.columns]
    t = register(pctx, cols, T.types)
    prog = encode(configs.c2_probes()["listing"], T.types)
    want = oracle.count(cols, T.types, prog)
    ids = torch.full((want,), -7, dtype=torch.int32, device=pctx.device)
    outs = [torch.full((want,), 5, dtype=d, device=pctx.device) for d in (torch.int32, torch.uint8, torch.int32)]
    q = t.prepare_execute(prog, project=configs.C2_PROJECT, max_size=want - 1, capacity=want,
                          out=(ids, outs))
    for _ in range(2):
        assert q.run() == want and not q.materialized and q.local_count == 0
        assert bool((ids == -7).all()) and all(bool((o == 5).all()) for o in outs)
    q2 = t.prepare_execute(prog, project=configs.C2_PROJECT, max_size=want, capacity=want,
                           out=(ids, outs))
    assert q2.run() == want and q2.materialized
    assert not bool((ids == -7).any())
    q.release()
    q2.release()
    t.release()


def test_prepared_recaptures_after_realloc_and_timing(pctx):
    rng = np.random.default_rng(11)
    types = [INT32, DICT8, INT64]
    small_cols, pools = random_table(rng, types, 5000)
    t_small = register(pctx, small_cols, types)
    node = random_program(rng, types, pools, max_depth=3)
    while sel.program_path(encode(node, types), types) == 2:
        node = random_program(rng, types, pools, max_depth=3)
    prog = encode(node, types)
    q = t_small.prepare_execute(prog, project=[0, 2], max_size=5000)
    _check(q, small_cols, types, prog, [0, 2])
    # a keeping probe of a much larger table reallocates the context's selection buffers
    big_cols, _ = random_table(rng, types, 3_000_000)
    t_big = register(pctx, big_cols, types)
    assert t_big.count(prog, keep_selection=True, keep_columns=[0, 2]) == oracle.count(big_cols, types, prog)
    _check(q, small_cols, types, prog, [0, 2])      # re-captured against the new buffers
    pctx.enable_timing(True)
    try:
        _check(q, small_cols, types, prog, [0, 2])
        c_ms, p_ms = pctx.last_times()
        assert c_ms > 0 and p_ms > 0
    finally:
        pctx.enable_timing(False)
    _check(q, small_cols, types, prog, [0, 2])
    q.release()
    t_big.release()
    t_small.release()


def test_prepared_bitmap_registry_and_release(pctx):
    n = 50_000
    x = (np.arange(n) % 1000).astype(np.int32)
    y = (np.arange(n) % 7).astype(np.uint8)
    t = register(pctx, [x, y], [INT32, DICT8])
    w1 = torch.from_numpy(make_bitmap(range(0, 1000, 3), 1000)[0].view(np.int64).copy()).to(pctx.device)
    bid = pctx.register_bitmap(w1, 1000)
    prog = encode(And(InSet(0, bid), Cmp("<", 1, 4)), [INT32, DICT8])
    q = t.prepare_execute(prog, project=[0], max_size=n)
    want1 = int((((x % 3) == 0) & (y < 4)).sum())
    assert q.run() == want1 and q.materialized
    pctx.release_bitmap(bid)
    with pytest.raises(sel.SelError) as e:
        q.run()
    assert e.value.status == 1
    w2 = torch.from_numpy(make_bitmap(range(0, 1000, 5), 1000)[0].view(np.int64).copy()).to(pctx.device)
    assert pctx.register_bitmap(w2, 1000) == bid
    want2 = int((((x % 5) == 0) & (y < 4)).sum())
    assert q.run() == want2
    np.testing.assert_array_equal(q.result().columns[0].cpu().numpy() % 5, 0)
    pctx.release_bitmap(bid)
    t.release()
    with pytest.raises(sel.SelError) as e:
        q.run()
    assert e.value.status == 8
    q.release()


def test_prepared_non_graph_cases(pctx):
    x = np.arange(10_000, dtype=np.int32)
    t = register(pctx, [x], [INT32])
    q_true = t.prepare_execute(encode(Const(True), [INT32]), project=[0], max_size=10_000)
    assert q_true.run() == 10_000 and q_true.materialized
    np.testing.assert_array_equal(q_true.result().columns[0].cpu().numpy(), x)
    q_false = t.prepare_execute(encode(Const(False), [INT32]), project=[0], max_size=0)
    assert q_false.run() == 0 and q_false.materialized
    with pytest.raises(sel.SelError) as e:
        t.prepare_execute(b"nope", max_size=1)
    assert e.value.status == 4
    q_true.release()
    q_false.release()
    t.release()


def test_prepared_with_single_rank_communicator(cuda_device):
    """With a (one-rank) NCCL communicator the prepared Execute captures the count all-reduce and
    the all-gather of per-rank counts into its graph; results, offset and the gate are unchanged.
    The host-gated path (constant program) issues the same collectives."""
    c = sel.Context(cuda_device)
    c.set_comm(1, 0, sel.Context.new_unique_id())
    n = 600_000
    T = configs.gen_c2(n)
    cols = [x.numpy() for x in T.columns]
    t = register(c, cols, T.types)
    prog = encode(configs.c2_probes()["listing"], T.types)
    proj = configs.C2_PROJECT
    q = t.prepare_execute(prog, project=proj, max_size=n)
    for _ in range(3):
        assert _check(q, cols, T.types, prog, proj) == 100_200
        assert q.result().offset == 0
    gated = t.prepare_execute(prog, project=proj, max_size=100_199, capacity=16)
    assert gated.run() == 100_200 and not gated.materialized
    for node in (Const(True), Const(False)):
        p = encode(node, T.types)
        qc = t.prepare_execute(p, project=[3], max_size=n if node.value else 0)
        want = n if node.value else 0
        assert qc.run() == want
        qc.release()
        r = t.execute(p, project=[3], max_size=0)           # host-gated, gated: all-gather too
        assert r.count == want and r.materialized == (want == 0)
    # collectives still line up: a plain count afterwards
    assert t.count(prog) == 100_200
    for h in (q, gated):
        h.release()
    t.release()
    c.close()


def _check_async(q, cols, types, prog, proj, stream=None):
    """sel_prepared_execute_async: the count is final at return; the outputs once the stream is."""
    want_c, want_ids, want_cols = oracle.pushdown(cols, types, prog, proj=proj)
    assert q.run(wait=False) == want_c
    assert q.materialized and q.local_count == want_c
    (stream or torch.cuda.current_stream(q.table.ctx.device)).synchronize()
    r = q.result()
    np.testing.assert_array_equal(r.rowids.cpu().numpy().view(np.uint32), want_ids)
    for j, c in enumerate(proj):
        np.testing.assert_array_equal(r.columns[c].cpu().numpy().view(want_cols[j].dtype), want_cols[j])
    return want_c


def test_prepared_async_parity_and_interleaving(pctx):
    """Async runs back to back (each launched while the previous materialisation may still run),
    interleaved with blocking runs, plain counts and executes of the same context, and a gated
    async run that writes nothing."""
    n = 3_006_000                            # ragged: 560 rows in the tail chunk
    T = configs.gen_c2(n)
    cols = [c.numpy().copy() for c in T.columns]
    t = register(pctx, cols, T.types)
    prog = encode(configs.c2_probes()["listing"], T.types)
    proj = configs.C2_PROJECT
    want = oracle.count(cols, T.types, prog)
    q = t.prepare_execute(prog, project=proj, max_size=n)
    for _ in range(20):                      # no synchronisation between the runs
        assert q.run(wait=False) == want and q.materialized
    _check_async(q, cols, T.types, prog, proj)
    assert _check(q, cols, T.types, prog, proj) == want
    # a second prepared execute (other program) alternating with the first
    prog2 = encode(configs.c2_probes()["between_in"], T.types)
    q2 = t.prepare_execute(prog2, project=[3], max_size=n)
    want2 = oracle.count(cols, T.types, prog2)
    for _ in range(5):
        assert q.run(wait=False) == want
        assert q2.run(wait=False) == want2
    _check_async(q2, cols, T.types, prog2, [3])
    _check_async(q, cols, T.types, prog, proj)
    # other calls of the context between async runs
    assert t.count(prog) == want
    assert q.run(wait=False) == want
    assert t.execute(prog, project=[3], max_size=n).count == want
    _check_async(q, cols, T.types, prog, proj)
    # the gate: count > max_size writes nothing, also when returning at the count
    ids = torch.full((want,), -7, dtype=torch.int32, device=pctx.device)
    outs = [torch.full((want,), 5, dtype=d, device=pctx.device) for d in (torch.int32, torch.uint8, torch.int32)]
    g = t.prepare_execute(prog, project=proj, max_size=want - 1, capacity=want, out=(ids, outs))
    assert g.run(wait=False) == want and not g.materialized and g.local_count == 0
    torch.cuda.synchronize(pctx.device)
    assert bool((ids == -7).all()) and all(bool((o == 5).all()) for o in outs)
    # with timing on the call blocks (the events are read at return) and still agrees
    pctx.enable_timing(True)
    try:
        assert q.run(wait=False) == want
        c_ms, p_ms = pctx.last_times()
        assert c_ms > 0 and p_ms > 0
    finally:
        pctx.enable_timing(False)
    for h in (q, q2, g):
        h.release()
    t.release()


def test_prepared_async_non_graph_and_communicator(cuda_device):
    """The async call on the uncaptured cases (constant program) and with a one-rank NCCL
    communicator (the result words come from the kernel after the all-gather)."""
    c = sel.Context(cuda_device)
    c.set_comm(1, 0, sel.Context.new_unique_id())
    n = 600_000
    T = configs.gen_c2(n)
    cols = [x.numpy() for x in T.columns]
    t = register(c, cols, T.types)
    prog = encode(configs.c2_probes()["listing"], T.types)
    q = t.prepare_execute(prog, project=configs.C2_PROJECT, max_size=n)
    for _ in range(3):
        assert _check_async(q, cols, T.types, prog, configs.C2_PROJECT) == 100_200
    qc = t.prepare_execute(encode(Const(True), T.types), project=[3], max_size=n)
    assert qc.run(wait=False) == n and qc.materialized
    torch.cuda.synchronize(cuda_device)
    np.testing.assert_array_equal(qc.result().columns[3].cpu().numpy(), cols[3])
    for h in (q, qc):
        h.release()
    t.release()
    c.close()


def test_prepared_async_capacity_cut(pctx):
    """Capacity below the count (the gated single-pass use without the gate firing): the async run
    returns the exact count and, once the stream has passed, exactly the first `capacity` selected
    rows (ascending) with nothing past them."""
    n = 606_000
    T = configs.gen_c2(n)
    cols = [c.numpy() for c in T.columns]
    t = register(pctx, cols, T.types)
    prog = encode(configs.c2_probes()["listing"], T.types)
    want_c, want_ids, want_cols = oracle.pushdown(cols, T.types, prog, proj=configs.C2_PROJECT)
    for cap in (1, 1023, 1024, 4097, want_c - 1):
        ids = torch.full((cap + 64,), -7, dtype=torch.int32, device=pctx.device)
        outs = [torch.full((cap + 64,), 5, dtype=d, device=pctx.device)
                for d in (torch.int32, torch.uint8, torch.int32)]
        q = t.prepare_execute(prog, project=configs.C2_PROJECT, max_size=n, capacity=cap,
                              out=(ids, outs))
        assert q.run(wait=False) == want_c and q.materialized and q.local_count == want_c
        torch.cuda.synchronize(pctx.device)
        np.testing.assert_array_equal(ids[:cap].cpu().numpy().view(np.uint32), want_ids[:cap])
        assert bool((ids[cap:] == -7).all())
        for o, w in zip(outs, want_cols):
            np.testing.assert_array_equal(o[:cap].cpu().numpy().view(w.dtype), w[:cap])
            assert bool((o[cap:] == 5).all())
        q.release()
    t.release()


def test_prepared_async_then_other_stream(pctx):
    """An async Execute on stream A, then at once a keeping count and an Execute of another program
    on stream B (they overwrite the context's selection): the library orders B after A's
    materialisation, so both results equal the oracle. Repeated to give a race room to show."""
    n = 6_000_000
    T = configs.gen_c2(n)
    cols = [c.numpy() for c in T.columns]
    t = register(pctx, cols, T.types)
    prog = encode(configs.c2_probes()["listing"], T.types)
    prog2 = encode(Cmp("<", 1, 1500), T.types)
    want_c, want_ids, want_cols = oracle.pushdown(cols, T.types, prog, proj=configs.C2_PROJECT)
    want2_c, want2_ids, _ = oracle.pushdown(cols, T.types, prog2, proj=[3])
    sa, sb = torch.cuda.Stream(pctx.device), torch.cuda.Stream(pctx.device)
    q = t.prepare_execute(prog, project=configs.C2_PROJECT, max_size=n, stream=sa)
    for _ in range(4):
        assert q.run(wait=False) == want_c
        assert t.count(prog2, stream=sb, keep_selection=True) == want2_c
        r2 = t.execute(prog2, project=[3], max_size=n, stream=sb)
        torch.cuda.synchronize(pctx.device)
        r = q.result()
        np.testing.assert_array_equal(r.rowids.cpu().numpy().view(np.uint32), want_ids)
        for j, c in enumerate(configs.C2_PROJECT):
            np.testing.assert_array_equal(r.columns[c].cpu().numpy().view(want_cols[j].dtype), want_cols[j])
        assert r2.count == want2_c
        np.testing.assert_array_equal(r2.rowids.cpu().numpy().view(np.uint32), want2_ids)
    q.release()
    t.release()
