"""Full-size parity on the BASELINE.json configs, in bench.py's launch configuration.

C1 (60K rows) is checked element by element against the oracle. C3 (300M), C4 (480M) and
C5 (1e9) are too large for the oracle to scan whole within a test, so they are checked
  * on sampled windows: zero-copy sub-tables registered over 1M-row windows of the resident
    columns (row offsets exercise the shard path) are compared with the oracle on the same rows;
  * by properties that hold at any size: count(P) + count(NOT P) = N, the push-down count equals
    the probe count, its row ids are strictly increasing and inside [0, N), projected values
    equal the column at those ids, and every row id of a sampled window matches the oracle's;
  * C5 by its closed form: count(x < t) = t and ids = sort((v - b)/a mod N).
"""

import numpy as np
import pytest
import torch

import oracle
import paper_1806_08384_b200 as sel
from selgen import configs, encode
from selgen.program import Not

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(cuda_device):
    c = sel.Context(cuda_device)
    yield c
    c.close()


def _np(col, s, e):
    return col.data[s:e].cpu().numpy().view(
        {1: np.int32, 2: np.int64, 3: np.float32, 4: np.int32, 5: np.uint8, 6: np.uint16, 7: np.uint32}[col.ctype])


def _windows(n, k, size, seed):
    rng = np.random.default_rng(seed)
    starts = sorted(set(int(x) // 1024 * 1024 for x in rng.integers(0, max(1, n - size), k)))
    return [(s, min(n, s + size)) for s in starts] + [(max(0, n - 777_777) // 1024 * 1024, n)]  # + the tail


def check_large(ctx, T, probes, proj, seed):
    n = T.n_rows
    names = [c.name for c in T.columns]
    t = sel.Table(ctx, names, T.types, [c.data for c in T.columns])
    for name, node in probes.items():
        prog = encode(node, T.types)
        cnt = t.count(prog)
        assert cnt + t.count(encode(Not(node), T.types)) == n, name
        res = t.execute(prog, project=[names[j] for j in proj], max_size=n, capacity=cnt)
        assert res.materialized and res.count == cnt and res.rowids.numel() == cnt
        ids = res.rowids.to(torch.int64) & 0xFFFFFFFF
        if cnt > 1:
            assert bool((ids[1:] > ids[:-1]).all()), name
        if cnt:
            assert int(ids[0]) >= 0 and int(ids[-1]) < n
        for j in proj:
            assert torch.equal(res.columns[names[j]], T.columns[j].data[ids]), (name, names[j])
        for (s, e) in _windows(n, 6, 1_000_000, seed):
            host = [_np(c, s, e) for c in T.columns]
            want_c, want_ids, _ = oracle.pushdown(host, T.types, prog, row_offset=s)
            # the resident columns, registered as a zero-copy shard of the window
            w = sel.Table(ctx, names, T.types, [c.data[s:e] for c in T.columns], row_offset=s,
                          global_rows=n)
            assert w.count(prog) == want_c, (name, s, e)
            lo = int(torch.searchsorted(ids, torch.tensor(s, device=ids.device)))
            hi = int(torch.searchsorted(ids, torch.tensor(e, device=ids.device)))
            np.testing.assert_array_equal(ids[lo:hi].cpu().numpy().astype(np.uint32), want_ids)
            w.release()
    t.release()


def test_c1_lineitem_sf001_exact(ctx):
    T = configs.gen_lineitem(60_000, device=ctx.device)
    host = [c.data.cpu().numpy().view({1: np.int32, 2: np.int64, 4: np.int32, 5: np.uint8}[c.ctype])
            for c in T.columns]
    t = sel.Table(ctx, [c.name for c in T.columns], T.types, [c.data for c in T.columns])
    for name, node in configs.lineitem_probes(T).items():
        prog = encode(node, T.types)
        want_c, want_ids, want_cols = oracle.pushdown(host, T.types, prog, proj=[0, 3])
        assert t.count(prog) == want_c, name
        res = t.execute(prog, project=["l_orderkey", "l_extendedprice"], max_size=60_000)
        np.testing.assert_array_equal(res.rowids.cpu().numpy().view(np.uint32), want_ids)
        np.testing.assert_array_equal(res.columns["l_extendedprice"].cpu().numpy(), want_cols[1])


def test_c3_lineitem_sf50(ctx):
    T = configs.gen_lineitem(300_000_000, device=ctx.device,
                             columns=["l_orderkey", "l_discount", "l_extendedprice", "l_returnflag",
                                      "l_shipdate", "l_shipmode"])
    probes = configs.lineitem_probes(T)
    check_large(ctx, T, probes, [T.index("l_orderkey"), T.index("l_extendedprice"),
                                 T.index("l_discount")], seed=3)


def test_c4_lineorder_sf80(ctx):
    T = configs.gen_lineorder(480_000_000, device=ctx.device)
    check_large(ctx, T, configs.lineorder_probes(), [3], seed=4)


def test_c5_sweep_1e9_closed_form(ctx):
    n = configs.C5_ROWS
    T = configs.gen_sweep(n, device=ctx.device)
    a, b, a_inv = T.meta["affine"]
    t = sel.Table(ctx, ["x", "y"], T.types, [c.data for c in T.columns])
    for s in configs.C5_SELECTIVITIES:
        thr = configs.sweep_threshold(n, s)
        prog = encode(configs.sweep_probe(thr), T.types)
        assert t.count(prog) == thr, s
        if thr <= 50_000_000:
            res = t.execute(prog, project=["y"], max_size=n, capacity=thr)
            assert res.count == thr
            v = torch.arange(thr, dtype=torch.int64, device=ctx.device)
            want = torch.sort((a_inv * ((v - b) % n)) % n).values
            got = res.rowids.to(torch.int64) & 0xFFFFFFFF
            assert torch.equal(got, want), s
            assert torch.equal(res.columns["y"], T.col("y").data[got])


def test_c0_orders_sf50_paper_probes(ctx):
    """C0 (SURVEY §8d optional context): TPC-H SF-50 orders, 75M rows, with the paper's Table 5.1 /
    5.2 probes — `o_orderkey = 1` selects exactly one row and `o_orderkey >= 1` every row
     — the Listing 5.3 attribute sweep and Q5's one-year range (15.2 % of
    orders), on sampled windows and properties."""
    T = configs.gen_orders(75_000_000, device=ctx.device)
    probes = configs.orders_probes()
    t = sel.Table(ctx, [c.name for c in T.columns], T.types, [c.data for c in T.columns])
    assert t.count(encode(probes["l5.1"], T.types)) == 1
    assert t.count(encode(probes["l5.2"], T.types)) == 75_000_000
    q5 = t.count(encode(probes["q5_orderdate"], T.types))
    assert abs(q5 / 75_000_000 - 365 / 2406) < 0.002
    t.release()
    check_large(ctx, T, {k: probes[k] for k in ("attr2", "attr4", "q5_orderdate")}, [0, 1], 50)
