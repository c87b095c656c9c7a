"""sel_count_sampled: the block sample's count is exact on its rows (oracle
parity over the same chunks), stride 1 is the full count, and the sampling estimator of
PAPER.md:199-203 misses rare selections the exact probe gets right ("less suitable for queries
which select only a single or a few tuples")."""

import numpy as np
import pytest
import torch

import oracle
import paper_1806_08384_b200 as sel
from selgen import configs, encode
from selgen.program import random_program, INT32, INT64, FLOAT32, DICT8

from helpers import random_table

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(cuda_device):
    c = sel.Context(cuda_device)
    yield c
    c.close()


def _sample_rows(n, stride, phase):
    idx = np.arange(n)
    return (idx // 1024) % stride == phase


@pytest.mark.parametrize("n", [1000, 1025, 70_001, 1_000_000])
def test_sample_count_parity(ctx, n):
    rng = np.random.default_rng(n)
    types = [INT32, DICT8, INT64, FLOAT32]
    cols, pools = random_table(rng, types, n)
    view = {INT32: np.int32, INT64: np.int64, FLOAT32: np.float32, DICT8: np.uint8}
    t = sel.Table(ctx, ["a", "b", "c", "d"], types,
                  [torch.from_numpy(np.ascontiguousarray(x).view(view[ty]).copy()).to(ctx.device)
                   for x, ty in zip(cols, types)])
    for _ in range(5):
        prog = encode(random_program(rng, types, pools, max_depth=3), types)
        assert t.count_sampled(prog, 1)[0] == t.count(prog) == oracle.count(cols, types, prog)
        for stride in (2, 3, 7, 64):
            phase = int(rng.integers(stride))
            sel_rows = _sample_rows(n, stride, phase)
            want = oracle.count([x[sel_rows] for x in cols], types, prog)
            got, rows, _ = t.count_sampled(prog, stride, phase)
            assert (got, rows) == (want, int(sel_rows.sum())), (stride, phase)


def test_sampling_misses_rare_selections(ctx):
    n = 1_500_000                                       # orders at SF 1
    T = configs.gen_orders(n, device=ctx.device)
    t = sel.Table(ctx, [c.name for c in T.columns], T.types, [c.data for c in T.columns])
    rare = encode(configs.orders_probes()["l5.1"], T.types)          # o_orderkey = 1 (1 row)
    common = encode(configs.orders_probes()["q5_orderdate"], T.types)  # ~15%
    assert t.count(rare) == 1
    ests = [t.count_sampled(rare, 100, ph)[2] for ph in range(100)]
    assert sum(e == 0 for e in ests) == 99 and max(ests) > 50           # 0 or ~98 (|R|/|R'|), never 1
    exact = t.count(common)
    est = t.count_sampled(common, 100, 17)[2]
    assert abs(est - exact) / exact < 0.05                             # broad patterns: fine


def test_equi_depth_histogram_parity(ctx):
    """sel_histogram vs oracle/synopsis.equi_depth over the same block sample:
    bucket bounds, rows and distinct counts bit-exact, for every integer column type, ragged
    sizes, several bucket counts, strides and phases; and the equality estimate beside the exact
    count."""
    import paper_1806_08384_b200 as sel
    from oracle import synopsis
    from helpers import random_table
    from selgen.program import INT32, DATE32, DICT8, DICT16, DICT32, INT64, FLOAT32, Cmp, encode
    from test_gpu_parity import register
    rng = np.random.default_rng(12)
    types = [INT32, DATE32, DICT8, DICT16, DICT32, INT64, FLOAT32]
    for n in (1, 1000, 5001, 70_001):
        cols, _ = random_table(rng, types, n)
        cols[0] = rng.integers(-3000, 3000, n).astype(np.int32)     # many duplicates per bucket
        t = register(ctx, cols, types)
        for j in range(5):
            for B, stride, phase in ((1, 1, 0), (7, 1, 0), (64, 3, 1), (16, 2, 1)):
                if phase >= (n + 1023) // 1024:
                    continue
                h = t.histogram(j, buckets=B, stride=stride, phase=phase)
                want = synopsis.equi_depth(synopsis.block_sample(cols[j], stride, phase), B)
                assert h["sample_rows"] == want["sample_rows"]
                for k in ("lo", "hi", "rows", "distinct"):
                    np.testing.assert_array_equal(h[k], want[k], err_msg=f"n={n} col={j} {k}")
        for j in (5, 6):
            with pytest.raises(sel.SelError):
                t.histogram(j)
        t.release()
    # the estimate vs the exact probe on a skewed column (the baseline the paper argues against)
    v = np.concatenate([np.full(90_000, 7, np.int32), rng.integers(0, 1000, 10_000).astype(np.int32)])
    rng.shuffle(v)
    t = register(ctx, [v], [INT32])
    h = t.histogram(0, buckets=16)
    for x in (7, 500):
        est = sel.equi_depth_estimate(h, x)
        assert est == pytest.approx(synopsis.estimate_eq(synopsis.equi_depth(v, 16), x, len(v)))
        exact = t.count(encode(Cmp("=", 0, x), [INT32]))
        print(f"x={x}: equi-depth estimate {est:.1f}, exact {exact}")
    t.release()
