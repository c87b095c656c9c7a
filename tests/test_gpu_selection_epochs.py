"""GPU parity of the kept selection's bookkeeping (sel_internal.h SelectionBufs, round 2): the
count's last CTA forms the exclusive prefix of 4,096-chunk hyperblocks from the superblock sums,
and the superblock sums alternate between two halves by a device epoch (each keeping count zeroes
the other half). Checked against the CPU oracle, element by element:
  * output positions across hyperblock boundaries (tables of 4,096 chunks +- a row / a chunk /
    a superblock, several hyperblocks with a ragged last one);
  * keeping counts over tables of different sizes in a row (the zeroed extents of both halves),
    then the push-down from the last kept selection;
  * prepared (graph) executes replayed an odd and an even number of times, interleaved with plain
    executes and push-downs of other tables (the epoch lives on the device, not in the graph)."""

import numpy as np
import pytest
import torch

import oracle
import paper_1806_08384_b200 as sel
from selgen.program import Cmp, And, encode, INT32, DICT8

pytestmark = pytest.mark.gpu

HB_ROWS = 4096 * 1024          # rows per hyperblock (4,096 chunks of 1,024 rows)


@pytest.fixture(scope="module")
def ctx(cuda_device):
    c = sel.Context(cuda_device)
    yield c
    c.close()


def make(ctx, n, seed):
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 1000, n, dtype=np.int32)
    y = rng.integers(0, 7, n, dtype=np.uint8)
    t = sel.Table(ctx, ["x", "y"], [INT32, DICT8],
                  [torch.from_numpy(x).to(ctx.device), torch.from_numpy(y).to(ctx.device)])
    return t, [x, y]


def want(cols, prog, proj=(0, 1)):
    return oracle.pushdown(cols, [INT32, DICT8], prog, proj=list(proj))


def check(res, w):
    cnt, ids, vals = w
    assert res.count == cnt
    np.testing.assert_array_equal(res.rowids.cpu().numpy().view(np.uint32), ids)
    for key, v in zip(("x", "y"), vals):
        np.testing.assert_array_equal(res.columns[key].cpu().numpy().view(v.dtype), v)


PROGS = [Cmp("<", 0, 300), And(Cmp(">=", 0, 100), Cmp("=", 1, 3)), Cmp("<", 0, 1000)]


@pytest.mark.parametrize("n", [HB_ROWS - 1, HB_ROWS, HB_ROWS + 1, HB_ROWS + 1024,
                               HB_ROWS + 65536 + 17, 3 * HB_ROWS + 5000])
def test_hyperblock_boundaries(ctx, n):
    t, cols = make(ctx, n, n)
    for node in PROGS:
        prog = encode(node, [INT32, DICT8])
        w = want(cols, prog)
        assert t.count(prog, keep_selection=True) == w[0]
        check(t.pushdown(prog, project=["x", "y"], capacity=w[0]), w)
        check(t.execute(prog, project=["x", "y"]), w)
    t.release()


def test_epochs_across_tables(ctx):
    big, big_cols = make(ctx, 2 * HB_ROWS + 333, 1)
    small, small_cols = make(ctx, 70_001, 2)
    mid, mid_cols = make(ctx, HB_ROWS // 2 + 7, 3)
    prog = encode(PROGS[1], [INT32, DICT8])
    wb, ws, wm = want(big_cols, prog), want(small_cols, prog), want(mid_cols, prog)
    # keeping counts back to back: each zeroes the other half over the extent its user left
    order = [(big, wb), (small, ws), (big, wb), (mid, wm), (small, ws), (small, ws), (big, wb),
             (mid, wm)]
    for t, w in order:
        assert t.count(prog, keep_selection=True) == w[0]
    check(mid.pushdown(prog, project=["x", "y"], capacity=wm[0]), wm)
    check(mid.pushdown(prog, project=["x", "y"], capacity=wm[0]), wm)   # the selection serves twice
    for t, w in order[::-1]:
        check(t.execute(prog, project=["x", "y"]), w)
    for t in (big, small, mid):
        t.release()


def test_prepared_replays_alternate_epochs(ctx):
    a, a_cols = make(ctx, HB_ROWS + 4099, 11)
    b, b_cols = make(ctx, 1_000_003, 12)
    pa = encode(PROGS[0], [INT32, DICT8])
    pb = encode(PROGS[1], [INT32, DICT8])
    wa, wb = want(a_cols, pa), want(b_cols, pb)
    qa = a.prepare_execute(pa, project=["x", "y"], max_size=a.local_rows)
    qb = b.prepare_execute(pb, project=["x", "y"], max_size=b.local_rows)
    for reps in (1, 2, 3, 5):
        for _ in range(reps):
            assert qa.run() == wa[0]
        check(qa.result(), wa)
        assert qb.run() == wb[0]
        check(qb.result(), wb)
        check(b.execute(pb, project=["x", "y"]), wb)
        # the prepared run leaves its selection kept: a push-down of the same program reuses it
        assert qa.run() == wa[0]
        check(a.pushdown(pa, project=["x", "y"], capacity=wa[0]), wa)
    qa.release()
    qb.release()
    a.release()
    b.release()
