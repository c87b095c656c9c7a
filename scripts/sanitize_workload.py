"""Small-size exercise of every kernel path (count, selection push-down, single pass, kept values,
batch) for compute-sanitizer; see scripts/sanitize.sh."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import oracle, paper_1806_08384_b200 as sel
from selgen import configs, encode
from selgen.program import *
from helpers import random_table
dev = torch.device('cuda:0')
ctx = sel.Context(dev)
for n in [5, 1025, 70_001]:
    rng = np.random.default_rng(n)
    types = [INT32, DICT8, INT64, FLOAT32, DICT16]
    cols, pools = random_table(rng, types, n)
    view = {INT32: np.int32, INT64: np.int64, FLOAT32: np.float32, DICT8: np.uint8, DICT16: np.int16}
    t = sel.Table(ctx, [f"c{i}" for i in range(5)], types,
                  [torch.from_numpy(np.ascontiguousarray(c).view(view[ty]).copy()).to(dev) for c, ty in zip(cols, types)])
    for _ in range(4):
        node = random_program(rng, types, pools, max_depth=3)
        prog = encode(node, types)
        want = oracle.pushdown(cols, types, prog, proj=[0, 1, 2])
        c = t.count(prog)
        r1 = t.execute(prog, project=[0, 1, 2], max_size=n)                  # selection path
        t.count(encode(Const(True), types), keep_selection=True)
        r2 = t.pushdown(prog, project=[0, 1, 2], capacity=max(want[0], 1))    # single pass
        t.count(prog, keep_selection=True, keep_columns=[0, 1, 2])
        r3 = t.pushdown(prog, project=[0, 1, 2], capacity=max(want[0], 1))    # kept values
        b = t.count_batch([prog, encode(Not(node), types)])
        assert c == want[0] == r1.count == r2.count == r3.count and b[0] + b[1] == n
        for r in (r1, r2, r3):
            assert np.array_equal(r.rowids.cpu().numpy().view(np.uint32), want[1])
# IN_BITMAP leaves: a staged small set and a global (too large to stage) set; prepared executes;
# the block-sampled count
from helpers import make_bitmap
for n in [1025, 70_001]:
    rng = np.random.default_rng(7 + n)
    a = rng.integers(0, (1 << 21) + 100, n).astype(np.int32)
    b = rng.integers(0, 3000, n).astype(np.int32)
    big = make_bitmap(np.flatnonzero(rng.random(1 << 21) < 0.3), 1 << 21)
    small = make_bitmap(np.flatnonzero(rng.random(3000) < 0.5), 3000)
    ids = [ctx.register_bitmap(torch.from_numpy(w.view(np.int64).copy()).to(dev), nb) for w, nb in (big, small)]
    t = sel.Table(ctx, ["a", "b"], [INT32, INT32], [torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)])
    for node in (And(InSet(0, ids[0]), InSet(1, ids[1])), Or(Not(InSet(0, ids[0])), Cmp("<", 1, 100))):
        prog = encode(node, [INT32, INT32])
        want = oracle.pushdown([a, b], [INT32, INT32], prog, proj=[0, 1], bitmaps=[big, small])
        r1 = t.execute(prog, project=[0, 1], max_size=n)
        q = t.prepare_execute(prog, project=[0, 1], max_size=n)
        assert q.run() == want[0] == r1.count
        assert np.array_equal(q.result().rowids.cpu().numpy().view(np.uint32), want[1])
        q.release()
        t.count(encode(Const(True), [INT32, INT32]), keep_selection=True)
        r2 = t.pushdown(prog, project=[0, 1], capacity=max(want[0], 1))       # single pass, global sets
        assert np.array_equal(r2.rowids.cpu().numpy().view(np.uint32), want[1])
        assert t.count_sampled(prog, 3, 1)[1] > 0
    t.release()
    for i in ids:
        ctx.release_bitmap(i)
# conjunctive fast path (count kernel FASTN = 1..4) through count, execute and the two-pass
# push-down; a one-rank communicator (the Execute's all-gather, captured in a prepared graph)
sys.path.insert(0, 'tests')
from test_gpu_fastpath import TYPES as FT, fast_conjunction
cctx = sel.Context(dev)
cctx.set_comm(1, 0, sel.Context.new_unique_id())
pctx = sel.Context(dev)                                  # one-rank peer-memory exchange
pctx.set_peers(1, 0, [pctx.peer_handle()])
for n in [1025, 70_001]:
    rng = np.random.default_rng(11 + n)
    cols, pools = random_table(rng, FT, n)
    view = {INT32: np.int32, DATE32: np.int32, DICT32: np.int32, INT64: np.int64, DICT8: np.uint8}
    tens = [torch.from_numpy(np.ascontiguousarray(c).view(view[ty]).copy()).to(dev) for c, ty in zip(cols, FT)]
    for cx in (ctx, cctx, pctx):
        t = sel.Table(cx, [f"c{i}" for i in range(len(FT))], FT, tens)
        for _ in range(6):
            node = fast_conjunction(rng, pools)
            prog = encode(node, FT)
            want = oracle.pushdown(cols, FT, prog, proj=[0, 3, 4])
            assert t.count(prog) == want[0]
            r1 = t.execute(prog, project=[0, 3, 4], max_size=n)
            cx.set_pushdown_path(2)
            t.count(encode(Const(True), FT), keep_selection=True)
            r2 = t.pushdown(prog, project=[0, 3, 4], capacity=max(want[0], 1))   # two passes
            cx.set_pushdown_path(-1)
            q = t.prepare_execute(prog, project=[0, 3, 4], max_size=n)
            assert q.run() == want[0]
            for r in (r1, r2, q.result()):
                assert np.array_equal(r.rowids.cpu().numpy().view(np.uint32), want[1])
            q.release()
        t.release()
cctx.close()
pctx.drop_peers()
pctx.close()
# coded projection (C2's C IN (1, 4) projected) through execute, prepared execute, two passes
T = configs.gen_c2(60_000, device=dev)
t = sel.Table(ctx, ["A", "B", "C", "D"], T.types, [c.data for c in T.columns])
host = [c.numpy() for c in configs.gen_c2(60_000).columns]
prog = encode(configs.c2_probes()["listing"], T.types)
want = oracle.pushdown(host, T.types, prog, proj=[0, 2, 3])
r1 = t.execute(prog, project=[0, 2, 3], max_size=60_000)
q = t.prepare_execute(prog, project=[0, 2, 3], max_size=60_000)
assert q.run() == want[0] == r1.count
for r in (r1, q.result()):
    assert np.array_equal(r.rowids.cpu().numpy().view(np.uint32), want[1])
    assert np.array_equal(r.columns[2].cpu().numpy(), want[2][1])
# the async run (returns at the count; sequence word in pinned memory), back to back
for _ in range(3):
    assert q.run(wait=False) == want[0]
torch.cuda.synchronize()
assert np.array_equal(q.result().rowids.cpu().numpy().view(np.uint32), want[1])
q.release()
# sel_execute_to into the context's own buffers (offset 0)
ids = torch.empty(want[0], dtype=torch.int32, device=dev)
cd = [torch.empty(want[0], dtype=c.dtype, device=dev) for c in (T.columns[0].data, T.columns[2].data, T.columns[3].data)]
cnt, loc, off, mat = t.execute_to(prog, [0, 2, 3], 60_000, want[0], ids.data_ptr(), [x.data_ptr() for x in cd])
assert cnt == want[0] and mat and off == 0
assert np.array_equal(ids.cpu().numpy().view(np.uint32), want[1])
t.release()
torch.cuda.synchronize()
print("sanitize workload ok")
