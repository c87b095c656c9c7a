"""Multi-rank probes for real, on one GPU: 2 and 3 processes share cuda:0 and combine their
shards over the library's own peer-memory exchange (include/sel.h sel_ctx_set_peers — CUDA IPC
maps a buffer of the same device too; NCCL would refuse two ranks on one GPU). Every cross-rank
path runs: count sums, push-down offsets (single pass and two passes), Execute's one exchange
(device-gated, host-gated on empty shards and constant programs, gated and not), prepared
(graph) executes, batch and sampled counts. Rank 0 checks the rank-ordered concatenation against
the oracle over the whole table (ascending global row ids, bit-exact)."""

import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_global, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    import oracle
    import paper_1806_08384_b200 as sel
    from paper_1806_08384_b200 import dist as sdist
    from selgen import configs
    from selgen.program import Cmp, Const, encode

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    ctx = sel.Context(dev)
    sdist.setup_peers(ctx)
    s, e = sdist.shard_range(n_global, world, rank)
    types, host = _table(n_global)
    names = ["A", "B", "C", "D"]
    t = sel.Table(ctx, names, types, [torch.from_numpy(h[s:e].copy()).to(dev) for h in host],
                  row_offset=s, global_rows=n_global)
    progs = [encode(p, types) for p in configs.c2_probes().values()]
    progs += [encode(Cmp("=", 0, 99), types), encode(Const(True), types),
              encode(Cmp(">", 3, 0), types)]
    rec = []
    for prog in progs:
        r = {"count": t.count(prog)}
        for mode in (0, 2):
            ctx.set_pushdown_path(mode)
            pd = t.pushdown(prog, project=["C", "D"])
            ctx.set_pushdown_path(-1)
            r[f"pd{mode}"] = (pd.count, pd.offset, pd.rowids.cpu().numpy().view(np.uint32).copy(),
                              pd.columns["D"].cpu().numpy().copy())
        ex = t.execute(prog, project=["C", "D"], max_size=n_global)
        r["ex"] = (ex.count, ex.offset, ex.materialized, ex.rowids.cpu().numpy().view(np.uint32).copy())
        g = t.execute(prog, project=["D"], max_size=max(r["count"] - 1, 0), capacity=8)
        r["gated"] = (g.count, g.materialized)
        q = t.prepare_execute(prog, project=["D"], max_size=n_global)
        c1, c2 = q.run(), q.run(wait=False)   # the second returns at its count (async)
        torch.cuda.synchronize()
        res = q.result()
        r["prep"] = (c1, c2, res.offset, res.rowids.cpu().numpy().view(np.uint32).copy())
        q.release()
        r["sampled"] = t.count_sampled(prog, 3, 1)[:2]
        rec.append(r)
    r_batch = t.count_batch(progs[:5])
    # gather to one rank: every rank's materialisation writes into the root's buffers (P2P)
    keep_alive = []
    for i, prog in enumerate(progs):
        root = i % world
        cnt, mat, ids, cols = sdist.gather_execute(t, prog, ["C", "D"], max_size=n_global, root=root)
        keep_alive.append((ids, cols))
        if rank == root:
            want_c, want_ids, want_cols = oracle.pushdown(host, types, prog, proj=[2, 3])
            assert cnt == want_c and mat, ("gather", i)
            np.testing.assert_array_equal(ids.cpu().numpy().view(np.uint32), want_ids)
            np.testing.assert_array_equal(cols["C"].cpu().numpy(), want_cols[0])
            np.testing.assert_array_equal(cols["D"].cpu().numpy(), want_cols[1])
    cnt, mat, ids, cols = sdist.gather_execute(t, progs[0], ["D"], max_size=0, root=0)
    keep_alive.append((ids, cols))
    want0 = oracle.count(host, types, progs[0])
    assert cnt == want0 and mat == (want0 == 0)
    torch.cuda.synchronize()
    gathered = [None] * world
    dist.all_gather_object(gathered, (rec, r_batch, s, e))
    if rank == 0:
        ok = []
        for i, prog in enumerate(progs):
            want_c, want_ids, want_cols = oracle.pushdown(host, types, prog, proj=[2, 3])
            ranks = [gathered[k][0][i] for k in range(world)]
            assert all(r["count"] == want_c for r in ranks), ("count", i)
            for key in ("pd0", "pd2"):
                assert all(r[key][0] == want_c for r in ranks), (key, i)
                ids = np.concatenate([r[key][2] for r in ranks])
                np.testing.assert_array_equal(ids, want_ids)
                np.testing.assert_array_equal(np.concatenate([r[key][3] for r in ranks]), want_cols[1])
                offs = [r[key][1] for r in ranks]
                assert offs == list(np.cumsum([0] + [len(r[key][2]) for r in ranks])[:-1]), (key, i)
            assert all(r["ex"][0] == want_c and r["ex"][2] for r in ranks)
            np.testing.assert_array_equal(np.concatenate([r["ex"][3] for r in ranks]), want_ids)
            assert [r["ex"][1] for r in ranks] == [r["pd0"][1] for r in ranks]
            assert all(r["gated"] == (want_c, want_c == 0) for r in ranks), ("gated", i)
            assert all(r["prep"][0] == r["prep"][1] == want_c for r in ranks), ("prep", i)
            np.testing.assert_array_equal(np.concatenate([r["prep"][3] for r in ranks]), want_ids)
            samp = [gathered[k][0][i]["sampled"] for k in range(world)]
            assert len({tuple(x) for x in samp}) == 1, ("sampled agree", i)
            ok.append(i)
        batch = gathered[0][1]
        assert all(gathered[k][1] == batch for k in range(world))
        assert list(batch) == [oracle.count(host, types, p) for p in progs[:5]]
        with open(out_path, "w") as f:
            f.write(f"ok {len(ok)}\n")
    t.release()
    ctx.drop_peers()            # every rank unmaps the others' buffers before any rank frees its own
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def _table(n_global):
    """The worked example's R (C2 generator, n a multiple of 6,000) or, below that, a tiny table
    of the same column types; host arrays of the whole table (every rank builds the same)."""
    from selgen import configs
    from selgen.program import INT32, DICT8
    if n_global % 6000 == 0 and n_global > 0:
        T = configs.gen_c2(n_global, device="cpu")
        return T.types, [c.numpy() for c in T.columns]
    a = np.array([2, 5, 2][:n_global], np.int32)
    b = np.array([1500, 0, 2000][:n_global], np.int32)
    c = np.array([1, 4, 4][:n_global], np.uint8)
    d = np.array([10, 20, 30][:n_global], np.int32)
    return [INT32, INT32, DICT8, INT32], [a, b, c, d]


def _run(world, n_global, tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / f"peers_{world}_{n_global}.txt")
    mp.spawn(_worker, args=(world, _free_port(), n_global, out), nprocs=world, join=True)
    assert open(out).read().startswith("ok")


@pytest.mark.parametrize("world,n_global", [(2, 600_000), (3, 606_000)])
def test_peers_multi_rank_one_gpu(world, n_global, tmp_path, cuda_device):
    _run(world, n_global, tmp_path)


def test_peers_with_an_empty_shard(tmp_path, cuda_device):
    """Two rows over three ranks: rank 0 holds no row, so its Execute takes the host-gated path
    while the others gate on the device — the exchange sequence must still match."""
    _run(3, 2, tmp_path)


def _timeout_worker(rank, world, port, out_path):
    """A rank that skips an exchange: the other rank's probe times out. Its Execute must fail with
    SEL_E_STATE and write NOTHING (the failed exchange's sums are the failure marker, which the
    gated push-down kernels test) — into its own outputs (phase A, rank 0 alone) and into another
    rank's buffers through sel_execute_to (phase B, rank 1 alone); every later probe of the
    context fails at once (sticky); after every rank drops and re-sets its peers the group works
    again. (Each phase recovers before the next: a rank that wrote epoch e and timed out leaves
    its row behind, which a later lone exchange of the other rank at epoch e would accept —
    the recovery resets the epochs.)"""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_1806_08384_b200 as sel
    from paper_1806_08384_b200 import dist as sdist
    from selgen import configs
    from selgen.program import encode

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    ctx = sel.Context(dev)
    ctx.set_peer_timeout(300)
    sdist.setup_peers(ctx)
    n = 600_000
    T = configs.gen_c2(n, device="cpu")
    s, e = sdist.shard_range(n, world, rank)
    t = sel.Table(ctx, ["A", "B", "C", "D"], T.types,
                  [c.data[s:e].contiguous().to(dev) for c in T.columns], row_offset=s, global_rows=n)
    prog = encode(configs.c2_probes()["listing"], T.types)
    want = t.count(prog)                     # both ranks: a working exchange first
    ok = [want == n // 6000 * 1002]

    def fails(fn):
        try:
            fn()
            return "no error"
        except sel.SelError as ex:
            return ex.status == sel._native.SEL_E_STATE

    def recover():
        dist.barrier()
        ctx.drop_peers()
        dist.barrier()
        sdist.setup_peers(ctx)
        ok.append(t.count(prog) == want)

    # phase A: rank 0 alone; its local outputs stay untouched
    if rank == 0:
        ids = torch.full((want,), -7, dtype=torch.int32, device=dev)
        d = torch.full((want,), -7, dtype=torch.int32, device=dev)
        ok.append(fails(lambda: t.execute(prog, project=["D"], max_size=n, capacity=want,
                                          out=(ids, [d]))))
        torch.cuda.synchronize()
        ok.append(bool((ids == -7).all()) and bool((d == -7).all()))
        ok.append(fails(lambda: t.count(prog)))            # sticky
    recover()
    # phase B: rank 1 alone writes (would write) into rank 0's buffers over peer memory
    root_ids = torch.full((want,), -7, dtype=torch.int32, device=dev)
    root_d = torch.full((want,), -7, dtype=torch.int32, device=dev)
    hs = [[ctx.export_buffer(root_ids), ctx.export_buffer(root_d)] if rank == 0 else None]
    dist.broadcast_object_list(hs, src=0)
    ptrs = ([root_ids.data_ptr(), root_d.data_ptr()] if rank == 0
            else [ctx.import_buffer(h) for h in hs[0]])
    dist.barrier()
    if rank == 1:
        ok.append(fails(lambda: t.execute_to(prog, ["D"], n, want, ptrs[0], ptrs[1:])))
        torch.cuda.synchronize()
        ok.append(fails(lambda: t.count(prog)))            # sticky
    dist.barrier()
    if rank == 0:
        ok.append(bool((root_ids == -7).all()) and bool((root_d == -7).all()))   # nothing stored
    recover()
    r = t.execute(prog, project=["D"], max_size=n)
    ok.append(r.materialized and r.count == want)
    torch.cuda.synchronize()
    res = [None] * world
    dist.all_gather_object(res, ok)
    if rank == 0:
        with open(out_path, "w") as f:
            f.write(("ok" if all(x is True for o in res for x in o) else "FAIL") + f" {res}\n")
    t.release()
    ctx.drop_peers()
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def test_peer_timeout_fails_without_writing(tmp_path, cuda_device):
    import torch.multiprocessing as mp
    out = str(tmp_path / "timeout.txt")
    mp.spawn(_timeout_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert open(out).read().startswith("ok"), open(out).read()
