"""The N > 1 host path on CPU: two processes over gloo (world_size 2, 127.0.0.1).

What runs here is everything of the multi-GPU path that is not a device collective: the
contiguous sharding, the ncclUniqueId hand-off from rank 0 (produced by libsel's own
sel_nccl_unique_id, which needs no GPU) and the count / offset combination the library performs
with NCCL (sum of local counts; exclusive prefix of local counts in rank order). Each rank's
local probe is the CPU oracle on its shard (tests may use it); the combined result must equal the
unsharded oracle result: count and the ascending concatenation of row ids.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1806_08384_b200 import dist as sdist
        from paper_1806_08384_b200 import Context
        from selgen import configs, encode

        uid = sdist.broadcast_unique_id(Context.new_unique_id() if rank == 0 else None)
        ids_all = [None] * world
        dist.all_gather_object(ids_all, uid)
        assert all(u == uid for u in ids_all) and len(uid) == 128

        start, end = sdist.shard_range(n, world, rank)
        T = configs.gen_c2(n, start, end - start)             # this rank's shard only
        cols = [c.numpy() for c in T.columns]
        results = {}
        for name, node in configs.c2_probes().items():
            prog = encode(node, T.types)
            local, ids, (d,) = oracle.pushdown(cols, T.types, prog, proj=[3], row_offset=start)
            total = torch.tensor([local], dtype=torch.int64)
            dist.all_reduce(total)                                # the count all-reduce (a4)
            counts = [None] * world
            dist.all_gather_object(counts, local)                 # the offset all-gather (a7)
            off = sdist.exclusive_offset(counts, rank)
            results[name] = (int(total.item()), off, ids, d)
        q.put((rank, start, end, results))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [600_000, 6_000 * 37])
def test_two_rank_shards_combine_to_the_unsharded_result(n):
    import oracle
    from selgen import configs, encode
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict()
    for _ in range(world):
        rank, s, e, res = q.get(timeout=300)
        out[rank] = (s, e, res)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][0] == 0 and out[0][1] == out[1][0] and out[1][1] == n
    T = configs.gen_c2(n)
    cols = [c.numpy() for c in T.columns]
    for name, node in configs.c2_probes().items():
        want_c, want_ids, (want_d,) = oracle.pushdown(cols, T.types, encode(node, T.types), proj=[3])
        tot0, off0, ids0, d0 = out[0][2][name]
        tot1, off1, ids1, d1 = out[1][2][name]
        assert tot0 == tot1 == want_c
        assert off0 == 0 and off1 == len(ids0)
        np.testing.assert_array_equal(np.concatenate([ids0, ids1]), want_ids)
        np.testing.assert_array_equal(np.concatenate([d0, d1]), want_d)


def test_shard_range_partitions():
    from paper_1806_08384_b200.dist import shard_range
    for n in [0, 1, 7, 600_000_000, 2**32 - 1]:
        for world in [1, 2, 3, 4, 8]:
            r = [shard_range(n, world, k) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
            assert max(e - s for s, e in r) - min(e - s for s, e in r) <= 1


# ---- the choice of exchange at N > 1 (dist.setup_exchange, used by bench.py and the example) ---

def _exchange_worker(rank, world, port, scenario, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1806_08384_b200 import dist as sdist
        log = []

        class Ctx:
            device = "cpu"

            def peer_handle(self):
                if scenario == "handle" and rank == 1:
                    raise RuntimeError("no IPC")
                return bytes([rank]) * 64

            def set_peers(self, n, r, handles):
                assert len(handles) == n == world and r == rank
                if scenario == "map" and rank == 0:
                    raise RuntimeError("cudaIpcOpenMemHandle failed")
                log.append("mapped")

            def drop_peers(self):
                log.append("dropped")

        class Probe:
            def __init__(self, *a, **k):
                pass

            def count(self, prog):
                return world - 1 if (scenario == "verify" and rank == 1) else world

            def release(self):
                pass

        sdist.Table = Probe
        sdist.setup_comm = lambda ctx, group=None: log.append("nccl")
        got = sdist.setup_exchange(Ctx(), "nccl" if scenario == "nccl" else "peers")
        q.put((rank, got.split(" ")[0], log))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scenario,want", [("ok", "peers"), ("handle", "nccl"),
                                           ("map", "nccl"), ("verify", "nccl"), ("nccl", "nccl")])
def test_setup_exchange_agreement(scenario, want):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, scenario, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [want, want], res
    for rank, _, log in res:
        if want == "nccl":
            assert log[-1] == "nccl"
            if "mapped" in log:                     # a rank that mapped the others unmaps them
                assert "dropped" in log
        else:
            assert log == ["mapped"]
