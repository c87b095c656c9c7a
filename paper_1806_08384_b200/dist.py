"""Multi-GPU plumbing: one process per GPU, rows sharded contiguously.

Rank r of P owns rows [floor(rN/P), floor((r+1)N/P)) and registers them with
global_row_offset = floor(rN/P). libsel combines the shards itself over NCCL (one 8-byte
all-reduce per count, one P x 8-byte all-gather per push-down); torch.distributed is used only
to hand rank 0's ncclUniqueId to every rank (any backend: gloo or nccl) and for barriers.
"""

from __future__ import annotations

import torch.distributed as dist

from .api import Context, Table


def shard_range(n: int, world: int, rank: int) -> tuple:
    """Contiguous row range [start, end) of `rank` among `world` ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return n * rank // world, n * (rank + 1) // world


def broadcast_unique_id(unique_id: bytes | None, group=None) -> bytes:
    """Rank 0's 128-byte ncclUniqueId delivered to every rank of `group`."""
    obj = [unique_id if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad ncclUniqueId broadcast")
    return bytes(uid)


def setup_comm(ctx: Context, group=None) -> Context:
    """Make `ctx` one rank of the current torch.distributed group (collective)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    uid = broadcast_unique_id(Context.new_unique_id() if rank == 0 else None, group)
    ctx.set_comm(world, rank, uid)
    return ctx


def setup_peers(ctx: Context, group=None) -> Context:
    """Make `ctx` one rank of the current group over peer memory (collective): every rank's
    exchange-buffer IPC handle is all-gathered through torch.distributed and mapped by every
    other rank (include/sel.h sel_ctx_set_peers)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    handles = [None] * world
    dist.all_gather_object(handles, ctx.peer_handle(), group=group)
    ctx.set_peers(world, rank, handles)
    return ctx


def setup_exchange(ctx: Context, mechanism: str = "peers", group=None) -> str:
    """Join the group with one exchange mechanism that EVERY rank agrees on (collective):
    "peers" — the library's own exchange over peer memory (CUDA IPC + NVLink stores, fused into
    the count and push-down kernels; include/sel.h sel_ctx_set_peers) when every rank can map
    every other rank's buffer and a real test exchange sees all ranks, else NCCL on every rank;
    "nccl" — the library's NCCL communicator (an 8-byte all-reduce per count, an all-gather per
    Execute). Every rank reaches every collective below whatever fails locally, so no rank is left
    waiting and no two ranks use different mechanisms. Returns a description of the mechanism."""
    import torch
    from selgen.program import Const, INT32, encode   # the test exchange's one-row program
    if mechanism not in ("peers", "nccl"):
        raise ValueError("mechanism must be 'peers' or 'nccl'")
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    ok, why, mapped = mechanism == "peers", f"requested {mechanism}", False
    if ok:
        try:
            h = ctx.peer_handle()
        except Exception as ex:  # noqa: BLE001 - any failure falls back to NCCL on every rank
            h, ok, why = None, False, f"peers unavailable: {type(ex).__name__}: {ex}"
        handles = [None] * world
        dist.all_gather_object(handles, h, group=group)
        if ok and all(x is not None for x in handles):
            try:
                ctx.set_peers(world, rank, handles)
                mapped = True
                one = torch.zeros(1, dtype=torch.int32, device=ctx.device)
                probe = Table(ctx, ["x"], [INT32], [one], row_offset=rank, global_rows=world)
                got = probe.count(encode(Const(True), [INT32]))
                probe.release()
                if got != world:
                    ok, why = False, f"peer exchange counted {got} of {world}"
            except Exception as ex:  # noqa: BLE001
                ok, why = False, f"peers unavailable: {type(ex).__name__}: {ex}"
        else:
            ok = False
            if why.startswith("requested"):
                why = "a rank could not export its buffer"
        on_cpu = dist.get_backend(group) == "gloo"
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                            device="cpu" if on_cpu else ctx.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if not bool(flag.item()):
            if mapped:
                ctx.drop_peers()
            if ok:
                why = "another rank could not map the peers' buffers"
            ok = False
    if ok:
        return "peers (CUDA IPC, NVLink release stores, fused into the count kernel)"
    setup_comm(ctx, group)
    return f"nccl ({why})"


def gather_execute(table: Table, pred, project, max_size: int, root: int = 0, group=None):
    """Algorithm 1's Execute over the sharded table with the result gathered on rank `root`
    (SURVEY §8e's optional gather-to-one-rank): the root allocates the global outputs
    (min(max_size, global rows) rows), every rank maps them (CUDA IPC over NVLink/NVSwitch) and
    its materialisation kernel writes its rows straight into them at its offset
    (include/sel.h sel_execute_to). Collective. Returns (global count, materialized, and on the
    root the rowids tensor and the {column: tensor} of the whole ascending result; None
    elsewhere)."""
    import torch
    ctx = table.ctx
    rank = dist.get_rank(group)
    proj = table._col_indices(project)
    cap = int(min(max_size, table.global_rows))
    out = None
    handles = None
    if rank == root:
        from .api import _OUT_DTYPE
        dev = ctx.device
        out = (torch.empty(max(cap, 1), dtype=torch.int32, device=dev),
               [torch.empty(max(cap, 1), dtype=_OUT_DTYPE[table.types[j]], device=dev) for j in proj])
        handles = [ctx.export_buffer(out[0])] + [ctx.export_buffer(t) for t in out[1]]
    obj = [handles]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, root) if group else root,
                               group=group)
    handles = obj[0]
    if rank == root:
        ptrs = [out[0].data_ptr()] + [t.data_ptr() for t in out[1]]
    else:
        ptrs = [ctx.import_buffer(h) for h in handles]
    count, _, _, mat = table.execute_to(pred, project, max_size, cap, ptrs[0], ptrs[1:])
    torch.cuda.synchronize(ctx.device)
    dist.barrier(group)          # every rank's stores are complete before the root reads
    if rank != root:
        return count, mat, None, None
    k = min(count, cap) if mat else 0
    keys = [table.names[j] if isinstance(p, str) else j for p, j in zip(project, proj)]
    return count, mat, out[0][:k], {key: t[:k] for key, t in zip(keys, out[1])}


def exclusive_offset(local_counts, rank: int) -> int:
    """Position of rank `rank`'s slice in the rank-ordered (= ascending row id) concatenation."""
    return int(sum(local_counts[:rank]))


def register_shard(ctx: Context, names, types, tensors, global_rows: int, dicts=None,
                   group=None) -> Table:
    """Register this rank's shard; its row offset follows shard_range."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    start, end = shard_range(global_rows, world, rank)
    if tensors and tensors[0].numel() != end - start:
        raise ValueError(f"rank {rank} holds {tensors[0].numel()} rows, expected {end - start}")
    return Table(ctx, names, types, tensors, dicts=dicts, row_offset=start, global_rows=global_rows)
