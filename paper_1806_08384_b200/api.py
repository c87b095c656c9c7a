"""Python API over libsel (argument marshalling only; torch provides device memory and streams).

    ctx = Context()                                   # one per process / GPU
    t = Table.from_tensors(ctx, {"A": a, "B": b, "C": c}, dicts={"C": [...]})
    n = t.count((col("A") == 2) & (col("B") < 2001) & (col("B") > 1000) & col("C").isin([1, 4]))
    res = t.pushdown(pred, project=["A", "C", "D"])    # count first, then materialise (Alg. 1)
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _native
from ._native import SEL_ERR, SelError, check, last_error, lib, sel_column
from .predicate import (Expr, compile_predicate, INT32, INT64, FLOAT32, DATE32, DICT8, DICT16,
                        DICT32)

_DEFAULT_TYPE = {torch.int32: INT32, torch.int64: INT64, torch.float32: FLOAT32,
                 torch.uint8: DICT8, torch.int16: DICT16, torch.uint16: DICT16}
_WIDTH = {INT32: 4, INT64: 8, FLOAT32: 4, DATE32: 4, DICT8: 1, DICT16: 2, DICT32: 4}
_OUT_DTYPE = {INT32: torch.int32, INT64: torch.int64, FLOAT32: torch.float32, DATE32: torch.int32,
              DICT8: torch.uint8, DICT16: torch.int16, DICT32: torch.int32}


def _fit_capacity(capacity, default: int, out) -> int:
    """Rows the kernels may write: `capacity`, or `default` when None; never more than the caller's
    buffers hold when `out` = (rowids, [columns]) is given (a larger explicit capacity would let
    the kernels write past them: refused)."""
    if out is None:
        return int(default if capacity is None else capacity)
    rowids, outs = out
    room = min([int(rowids.numel())] + [int(o.numel()) for o in outs])
    if capacity is None:
        return min(int(default), room)
    if int(capacity) > room:
        raise ValueError(f"capacity {capacity} exceeds the output buffers ({room} rows)")
    return int(capacity)


def _stream_ptr(stream, device) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


class Context:
    """A libsel context bound to one CUDA device (one process per GPU)."""

    def __init__(self, device=None):
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", int(torch.device(device).index if not isinstance(device, int) else device))
        h = ctypes.c_void_p()
        check(lib().sel_ctx_create(self.device.index, ctypes.byref(h)))
        self._h = h
        self.nranks, self.rank = 1, 0

    @staticmethod
    def new_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(lib().sel_nccl_unique_id(buf))
        return buf.raw

    def set_comm(self, nranks: int, rank: int, unique_id: bytes) -> None:
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        check(lib().sel_ctx_set_comm(self._h, nranks, rank, buf))
        self.nranks, self.rank = nranks, rank

    def peer_handle(self) -> bytes:
        """This rank's 64-byte CUDA IPC handle of its exchange buffer (include/sel.h)."""
        buf = ctypes.create_string_buffer(64)
        check(lib().sel_ctx_peer_handle(self._h, buf))
        return buf.raw

    def set_peers(self, nranks: int, rank: int, handles) -> None:
        """Exchange counts over peer memory with the ranks whose handles are given (one per rank,
        in rank order): the library's own collective, replacing NCCL for every combination."""
        handles = [bytes(h) for h in handles]
        if len(handles) != nranks or any(len(h) != 64 for h in handles):
            raise ValueError("need nranks 64-byte handles")
        buf = ctypes.create_string_buffer(b"".join(handles), 64 * nranks)
        check(lib().sel_ctx_set_peers(self._h, nranks, rank, buf))
        self.nranks, self.rank = nranks, rank

    def set_peer_timeout(self, ms: int) -> None:
        """Bound of the peer exchange's waits (include/sel.h sel_ctx_set_peer_timeout): a rank
        that does not take part within `ms` fails the probe (and, sticky, every later one until
        the peers are dropped and set again) instead of hanging."""
        check(lib().sel_ctx_set_peer_timeout(self._h, int(ms)))

    def drop_peers(self) -> None:
        """Unmap the other ranks' exchange buffers (every rank before any rank closes)."""
        check(lib().sel_ctx_set_peers(self._h, 0, 0, None))

    def export_buffer(self, tensor: torch.Tensor) -> bytes:
        """72-byte handle of a device tensor's memory for other ranks (include/sel.h)."""
        buf = ctypes.create_string_buffer(72)
        check(lib().sel_ctx_export_buffer(self._h, ctypes.c_void_p(tensor.data_ptr()), buf))
        return buf.raw

    def import_buffer(self, handle: bytes) -> int:
        """Map another rank's exported buffer; returns the device pointer (an int)."""
        out = ctypes.c_void_p(0)
        buf = ctypes.create_string_buffer(bytes(handle), 72)
        check(lib().sel_ctx_import_buffer(self._h, buf, ctypes.byref(out)))
        return int(out.value)

    def enable_timing(self, on: bool = True) -> None:
        check(lib().sel_ctx_set_timing(self._h, 1 if on else 0))

    def set_option(self, name: str, value: int) -> None:
        """A tuning switch of this context (include/sel.h sel_ctx_set_option)."""
        check(lib().sel_ctx_set_option(self._h, name.encode(), int(value)))

    def last_times(self) -> tuple:
        """(count kernel ms, push-down kernels ms) of the most recent probes (timing enabled)."""
        c, p = ctypes.c_float(0.0), ctypes.c_float(0.0)
        check(lib().sel_ctx_last_times(self._h, ctypes.byref(c), ctypes.byref(p)))
        return float(c.value), float(p.value)

    def last_pushdown_path(self) -> int:
        """1: the last pushdown materialised from a kept selection; 2: two passes inside the call
        (keeping count, then 1's materialisation); 0: single pass; -1: none."""
        return int(lib().sel_ctx_last_pushdown_path(self._h))

    def last_pushdown_flags(self) -> int:
        """SEL_PD_* bits of the last materialisation from a kept selection (include/sel.h):
        coded / whole-chunk copies / constant fills / kept values; diagnostics."""
        return int(lib().sel_ctx_last_pushdown_flags(self._h))

    def set_pushdown_path(self, mode: int) -> None:
        """Path of a pushdown without a matching kept selection: -1 automatic (two passes at
        >= 3·2^20 local rows), 0 always the single pass, 2 always two passes (include/sel.h)."""
        check(lib().sel_ctx_set_pushdown_path(self._h, int(mode)))

    def register_bitmap(self, words: torch.Tensor, nbits: int) -> int:
        """Register a key set for IN_BITMAP leaves (selgen.InSet): `words` is a device tensor of
        ceil(nbits/64) 64-bit words (bit i = key i), kept alive by this context until
        release_bitmap. Returns the id programs refer to."""
        if not words.is_cuda or words.element_size() != 8 or not words.is_contiguous():
            raise ValueError("bitmap words must be a contiguous 64-bit CUDA tensor")
        if words.numel() * 64 < nbits:
            raise ValueError("bitmap shorter than nbits")
        out = ctypes.c_uint32(0)
        check(lib().sel_bitmap_register(self._h, ctypes.c_void_p(words.data_ptr()), int(nbits),
                                        ctypes.byref(out)))
        self._bitmaps = getattr(self, "_bitmaps", {})
        self._bitmaps[out.value] = words
        return int(out.value)

    def release_bitmap(self, bitmap_id: int) -> None:
        check(lib().sel_bitmap_release(self._h, int(bitmap_id)))
        getattr(self, "_bitmaps", {}).pop(int(bitmap_id), None)

    def last_kernel_ms(self) -> float:
        ms = ctypes.c_float(0.0)
        check(lib().sel_ctx_last_kernel_ms(self._h, ctypes.byref(ms)))
        return float(ms.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().sel_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class PushdownResult:
    rowids: torch.Tensor          # uint32 global row ids (as int32 storage), ascending
    columns: dict                 # name -> tensor of projected values
    count: int                    # global count (all ranks)
    local_count: int              # rows selected in this shard (may exceed capacity)
    offset: int                   # exclusive prefix over ranks (position of this shard's slice)

    @property
    def gated(self) -> bool:
        """Algorithm 1's 'count > maxSize' outcome: output truncated."""
        return self.local_count > self.rowids.numel()


@dataclass
class ExecuteResult(PushdownResult):
    materialized: bool = True     # False: count > max_size, Algorithm 1's "throw" (revert)


class PreparedExecute:
    """A prepared Algorithm 1 Execute (Table.prepare_execute). run() returns the global count;
    .materialized / .local_count describe the last run and .result() views its output."""

    def __init__(self, table, pred, project, max_size, capacity, stream, out):
        self.table = table
        prog = table.program(pred)
        proj = table._col_indices(project)
        if max_size is None:
            max_size = (1 << 64) - 2
        capacity = _fit_capacity(capacity, min(int(max_size), table.local_rows), out)
        dev = table.ctx.device
        if out is None:
            rowids = torch.empty(max(capacity, 1), dtype=torch.int32, device=dev)
            outs = [torch.empty(max(capacity, 1), dtype=_OUT_DTYPE[table.types[j]], device=dev) for j in proj]
        else:
            rowids, outs = out
        self.rowids, self.outs, self.capacity = rowids, list(outs), int(capacity)
        self._keys = [table.names[j] if isinstance(p, str) else j for p, j in zip(project, proj)]
        ptrs = (ctypes.c_void_p * max(len(outs), 1))(*[o.data_ptr() for o in outs])
        pj = (ctypes.c_uint32 * max(len(proj), 1))(*proj)
        h = ctypes.c_void_p()
        check(lib().sel_prepare_execute(table._h, prog, len(prog), pj, len(proj), int(max_size),
                                        rowids.data_ptr(), ptrs, int(capacity), ctypes.byref(h)))
        self._h = h
        self._local, self._off, self._mat = ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_int(0)
        self._refs = (ctypes.byref(self._local), ctypes.byref(self._off), ctypes.byref(self._mat))
        self._stream = _stream_ptr(stream, dev)
        self._fn = lib().sel_prepared_execute
        self._fn_async = lib().sel_prepared_execute_async
        self.count = 0

    def run(self, stream=None, wait: bool = True) -> int:
        """One Execute. wait=False returns once the count is final on the host
        (sel_prepared_execute_async): the materialisation completes in stream order."""
        fn = self._fn if wait else self._fn_async
        r = fn(self._h, *self._refs, self._stream if stream is None else _stream_ptr(stream, self.table.ctx.device))
        if r == SEL_ERR:
            raise last_error()
        self.count = r
        return r

    @property
    def materialized(self) -> bool:
        return bool(self._mat.value)

    @property
    def local_count(self) -> int:
        return int(self._local.value)

    def result(self) -> "ExecuteResult":
        k = min(self.local_count, self.capacity)
        cols = {key: o[:k] for key, o in zip(self._keys, self.outs)}
        return ExecuteResult(self.rowids[:k], cols, int(self.count), self.local_count,
                             int(self._off.value), self.materialized)

    def release(self) -> None:
        if getattr(self, "_h", None):
            lib().sel_prepared_release(self._h)
            self._h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class Table:
    """A registered table shard: rows [row_offset, row_offset + local_rows) of global_rows."""

    def __init__(self, ctx: Context, names: Sequence[str], types: Sequence[int],
                 tensors: Sequence[torch.Tensor], dicts: Mapping[str, list] | None = None,
                 row_offset: int = 0, global_rows: int | None = None):
        if not tensors:
            raise ValueError("a table needs at least one column")
        n = tensors[0].numel()
        for name, t, x in zip(names, types, tensors):
            if not x.is_cuda or x.device != ctx.device:
                raise ValueError(f"column {name} must live on {ctx.device}")
            if x.dim() != 1 or not x.is_contiguous() or x.numel() != n:
                raise ValueError(f"column {name} must be 1-D, contiguous, with {n} rows")
            if x.element_size() != _WIDTH[t]:
                raise ValueError(f"column {name}: element size {x.element_size()} != {_WIDTH[t]}")
        self.ctx = ctx
        self.names = list(names)
        self.types = [int(t) for t in types]
        self.tensors = list(tensors)          # keep the memory alive while registered
        self.dicts = dict(dicts or {})
        self.local_rows = n
        self.row_offset = int(row_offset)
        self.global_rows = int(global_rows if global_rows is not None else row_offset + n)
        arr = (sel_column * len(tensors))()
        for i, (t, x) in enumerate(zip(self.types, self.tensors)):
            arr[i].type = t
            arr[i].data = x.data_ptr() if n > 0 else None
            arr[i].dict_size = len(self.dicts.get(self.names[i], [])) if t in (DICT8, DICT16, DICT32) else 0
        h = ctypes.c_void_p()
        check(lib().sel_table_register(ctx._h, arr, len(tensors), n, self.row_offset,
                                       self.global_rows, ctypes.byref(h)))
        self._h = h

    @classmethod
    def from_tensors(cls, ctx: Context, columns, types: Mapping[str, int] | None = None,
                     dicts: Mapping[str, list] | None = None, row_offset: int = 0,
                     global_rows: int | None = None) -> "Table":
        items = list(columns.items()) if isinstance(columns, Mapping) else list(columns)
        types = dict(types or {})
        names = [k for k, _ in items]
        tensors = [v for _, v in items]
        tys = [types.get(k, _DEFAULT_TYPE.get(v.dtype)) for k, v in items]
        if any(t is None for t in tys):
            raise ValueError("column type could not be inferred; pass types={name: sel_type}")
        return cls(ctx, names, tys, tensors, dicts, row_offset, global_rows)

    @property
    def schema(self):
        return [(n, t, self.dicts.get(n)) for n, t in zip(self.names, self.types)]

    def program(self, pred) -> bytes:
        if isinstance(pred, (bytes, bytearray)):
            return bytes(pred)
        return compile_predicate(pred, self.schema)

    def count(self, pred, stream=None, keep_selection: bool = False, keep_columns=()) -> int:
        """Exact |sigma_P(R)| (Listing 3.1); global over ranks. With
        keep_selection the probe keeps its selection (and the selected values of the projected
        predicate columns named in keep_columns) so that a following pushdown() of the same
        predicate materialises without re-evaluating it."""
        prog = self.program(pred)
        keep = self._col_indices(keep_columns)
        arr = (ctypes.c_uint32 * max(len(keep), 1))(*keep)
        r = lib().sel_count_ex(self._h, prog, len(prog), _native.SEL_KEEP_SELECTION if keep_selection else 0,
                               arr, len(keep), _stream_ptr(stream, self.ctx.device))
        if r == SEL_ERR:
            raise last_error()
        return int(r)

    def count_async(self, pred, out: torch.Tensor, stream=None) -> torch.Tensor:
        """Enqueue the count without waiting: the global count lands in `out` (a one-element
        int64 CUDA tensor) when `stream` reaches it — capturable into a CUDA graph
        (include/sel.h sel_count_async). Enqueue a context's probes on one stream."""
        if not out.is_cuda or out.dtype != torch.int64 or out.numel() < 1:
            raise ValueError("out must be a CUDA int64 tensor")
        prog = self.program(pred)
        check(lib().sel_count_async(self._h, prog, len(prog), out.data_ptr(),
                                    _stream_ptr(stream, self.ctx.device)))
        return out

    def histogram(self, column, buckets: int = 64, stride: int = 1, phase: int = 0,
                  stream=None) -> dict:
        """Equi-depth histogram of an integer column over a block sample (
        include/sel.h sel_histogram): numpy arrays lo, hi (values), rows, distinct per bucket,
        and sample_rows. Local shard."""
        col = self._col_indices([column])[0]
        lo = np.zeros(buckets, np.int64)
        hi = np.zeros(buckets, np.int64)
        rows = np.zeros(buckets, np.uint64)
        distinct = np.zeros(buckets, np.uint64)
        m = ctypes.c_uint64(0)
        ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
        check(lib().sel_histogram(self._h, col, int(stride), int(phase), int(buckets), ptr(lo),
                                  ptr(hi), ptr(rows), ptr(distinct), ctypes.byref(m),
                                  _stream_ptr(stream, self.ctx.device)))
        return {"lo": lo, "hi": hi, "rows": rows, "distinct": distinct,
                "sample_rows": int(m.value), "table_rows": self.local_rows}

    def count_batch(self, preds, stream=None) -> list:
        """Exact counts of several predicates in ONE scan: each column read
        once, each distinct leaf evaluated once; e.g. the worked example's four leaves and their
        conjunction."""
        progs = [self.program(p) for p in preds]
        bufs = [ctypes.create_string_buffer(b, len(b)) for b in progs]
        ptrs = (ctypes.c_void_p * len(progs))(*[ctypes.addressof(b) for b in bufs])
        lens = (ctypes.c_size_t * len(progs))(*[len(b) for b in progs])
        out = (ctypes.c_uint64 * len(progs))()
        check(lib().sel_count_batch(self._h, ptrs, lens, len(progs), out,
                                    _stream_ptr(stream, self.ctx.device)))
        return [int(x) for x in out]

    def count_sampled(self, pred, stride: int, phase: int = 0, stream=None) -> tuple:
        """Exact count over the block sample of chunks c = phase (mod stride);
        returns (sample count, sample rows, estimate = count * rows / sample rows) — the sampling
        estimator of PAPER.md:199-203, to set beside the exact probe."""
        prog = self.program(pred)
        rows = ctypes.c_uint64(0)
        r = lib().sel_count_sampled(self._h, prog, len(prog), int(stride), int(phase),
                                    ctypes.byref(rows), _stream_ptr(stream, self.ctx.device))
        if r == SEL_ERR:
            raise last_error()
        est = lib().sel_sample_estimate(int(r), int(rows.value), self.global_rows)
        return int(r), int(rows.value), float(est)

    def _col_indices(self, cols):
        return [self.names.index(p) if isinstance(p, str) else int(p) for p in cols]

    def execute(self, pred, project: Sequence[str | int] = (), max_size: int | None = None,
                capacity: int | None = None, stream=None, out=None) -> "ExecuteResult":
        """Algorithm 1's Execute(compound, isSPD=true, maxSize): count keeping
        the selection, then "throw" if count > max_size (result.materialized is False, nothing
        written) else materialise. capacity (rows of the output buffers) defaults to
        min(max_size, local rows)."""
        prog = self.program(pred)
        proj = self._col_indices(project)
        if max_size is None:
            max_size = (1 << 64) - 2
        capacity = _fit_capacity(capacity, min(int(max_size), self.local_rows), out)
        dev = self.ctx.device
        if out is None:
            rowids = torch.empty(max(capacity, 1), dtype=torch.int32, device=dev)
            outs = [torch.empty(max(capacity, 1), dtype=_OUT_DTYPE[self.types[j]], device=dev) for j in proj]
        else:
            rowids, outs = out
        ptrs = (ctypes.c_void_p * max(len(outs), 1))(*[o.data_ptr() for o in outs])
        pj = (ctypes.c_uint32 * max(len(proj), 1))(*proj)
        local, off, mat = ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_int(0)
        r = lib().sel_execute(self._h, prog, len(prog), pj, len(proj), int(max_size), rowids.data_ptr(),
                              ptrs, capacity, ctypes.byref(local), ctypes.byref(off), ctypes.byref(mat),
                              _stream_ptr(stream, dev))
        if r == SEL_ERR:
            raise last_error()
        k = min(int(local.value), capacity)
        cols = {self.names[j] if isinstance(p, str) else j: o[:k] for p, j, o in zip(project, proj, outs)}
        return ExecuteResult(rowids[:k], cols, int(r), int(local.value), int(off.value), bool(mat.value))

    def execute_to(self, pred, project: Sequence[str | int], max_size: int, capacity: int,
                   rowids_ptr: int, col_ptrs: Sequence[int], stream=None) -> tuple:
        """Execute writing into the GLOBAL result at this rank's offset (include/sel.h
        sel_execute_to): rowids_ptr / col_ptrs are device pointers of the global output buffers
        as this context sees them (sel_ctx_import_buffer for another rank's memory); capacity is
        their global row capacity. Returns (global count, local count, offset, materialized).
        dist.gather_execute wraps the whole gather-to-one-rank."""
        prog = self.program(pred)
        proj = self._col_indices(project)
        ptrs = (ctypes.c_void_p * max(len(proj), 1))(*[int(x) for x in col_ptrs])
        pj = (ctypes.c_uint32 * max(len(proj), 1))(*proj)
        local, off, mat = ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_int(0)
        r = lib().sel_execute_to(self._h, prog, len(prog), pj, len(proj), int(max_size),
                                 int(rowids_ptr), ptrs, int(capacity), ctypes.byref(local),
                                 ctypes.byref(off), ctypes.byref(mat),
                                 _stream_ptr(stream, self.ctx.device))
        if r == SEL_ERR:
            raise last_error()
        return int(r), int(local.value), int(off.value), bool(mat.value)

    def prepare_execute(self, pred, project: Sequence[str | int] = (), max_size: int | None = None,
                        capacity: int | None = None, stream=None, out=None) -> "PreparedExecute":
        """execute() with every argument fixed: validated once and captured into a CUDA graph
        (include/sel.h sel_prepare_execute); each .run() is one graph launch + one sync."""
        return PreparedExecute(self, pred, project, max_size, capacity, stream, out)

    def pushdown(self, pred, project: Sequence[str | int] = (), capacity: int | None = None,
                 stream=None, out=None) -> PushdownResult:
        """Materialise sigma_P pi_project(R). capacity=None sizes the output
        exactly from a count probe first (Algorithm 1's order: count, then execute); an integer
        capacity is the single-pass gated form (count > capacity => truncated, see `.gated`)."""
        prog = self.program(pred)
        proj = [self.names.index(p) if isinstance(p, str) else int(p) for p in project]
        if capacity is None and out is None:
            capacity = self._local_count(prog, stream, proj)
        elif capacity is None:
            capacity = _fit_capacity(None, self._local_count(prog, stream, proj), out)
        else:
            capacity = _fit_capacity(capacity, capacity, out)
        dev = self.ctx.device
        if out is None:
            rowids = torch.empty(max(capacity, 1), dtype=torch.int32, device=dev)
            outs = [torch.empty(max(capacity, 1), dtype=_OUT_DTYPE[self.types[j]], device=dev) for j in proj]
        else:
            rowids, outs = out
        ptrs = (ctypes.c_void_p * max(len(outs), 1))(*[o.data_ptr() for o in outs])
        pj = (ctypes.c_uint32 * max(len(proj), 1))(*proj)
        local = ctypes.c_uint64(0)
        off = ctypes.c_uint64(0)
        r = lib().sel_pushdown(self._h, prog, len(prog), pj, len(proj), rowids.data_ptr(), ptrs,
                               capacity, ctypes.byref(local), ctypes.byref(off),
                               _stream_ptr(stream, dev))
        if r == SEL_ERR:
            raise last_error()
        k = min(int(local.value), capacity)
        cols = {self.names[j] if isinstance(p, str) else j: o[:k]
                for p, j, o in zip(project, proj, outs)}
        return PushdownResult(rowids[:k], cols, int(r), int(local.value), int(off.value))

    def _local_count(self, prog: bytes, stream, keep_columns=()) -> int:
        # Algorithm 1's order: count first (keeping the selection for the materialisation)
        c = self.count(prog, stream, keep_selection=True, keep_columns=keep_columns)
        if self.ctx.nranks == 1:
            return c
        # local count of this shard: a push-down with capacity 0 returns it without writing
        local = ctypes.c_uint64(0)
        r = lib().sel_pushdown(self._h, prog, len(prog), None, 0, None, None, 0,
                               ctypes.byref(local), None, _stream_ptr(stream, self.ctx.device))
        if r == SEL_ERR:
            raise last_error()
        return int(local.value)

    def release(self) -> None:
        if getattr(self, "_h", None):
            lib().sel_table_release(self._h)
            self._h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def program_check(prog: bytes, types: Sequence[int]) -> int:
    """Validation status of a program against column types (host only, no GPU needed)."""
    arr = (ctypes.c_int * max(len(types), 1))(*types)
    return int(lib().sel_program_check(prog, len(prog), arr, len(types)))


def program_path(prog: bytes, types: Sequence[int]) -> int:
    arr = (ctypes.c_int * max(len(types), 1))(*types)
    return int(lib().sel_program_path(prog, len(prog), arr, len(types)))


def equi_depth_estimate(hist: dict, value: int) -> float:
    """The paper's equi-depth equality estimate from a Table.histogram() result:
    include/sel.h sel_equi_depth_estimate (D / V(b_x), D = T(R) / B, summed over every bucket whose
    [lo, hi] holds x). A synopsis baseline to set beside the exact count."""
    lo = np.ascontiguousarray(hist["lo"], dtype=np.int64)
    hi = np.ascontiguousarray(hist["hi"], dtype=np.int64)
    dv = np.ascontiguousarray(hist["distinct"], dtype=np.uint64)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    return float(lib().sel_equi_depth_estimate(ptr(lo), ptr(hi), ptr(dv), len(lo),
                                               int(hist["table_rows"]), int(value)))


def program_plan(prog: bytes, types: Sequence[int]) -> dict:
    """The canonical device plan (include/sel.h sel_program_plan_json) as a dict."""
    import json
    arr = (ctypes.c_int * max(len(types), 1))(*types)
    n = lib().sel_program_plan_json(prog, len(prog), arr, len(types), None, 0)
    if n < 0:
        raise SelError(-n, "invalid program")
    buf = ctypes.create_string_buffer(n + 1)
    lib().sel_program_plan_json(prog, len(prog), arr, len(types), buf, n + 1)
    return json.loads(buf.value.decode())
