"""oracle — TEST INFRASTRUCTURE ONLY (task rule ③).

The plain CPU oracle of the exact-selectivity probe (oracle/oracle.c, row-at-a-time postfix
evaluation) plus a separately written recursive AST
evaluator (oracle/ast_eval.py) for tiny brute-force cases. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may import this
package. The product path (paper_1806_08384_b200) never imports it and shares no code with it.

Parity status: every function here is pinned by tests/test_oracle_pins.py.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

STATUS = {0: "OK", 1: "E_ARG", 2: "E_ALIGN", 3: "E_TYPE", 4: "E_PROGRAM", 5: "E_TOO_LARGE"}
_WIDTH = {1: 4, 2: 8, 3: 4, 4: 4, 5: 1, 6: 2, 7: 4}
_NP = {1: np.int32, 2: np.int64, 3: np.float32, 4: np.int32, 5: np.uint8, 6: np.uint16,
       7: np.uint32}


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc -O2 (never -ffast-math: IEEE compares must stay exact)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
               "-ffp-contract=off", "-Wall", "-Wextra", "-o", _LIB + ".tmp", _SRC, "-lpthread"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64, vp, sz = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t
        ip = ctypes.POINTER(ctypes.c_int)
        L.oracle_check.restype = ctypes.c_int
        L.oracle_check.argtypes = [ctypes.c_char_p, sz, vp, ctypes.c_uint32]
        L.oracle_count.restype = u64
        L.oracle_count.argtypes = [vp, vp, ctypes.c_uint32, u64, ctypes.c_char_p, sz, ip]
        L.oracle_count_mt.restype = u64
        L.oracle_count_mt.argtypes = [vp, vp, ctypes.c_uint32, u64, ctypes.c_char_p, sz,
                                      ctypes.c_int, ip]
        L.oracle_pushdown.restype = u64
        L.oracle_pushdown.argtypes = [vp, vp, ctypes.c_uint32, u64, ctypes.c_char_p, sz, vp,
                                      ctypes.c_uint32, u64, vp, vp, u64, ip]
        L.oracle_count_mt_bm.restype = u64
        L.oracle_count_mt_bm.argtypes = [vp, vp, ctypes.c_uint32, u64, ctypes.c_char_p, sz,
                                         ctypes.c_int, vp, vp, ctypes.c_uint32, ip]
        L.oracle_count_bm.restype = u64
        L.oracle_count_bm.argtypes = [vp, vp, ctypes.c_uint32, u64, ctypes.c_char_p, sz, vp, vp,
                                      ctypes.c_uint32, ip]
        L.oracle_pushdown_mt_bm.restype = u64
        L.oracle_pushdown_mt_bm.argtypes = [vp, vp, ctypes.c_uint32, u64, ctypes.c_char_p, sz, vp,
                                            ctypes.c_uint32, u64, vp, vp, u64, ctypes.c_int, vp,
                                            vp, ctypes.c_uint32, ip]
        L.oracle_pushdown_bm.restype = u64
        L.oracle_pushdown_bm.argtypes = [vp, vp, ctypes.c_uint32, u64, ctypes.c_char_p, sz, vp,
                                         ctypes.c_uint32, u64, vp, vp, u64, vp, vp,
                                         ctypes.c_uint32, ip]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status):
        super().__init__(f"oracle status {STATUS.get(status, status)}")
        self.status = status


def _marshal(columns: Sequence, types: Sequence[int]):
    arrs = []
    for a, t in zip(columns, types):
        a = np.ascontiguousarray(np.asarray(a))
        if a.dtype != _NP[t]:
            if a.dtype.itemsize != _WIDTH[t]:
                raise TypeError(f"column of type {t} needs {_WIDTH[t]}-byte elements, got {a.dtype}")
            a = a.view(_NP[t])              # same bytes, the column type's value semantics
        arrs.append(a)
    ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    tys = np.asarray(types, dtype=np.int32)
    return arrs, ptrs, tys


def check(prog: bytes, types: Sequence[int]) -> int:
    """Validation status of `prog` against column types (include/sel.h order)."""
    tys = np.asarray(types, dtype=np.int32)
    return int(_load().oracle_check(prog, len(prog), tys.ctypes.data, len(types)))


def _bitmaps(bitmaps):
    """[(uint64 words, nbits), ...] -> ctypes arrays for the IN_BITMAP key sets (id = index)."""
    bitmaps = list(bitmaps or [])
    words = [np.ascontiguousarray(w, dtype=np.uint64) for w, _ in bitmaps]
    wp = (ctypes.c_void_p * max(len(words), 1))(*[w.ctypes.data for w in words])
    nb = np.asarray([int(nbits) for _, nbits in bitmaps] or [0], dtype=np.uint64)
    return words, wp, nb, len(bitmaps)


def count(columns: Sequence, types: Sequence[int], prog: bytes, bitmaps=None) -> int:
    """count(T, P): rows of T (numpy columns) satisfying program P; `bitmaps` are the key sets
    of IN_BITMAP leaves as [(uint64 words, nbits), ...] (id = position)."""
    arrs, ptrs, tys = _marshal(columns, types)
    n = len(arrs[0]) if arrs else 0
    st = ctypes.c_int(0)
    keep, wp, nb, k = _bitmaps(bitmaps)
    r = _load().oracle_count_bm(ptrs, tys.ctypes.data, len(arrs), n, prog, len(prog), wp,
                                nb.ctypes.data, k, ctypes.byref(st))
    if st.value != 0:
        raise OracleError(st.value)
    return int(r)


def count_mt(columns: Sequence, types: Sequence[int], prog: bytes, nthreads: int,
             bitmaps=None) -> int:
    """Same count, row-sharded over nthreads host threads (for timing on all cores)."""
    arrs, ptrs, tys = _marshal(columns, types)
    n = len(arrs[0]) if arrs else 0
    st = ctypes.c_int(0)
    keep, wp, nb, k = _bitmaps(bitmaps)
    r = _load().oracle_count_mt_bm(ptrs, tys.ctypes.data, len(arrs), n, prog, len(prog), nthreads,
                                   wp, nb.ctypes.data, k, ctypes.byref(st))
    if st.value != 0:
        raise OracleError(st.value)
    return int(r)


def pushdown(columns: Sequence, types: Sequence[int], prog: bytes, proj: Sequence[int] = (),
             capacity: int | None = None, row_offset: int = 0, bitmaps=None):
    """pushdown(T, P, proj) -> (count, ids[:min(count, capacity)], [projected columns])."""
    arrs, ptrs, tys = _marshal(columns, types)
    n = len(arrs[0]) if arrs else 0
    cap = n if capacity is None else int(capacity)
    ids = np.zeros(max(cap, 1), dtype=np.uint32)
    outs = [np.zeros(max(cap, 1), dtype=_NP[types[j]]) for j in proj]
    optrs = (ctypes.c_void_p * max(len(outs), 1))(*[o.ctypes.data for o in outs])
    pj = np.asarray(list(proj), dtype=np.uint32)
    st = ctypes.c_int(0)
    keep, wp, nb, k = _bitmaps(bitmaps)
    r = _load().oracle_pushdown_bm(ptrs, tys.ctypes.data, len(arrs), n, prog, len(prog),
                                   pj.ctypes.data if len(pj) else None, len(pj), row_offset,
                                   ids.ctypes.data, optrs, cap, wp, nb.ctypes.data, k,
                                   ctypes.byref(st))
    if st.value != 0:
        raise OracleError(st.value)
    k = min(int(r), cap)
    return int(r), ids[:k].copy(), [o[:k].copy() for o in outs]


def pushdown_mt(columns: Sequence, types: Sequence[int], prog: bytes, proj: Sequence[int] = (),
                capacity: int | None = None, row_offset: int = 0, bitmaps=None,
                nthreads: int | None = None):
    """The same result as pushdown(), computed over contiguous row shards on `nthreads` host
    threads and concatenated in shard order (oracle.c oracle_pushdown_mt_bm); for checking whole
    full-size tables. Pinned equal to pushdown() in tests/test_oracle_pins.py."""
    arrs, ptrs, tys = _marshal(columns, types)
    n = len(arrs[0]) if arrs else 0
    nthreads = int(nthreads or os.cpu_count() or 1)
    st = ctypes.c_int(0)
    keep, wp, nb, k = _bitmaps(bitmaps)
    cnt = count_mt(columns, types, prog, nthreads, bitmaps=bitmaps)
    cap = cnt if capacity is None else min(int(capacity), cnt)
    ids = np.empty(max(cap, 1), dtype=np.uint32)
    outs = [np.empty(max(cap, 1), dtype=_NP[types[j]]) for j in proj]
    optrs = (ctypes.c_void_p * max(len(outs), 1))(*[o.ctypes.data for o in outs])
    pj = np.asarray(list(proj), dtype=np.uint32)
    r = _load().oracle_pushdown_mt_bm(ptrs, tys.ctypes.data, len(arrs), n, prog, len(prog),
                                      pj.ctypes.data if len(pj) else None, len(pj), row_offset,
                                      ids.ctypes.data, optrs, cap, nthreads, wp, nb.ctypes.data,
                                      k, ctypes.byref(st))
    if st.value != 0:
        raise OracleError(st.value)
    assert int(r) == cnt
    return int(r), ids[:cap], [o[:cap] for o in outs]
