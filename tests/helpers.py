"""Test-side helpers: boundary-heavy random tables and two independent renderers of a predicate
AST — to SQLite SQL (library pin) and to NumPy masks (library pin). SURVEY §8c P1."""

from __future__ import annotations

import math
import sqlite3
import struct

import numpy as np

from selgen.program import (Cmp, Between, In, InSet, And, Or, Not, Const, F32Bits, INT32, INT64, FLOAT32,
                            DATE32, DICT8, DICT16, DICT32)

NP_DTYPE = {INT32: np.int32, INT64: np.int64, FLOAT32: np.float32, DATE32: np.int32,
            DICT8: np.uint8, DICT16: np.uint16, DICT32: np.uint32}

I32_MIN, I32_MAX = -(1 << 31), (1 << 31) - 1
I64_MIN, I64_MAX = -(1 << 63), (1 << 63) - 1
F32_TINY = struct.unpack("<f", struct.pack("<I", 1))[0]            # smallest subnormal
F32_MAX = struct.unpack("<f", struct.pack("<I", 0x7F7FFFFF))[0]


def boundary_pool(ctype, rng, with_nan=False):
    if ctype in (INT32, DATE32):
        base = [I32_MIN, I32_MIN + 1, -2, -1, 0, 1, 2, 7, I32_MAX - 1, I32_MAX]
        base += [int(x) for x in rng.integers(-1000, 1000, 6)]
    elif ctype == INT64:
        base = [I64_MIN, I64_MIN + 1, I32_MIN - 1, -1, 0, 1, I32_MAX + 1, I64_MAX - 1, I64_MAX]
        base += [int(x) for x in rng.integers(-10**12, 10**12, 6)]
    elif ctype == FLOAT32:
        base = [-math.inf, -F32_MAX, -1.5, -F32_TINY, -0.0, 0.0, F32_TINY, 1.0, 1.5, F32_MAX,
                math.inf]
        base += [float(np.float32(x)) for x in rng.normal(0, 10, 5)]
        if with_nan:
            base += [math.nan]
    elif ctype == DICT8:
        base = [0, 1, 2, 127, 128, 254, 255] + [int(x) for x in rng.integers(0, 256, 4)]
    elif ctype == DICT16:
        base = [0, 1, 255, 256, 32767, 32768, 65534, 65535] + [int(x) for x in rng.integers(0, 65536, 4)]
    else:
        base = [0, 1, (1 << 31) - 1, 1 << 31, (1 << 32) - 2, (1 << 32) - 1] + \
               [int(x) for x in rng.integers(0, 1 << 32, 4)]
    return base


def random_table(rng, types, n, with_nan=False):
    cols, pools = [], []
    for t in types:
        pool = boundary_pool(t, rng, with_nan)
        idx = rng.integers(0, len(pool), n)
        arr = np.array([pool[i] for i in idx], dtype=object)
        cols.append(np.array(arr.tolist(), dtype=NP_DTYPE[t]) if n else np.zeros(0, NP_DTYPE[t]))
        # constant pool: data values and their integer neighbours (c±1 boundaries)
        cp = list(pool)
        if t not in (FLOAT32,):
            lo, hi = {INT32: (I32_MIN, I32_MAX), DATE32: (I32_MIN, I32_MAX), INT64: (I64_MIN, I64_MAX),
                      DICT8: (0, 255), DICT16: (0, 65535), DICT32: (0, (1 << 32) - 1)}[t]
            cp += [min(hi, v + 1) for v in pool] + [max(lo, v - 1) for v in pool]
        pools.append(cp)
    return cols, pools


def _c(v, t):
    if t == FLOAT32:
        if isinstance(v, F32Bits):
            return struct.unpack("<f", struct.pack("<I", v.bits))[0]
        return struct.unpack("<f", struct.pack("<f", float(v)))[0]
    return int(v)


# ---- NumPy renderer -------------------------------------------------------------------------

def bitmap_keys(words, nbits):
    """The key set of a bitmap given as uint64 words."""
    bits = np.unpackbits(np.asarray(words, dtype=np.uint64).view(np.uint8), bitorder="little")
    return np.flatnonzero(bits[:nbits])


def make_bitmap(keys, nbits):
    """(uint64 words, nbits) with exactly `keys` (all < nbits) set."""
    bits = np.zeros(((nbits + 63) // 64) * 64, dtype=np.uint8)
    keys = np.asarray(list(keys), dtype=np.int64)
    bits[keys] = 1
    return np.packbits(bits, bitorder="little").view(np.uint64).copy(), int(nbits)


def random_bitmaps(rng, pools):
    """Key sets for InSet leaves that hit the data: boundaries 0, nbits-1, nbits; non-negative
    pool values; an empty set; DICT8/DICT16 code-space edges."""
    nonneg = sorted({int(v) for p in pools for v in p if isinstance(v, (int, np.integer)) and v >= 0})
    out = [make_bitmap([0], 1), make_bitmap([], 64)]
    keys = [k for k in range(256) if rng.random() < 0.5] + [255]
    out.append(make_bitmap(keys, 256))
    keys = [v for v in nonneg if v < 1001 and rng.random() < 0.6] + [1000]
    keys += [int(k) for k in rng.integers(0, 1001, 50)]
    out.append(make_bitmap(keys, 1001))
    keys = [v for v in nonneg if v < 65543 and rng.random() < 0.6] + [65535, 65536, 65542]
    keys += [int(k) for k in rng.integers(0, 65543, 300)]
    out.append(make_bitmap(keys, 65543))
    return out


def np_mask(node, cols, types, n, bitmaps=None):
    if isinstance(node, Const):
        return np.full(n, bool(node.value))
    if isinstance(node, InSet):
        keys = bitmap_keys(*bitmaps[node.bitmap])
        return np.isin(cols[node.col].astype(np.int64), keys.astype(np.int64))
    if isinstance(node, Cmp):
        a = cols[node.col]
        c = NP_DTYPE[types[node.col]](_c(node.value, types[node.col]))
        return {"=": a == c, "<": a < c, ">": a > c, "<=": a <= c, ">=": a >= c}[node.op]
    if isinstance(node, Between):
        a = cols[node.col]
        t = types[node.col]
        return (NP_DTYPE[t](_c(node.lo, t)) <= a) & (a <= NP_DTYPE[t](_c(node.hi, t)))
    if isinstance(node, In):
        a = cols[node.col]
        t = types[node.col]
        m = np.zeros(n, dtype=bool)
        for v in node.values:
            m |= a == NP_DTYPE[t](_c(v, t))
        return m
    if isinstance(node, And):
        return np_mask(node.l, cols, types, n, bitmaps) & np_mask(node.r, cols, types, n, bitmaps)
    if isinstance(node, Or):
        return np_mask(node.l, cols, types, n, bitmaps) | np_mask(node.r, cols, types, n, bitmaps)
    if isinstance(node, Not):
        return ~np_mask(node.x, cols, types, n, bitmaps)
    raise TypeError(node)


# ---- SQLite renderer ------------------------------------------------------------------------

def sql_where(node, types, params, bitmaps=None):
    if isinstance(node, Const):
        return "1" if node.value else "0"
    if isinstance(node, InSet):
        keys = [int(k) for k in bitmap_keys(*bitmaps[node.bitmap])]
        if not keys:
            return "0"
        params += keys
        return f"(c{node.col} IN ({', '.join('?' * len(keys))}))"
    if isinstance(node, Cmp):
        params.append(_c(node.value, types[node.col]))
        return f"(c{node.col} {node.op} ?)"
    if isinstance(node, Between):
        params += [_c(node.lo, types[node.col]), _c(node.hi, types[node.col])]
        return f"(c{node.col} BETWEEN ? AND ?)"
    if isinstance(node, In):
        params += [_c(v, types[node.col]) for v in node.values]
        return f"(c{node.col} IN ({', '.join('?' * len(node.values))}))"
    if isinstance(node, And):
        return f"({sql_where(node.l, types, params, bitmaps)} AND {sql_where(node.r, types, params, bitmaps)})"
    if isinstance(node, Or):
        return f"({sql_where(node.l, types, params, bitmaps)} OR {sql_where(node.r, types, params, bitmaps)})"
    if isinstance(node, Not):
        return f"(NOT {sql_where(node.x, types, params, bitmaps)})"
    raise TypeError(node)


class SqliteTable:
    def __init__(self, cols, types):
        self.db = sqlite3.connect(":memory:")
        decl = ", ".join(f"c{i} {'REAL' if t == FLOAT32 else 'INTEGER'}" for i, t in enumerate(types))
        self.db.execute(f"CREATE TABLE t ({decl})")
        rows = zip(*[[float(x) if t == FLOAT32 else int(x) for x in c] for c, t in zip(cols, types)])
        self.db.executemany(f"INSERT INTO t VALUES ({', '.join('?' * len(types))})", rows)
        self.types = types

    def ids(self, node, bitmaps=None):
        params = []
        w = sql_where(node, self.types, params, bitmaps)
        return [r[0] for r in self.db.execute(f"SELECT rowid - 1 FROM t WHERE {w} ORDER BY rowid", params)]
