"""Predicate builder → program bytes (include/sel.h, version 1).

    from paper_1806_08384_b200 import col
    p = (col("A") == 2) & (col("B") < 2001) & (col("B") > 1000) & col("C").isin(["MAIL", "SHIP"])

is Listing 3.1 of the paper. Strings are mapped to dictionary codes on the
host through the column's sorted dictionary (code order = string order); an unknown string in
an equality/IN becomes a FALSE leaf, and string range bounds become the matching code bounds.
Dates (datetime.date) become DATE32 days since 1970-01-01.

FLOAT32 columns compare against the EXACT value of a Python constant (SQL: the binary32 value
widened, compared with the literal). A constant float32 cannot represent exactly is never equal to
any row, and a range bound is moved to the float32 neighbour on the side the operator needs:
x < 0.7 becomes x <= (largest float32 below 0.7), x >= 0.7 becomes x >= (smallest float32 above
it); = becomes FALSE, an IN drops such values, BETWEEN moves each bound inward. The program always
carries float32 bits (include/sel.h), so this is decided here, on the host.
"""

from __future__ import annotations

import bisect
import datetime
import math
import struct
from dataclasses import dataclass

import numpy as np

INT32, INT64, FLOAT32, DATE32, DICT8, DICT16, DICT32 = 1, 2, 3, 4, 5, 6, 7
_OPS = {"=": 0x10, "<": 0x11, ">": 0x12, "<=": 0x13, ">=": 0x14}
_EPOCH = datetime.date(1970, 1, 1)


class Expr:
    def __and__(self, other):
        return _And(self, _wrap(other))

    def __rand__(self, other):
        return _And(_wrap(other), self)

    def __or__(self, other):
        return _Or(self, _wrap(other))

    def __ror__(self, other):
        return _Or(_wrap(other), self)

    def __invert__(self):
        return _Not(self)


def _wrap(x):
    if isinstance(x, Expr):
        return x
    if isinstance(x, bool):
        return _Const(x)
    raise TypeError(f"not a predicate: {x!r}")


@dataclass(eq=False)
class _Const(Expr):
    value: bool


@dataclass(eq=False)
class _Cmp(Expr):
    op: str
    name: str
    value: object


@dataclass(eq=False)
class _Between(Expr):
    name: str
    lo: object
    hi: object


@dataclass(eq=False)
class _In(Expr):
    name: str
    values: tuple


@dataclass(eq=False)
class _InSet(Expr):
    name: str
    bitmap: int


@dataclass(eq=False)
class _And(Expr):
    l: Expr
    r: Expr


@dataclass(eq=False)
class _Or(Expr):
    l: Expr
    r: Expr


@dataclass(eq=False)
class _Not(Expr):
    x: Expr


TRUE = _Const(True)
FALSE = _Const(False)


class Col:
    """A column reference; comparison operators build predicate leaves."""

    __hash__ = object.__hash__

    def __init__(self, name: str):
        self.name = name

    def __eq__(self, v):
        return _Cmp("=", self.name, v)

    def __ne__(self, v):
        return _Not(_Cmp("=", self.name, v))

    def __lt__(self, v):
        return _Cmp("<", self.name, v)

    def __le__(self, v):
        return _Cmp("<=", self.name, v)

    def __gt__(self, v):
        return _Cmp(">", self.name, v)

    def __ge__(self, v):
        return _Cmp(">=", self.name, v)

    def between(self, lo, hi):
        return _Between(self.name, lo, hi)

    def isin(self, values):
        return _In(self.name, tuple(values))

    def in_set(self, bitmap_id: int):
        """Membership in a key set registered with Context.register_bitmap (IN_BITMAP, 0x31):
        e.g. lo_partkey IN {p_partkey : p_category = 12} as a semijoin filter."""
        return _InSet(self.name, int(bitmap_id))


def col(name: str) -> Col:
    return Col(name)


# ---- encoding --------------------------------------------------------------------------------

def _f32_neighbours(v):
    """(lo, hi) float32 values with lo <= v <= hi and nothing in float32 strictly between;
    lo == hi iff v is exactly a float32 (or +-inf). NaN gives (nan, nan)."""
    if isinstance(v, float) and math.isnan(v):
        return float("nan"), float("nan")
    with np.errstate(over="ignore"):
        f = np.float32(float(v))           # nearest (double rounding for huge ints: fixed below)
        while float(f) > v:                # Python compares int/float values exactly
            f = np.nextafter(f, np.float32(-np.inf))
        while float(f) < v and float(np.nextafter(f, np.float32(np.inf))) <= v:
            f = np.nextafter(f, np.float32(np.inf))
        if float(f) == v:
            return float(f), float(f)
        return float(f), float(np.nextafter(f, np.float32(np.inf)))   # f < v < next


def _exact_f32_cmp(op, v):
    """(op', c) with `x op v` == `x op' c` for every float32 x (c a float32), or None when the
    leaf is constant FALSE (an inexact equality)."""
    lo, hi = _f32_neighbours(v)
    if lo == hi or math.isnan(lo):
        return op, lo
    if op == "=":
        return None
    if op in ("<", "<="):
        return "<=", lo
    return ">=", hi


# ---- encoding --------------------------------------------------------------------------------

class _Writer:
    def __init__(self, schema):
        self.schema = schema            # list of (name, type, dictionary or None)
        self.index = {s[0]: i for i, s in enumerate(schema)}
        self.instrs = []
        self.consts = []

    def const_slot(self, v, t):
        if t == FLOAT32:
            k = struct.unpack("<I", struct.pack("<f", float(v)))[0]
        elif t in (INT32, DATE32):
            v = int(v)
            if not -(1 << 31) <= v < (1 << 31):
                raise ValueError(f"constant {v} does not fit a 32-bit column")
            k = v & 0xFFFFFFFFFFFFFFFF
        elif t == INT64:
            k = int(v) & 0xFFFFFFFFFFFFFFFF
        else:
            k = int(v)
            lim = {DICT8: 1 << 8, DICT16: 1 << 16, DICT32: 1 << 32}[t]
            if not 0 <= k < lim:
                raise ValueError(f"dictionary code {k} out of range")
        self.consts.append(k)
        return len(self.consts) - 1

    def leaf_false(self):
        self.instrs.append((0x02, 0, 0, 0))

    def value(self, name, v, how="eq"):
        """Map a Python value to the column's domain. Returns an int/float, or None when a string
        is not in the dictionary (for how='eq'); for range bounds returns the code bound."""
        c, t, d = self.index[name], self.schema[self.index[name]][1], self.schema[self.index[name]][2]
        if isinstance(v, datetime.date):
            return (v - _EPOCH).days
        if isinstance(v, str):
            if d is None:
                raise TypeError(f"column {name} has no dictionary for string {v!r}")
            if how == "eq":
                i = bisect.bisect_left(d, v)
                return i if i < len(d) and d[i] == v else None
            if how == "lo":       # smallest code whose string >= v
                return bisect.bisect_left(d, v)
            return bisect.bisect_right(d, v) - 1   # "hi": largest code whose string <= v
        return v

    def emit(self, e):
        if isinstance(e, _Const):
            self.instrs.append((0x01 if e.value else 0x02, 0, 0, 0))
        elif isinstance(e, _Cmp):
            c = self.index[e.name]
            t = self.schema[c][1]
            if isinstance(e.value, str):
                self._string_cmp(e, c, t)
                return
            v, op = self.value(e.name, e.value), e.op
            if t == FLOAT32:
                r = _exact_f32_cmp(op, v)
                if r is None:
                    self.leaf_false()
                    return
                op, v = r
            k = self.const_slot(v, t)
            self.instrs.append((_OPS[op], c, k, 0))
        elif isinstance(e, _InSet):
            self.instrs.append((0x31, self.index[e.name], e.bitmap, 0))
        elif isinstance(e, _Between):
            c = self.index[e.name]
            t = self.schema[c][1]
            lo = self.value(e.name, e.lo, "lo")
            hi = self.value(e.name, e.hi, "hi")
            if isinstance(e.lo, str) or isinstance(e.hi, str):
                if hi < 0 or lo > (1 << (8 * {DICT8: 1, DICT16: 2}.get(t, 4))) - 1:
                    self.leaf_false()
                    return
            if t == FLOAT32:       # each bound inward to a float32 (exact range semantics)
                lo = _f32_neighbours(lo)[1]
                hi = _f32_neighbours(hi)[0]
            a = self.const_slot(lo, t)
            b = self.const_slot(hi, t)
            self.instrs.append((0x20, c, a, b))
        elif isinstance(e, _In):
            c = self.index[e.name]
            t = self.schema[c][1]
            vals = [self.value(e.name, v) for v in e.values]
            vals = [v for v in vals if v is not None]
            if t == FLOAT32:       # a value no float32 equals never matches
                vals = [r[1] for r in (_exact_f32_cmp("=", v) for v in vals) if r is not None]
            if not vals:
                self.leaf_false()
                return
            first = len(self.consts)
            for v in vals:
                self.const_slot(v, t)
            self.instrs.append((0x30, c, first, len(vals)))
        elif isinstance(e, (_And, _Or)):
            self.emit(e.l)
            self.emit(e.r)
            self.instrs.append((0x40 if isinstance(e, _And) else 0x41, 0, 0, 0))
        elif isinstance(e, _Not):
            self.emit(e.x)
            self.instrs.append((0x42, 0, 0, 0))
        else:
            raise TypeError(f"not a predicate: {e!r}")

    def _string_cmp(self, e, c, t):
        if e.op == "=":
            v = self.value(e.name, e.value, "eq")
            if v is None:
                self.leaf_false()
            else:
                self.instrs.append((0x10, c, self.const_slot(v, t), 0))
            return
        # string order == code order: x < s  <=>  code < first code >= s
        if e.op in ("<", ">="):
            bound = self.value(e.name, e.value, "lo")
            if bound > (1 << (8 * {DICT8: 1, DICT16: 2}.get(t, 4))) - 1:
                # s sorts after every string of a full dictionary: every code is < the bound
                self.instrs.append((0x01 if e.op == "<" else 0x02, 0, 0, 0))
                return
            self.instrs.append((_OPS[e.op], c, self.const_slot(bound, t), 0))
        else:  # "<=", ">": compare against the last code <= s
            bound = self.value(e.name, e.value, "hi")
            if bound < 0:   # every string is > s
                self.instrs.append((0x01 if e.op == ">" else 0x02, 0, 0, 0))
            else:
                self.instrs.append((_OPS[e.op], c, self.const_slot(bound, t), 0))

    def bytes(self) -> bytes:
        out = bytearray(b"SELP")
        out += struct.pack("<HHHH", 1, len(self.instrs), len(self.consts), 0)
        for op, c, a, b in self.instrs:
            out += struct.pack("<BBHHH", op, c, a, b, 0)
        for k in self.consts:
            out += struct.pack("<Q", k)
        return bytes(out)


def compile_predicate(expr: Expr, schema) -> bytes:
    """schema: list of (name, sel_type, sorted dictionary list or None)."""
    w = _Writer(schema)
    w.emit(_wrap(expr))
    return w.bytes()
