"""Predicate programs as inputs: a tiny AST and the byte writer for the format of
`include/sel.h` (version 1). This module only *writes* program bytes; it never evaluates them.

Grammar (BASELINE.json north_star): AND/OR/NOT over `=`, `<`, `>`, `<=`, `>=`,
BETWEEN and IN-list comparisons of one column against constants, plus TRUE/FALSE.
The paper's own predicate (Listing 1.1; Listing 3.1) is
`A = x AND B < y1 AND B > y2 AND (C = z1 OR C = z2)`.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass
from typing import Sequence, Union

# Column type codes (the values `include/sel.h` fixes for `sel_type`).
INT32, INT64, FLOAT32, DATE32, DICT8, DICT16, DICT32 = 1, 2, 3, 4, 5, 6, 7
TYPE_WIDTH = {INT32: 4, INT64: 8, FLOAT32: 4, DATE32: 4, DICT8: 1, DICT16: 2, DICT32: 4}
TYPE_NAMES = {INT32: "INT32", INT64: "INT64", FLOAT32: "FLOAT32", DATE32: "DATE32",
              DICT8: "DICT8", DICT16: "DICT16", DICT32: "DICT32"}

# Opcodes (include/sel.h).
OP_TRUE, OP_FALSE = 0x01, 0x02
OP_EQ, OP_LT, OP_GT, OP_LE, OP_GE = 0x10, 0x11, 0x12, 0x13, 0x14
OP_BETWEEN, OP_IN, OP_IN_BITMAP = 0x20, 0x30, 0x31
OP_AND, OP_OR, OP_NOT = 0x40, 0x41, 0x42
CMP_OPS = {"=": OP_EQ, "<": OP_LT, ">": OP_GT, "<=": OP_LE, ">=": OP_GE}

MAGIC = b"SELP"
VERSION = 1


@dataclass(frozen=True)
class F32Bits:
    """A FLOAT32 constant given by its exact binary32 bit pattern (NaN payloads, -0.0, ...)."""
    bits: int


Value = Union[int, float, F32Bits]


@dataclass(frozen=True)
class Cmp:
    op: str          # one of = < > <= >=
    col: int
    value: Value


@dataclass(frozen=True)
class Between:
    col: int
    lo: Value
    hi: Value


@dataclass(frozen=True)
class In:
    col: int
    values: tuple


@dataclass(frozen=True)
class InSet:
    """Membership in a registered key set (IN_BITMAP); `bitmap` is its id."""
    col: int
    bitmap: int


@dataclass(frozen=True)
class And:
    l: object
    r: object


@dataclass(frozen=True)
class Or:
    l: object
    r: object


@dataclass(frozen=True)
class Not:
    x: object


@dataclass(frozen=True)
class Const:
    value: bool


def f32_bits(v: Value) -> int:
    if isinstance(v, F32Bits):
        return v.bits & 0xFFFFFFFF
    return struct.unpack("<I", struct.pack("<f", float(v)))[0]


def encode_const(v: Value, ctype: int) -> int:
    """u64 slot for constant v against a column of type ctype (include/sel.h, constants)."""
    if ctype == FLOAT32:
        return f32_bits(v)
    if isinstance(v, (F32Bits, float)):
        raise TypeError("integer column needs an integer constant")
    v = int(v)
    if ctype in (INT32, DATE32, INT64):
        return v & ((1 << 64) - 1)          # two's-complement sign extension to 64 bits
    if v < 0:
        raise ValueError("dictionary codes are unsigned")
    return v


def _walk(node, types, instrs, consts):
    if isinstance(node, Const):
        instrs.append((OP_TRUE if node.value else OP_FALSE, 0, 0, 0))
    elif isinstance(node, Cmp):
        consts.append(encode_const(node.value, types[node.col]))
        instrs.append((CMP_OPS[node.op], node.col, len(consts) - 1, 0))
    elif isinstance(node, Between):
        consts.append(encode_const(node.lo, types[node.col]))
        consts.append(encode_const(node.hi, types[node.col]))
        instrs.append((OP_BETWEEN, node.col, len(consts) - 2, len(consts) - 1))
    elif isinstance(node, In):
        first = len(consts)
        for v in node.values:
            consts.append(encode_const(v, types[node.col]))
        instrs.append((OP_IN, node.col, first, len(node.values)))
    elif isinstance(node, InSet):
        instrs.append((OP_IN_BITMAP, node.col, node.bitmap, 0))
    elif isinstance(node, (And, Or)):
        _walk(node.l, types, instrs, consts)
        _walk(node.r, types, instrs, consts)
        instrs.append((OP_AND if isinstance(node, And) else OP_OR, 0, 0, 0))
    elif isinstance(node, Not):
        _walk(node.x, types, instrs, consts)
        instrs.append((OP_NOT, 0, 0, 0))
    else:
        raise TypeError(f"not a predicate node: {node!r}")


def encode_raw(instrs: Sequence[tuple], consts: Sequence[int], *, magic: bytes = MAGIC,
               version: int = VERSION, n_instr: int | None = None, n_consts: int | None = None,
               reserved: int = 0) -> bytes:
    """Pack (op, col, a, b[, reserved]) tuples and u64 constants; overrides allow malformed
    headers for validator fuzzing."""
    n_i = len(instrs) if n_instr is None else n_instr
    n_c = len(consts) if n_consts is None else n_consts
    out = bytearray(magic)
    out += struct.pack("<HHHH", version & 0xFFFF, n_i & 0xFFFF, n_c & 0xFFFF, reserved & 0xFFFF)
    for ins in instrs:
        op, col, a, b = ins[:4]
        res = ins[4] if len(ins) > 4 else 0
        out += struct.pack("<BBHHH", op & 0xFF, col & 0xFF, a & 0xFFFF, b & 0xFFFF, res & 0xFFFF)
    for c in consts:
        out += struct.pack("<Q", c & ((1 << 64) - 1))
    return bytes(out)


def encode(node, types: Sequence[int]) -> bytes:
    """Postfix (post-order) encoding of an AST against column types `types`."""
    instrs: list = []
    consts: list = []
    _walk(node, types, instrs, consts)
    return encode_raw(instrs, consts)


# ----------------------------------------------------------------------------------------
# Random programs for property tests (seeded numpy Generator; boundary-heavy constants).

def _pick_value(rng, ctype, pool):
    if pool is not None and len(pool) and rng.random() < 0.8:
        v = pool[int(rng.integers(len(pool)))]
    else:
        if ctype in (INT32, DATE32):
            v = int(rng.choice([-(1 << 31), (1 << 31) - 1, 0, -1, 1, int(rng.integers(-1000, 1000))]))
        elif ctype == INT64:
            v = int(rng.choice([-(1 << 63), (1 << 63) - 1, 0, -1, 1, int(rng.integers(-10**12, 10**12))]))
        elif ctype == FLOAT32:
            v = float(rng.choice([0.0, -0.0, math.inf, -math.inf, 1.5, -2.25, 1e-45, -1e-45]))
        elif ctype == DICT8:
            v = int(rng.integers(0, 256))
        elif ctype == DICT16:
            v = int(rng.integers(0, 65536))
        else:
            v = int(rng.integers(0, 1 << 32))
    if ctype == FLOAT32:
        if isinstance(v, F32Bits):
            return v
        return float(v)
    return int(v)


def random_program(rng, types: Sequence[int], pools: Sequence | None = None, max_depth: int = 3,
                   in_max: int = 6, n_bitmaps: int = 0):
    """A random AST of depth ≤ max_depth over columns with `types`. pools[c] (optional) lists
    values that occur in column c, so that constants hit data boundaries often. With n_bitmaps,
    some leaves on integer columns are InSet(col, id < n_bitmaps)."""
    ncols = len(types)

    def leaf():
        c = int(rng.integers(ncols))
        pool = pools[c] if pools is not None else None
        if n_bitmaps and types[c] != FLOAT32 and rng.random() < 0.2:
            return InSet(c, int(rng.integers(n_bitmaps)))
        r = rng.random()
        if r < 0.04:
            return Const(bool(rng.integers(2)))
        if r < 0.60:
            op = ["=", "<", ">", "<=", ">="][int(rng.integers(5))]
            return Cmp(op, c, _pick_value(rng, types[c], pool))
        if r < 0.80:
            return Between(c, _pick_value(rng, types[c], pool), _pick_value(rng, types[c], pool))
        k = int(rng.integers(1, in_max + 1))
        return In(c, tuple(_pick_value(rng, types[c], pool) for _ in range(k)))

    def node(d):
        if d <= 1 or rng.random() < 0.3:
            return leaf()
        r = rng.random()
        if r < 0.4:
            return And(node(d - 1), node(d - 1))
        if r < 0.8:
            return Or(node(d - 1), node(d - 1))
        return Not(node(d - 1))

    return node(max_depth)
