"""TEST INFRASTRUCTURE ONLY — a second, independently written oracle for tiny inputs.

A recursive evaluator over selgen's predicate AST (no postfix, no stack, no bytes): used to
pin oracle.c's decoder and stack mechanics by brute force and to compute
closed-form counts over distinct tuples (P3). Semantics are SQL's two-valued comparisons in
the column's type (include/sel.h "Opcodes"); FLOAT32 constants are first
rounded to binary32 exactly as the program stores them, and all comparisons of float32
values widened to Python floats are exact.
"""

from __future__ import annotations

import struct

from selgen.program import (Cmp, Between, In, And, Or, Not, Const, F32Bits, FLOAT32)


def _const(v, ctype):
    if ctype == FLOAT32:
        if isinstance(v, F32Bits):
            return struct.unpack("<f", struct.pack("<I", v.bits & 0xFFFFFFFF))[0]
        return struct.unpack("<f", struct.pack("<f", float(v)))[0]
    return int(v)


def eval_row(node, row, types) -> bool:
    """P(row) for one row given as a sequence of Python values (floats for FLOAT32)."""
    if isinstance(node, Const):
        return bool(node.value)
    if isinstance(node, Cmp):
        v, c = row[node.col], _const(node.value, types[node.col])
        return {"=": v == c, "<": v < c, ">": v > c, "<=": v <= c, ">=": v >= c}[node.op]
    if isinstance(node, Between):
        v = row[node.col]
        return _const(node.lo, types[node.col]) <= v and v <= _const(node.hi, types[node.col])
    if isinstance(node, In):
        v = row[node.col]
        return any(v == _const(x, types[node.col]) for x in node.values)
    if isinstance(node, And):
        return eval_row(node.l, row, types) and eval_row(node.r, row, types)
    if isinstance(node, Or):
        return eval_row(node.l, row, types) or eval_row(node.r, row, types)
    if isinstance(node, Not):
        return not eval_row(node.x, row, types)
    raise TypeError(node)


def count_rows(node, rows, types) -> int:
    return sum(1 for r in rows if eval_row(node, r, types))


def ids_rows(node, rows, types) -> list:
    return [i for i, r in enumerate(rows) if eval_row(node, r, types)]
