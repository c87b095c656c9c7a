"""Pins of the CPU oracle to things other than itself (task rule ③).

P1  leaf/combinator semantics vs SQLite 3 (stdlib) and NumPy masks, boundary-heavy tables
P2  brute force vs a recursive AST evaluator (oracle/ast_eval.py) on exhaustive tiny domains
P3  closed-form counts and row ids of a tuple multiset (the worked-example generator C2)
P4  closed-form counts and row ids of an affine-threshold column (C5)
P5  the worked example's printed numbers (tests/golden/worked_example.json)
P6  invariants (complement, inclusion-exclusion, De Morgan, BETWEEN/IN decompositions, gate)
P7  the paper's fixed points on orders-shaped data
plus the validator against every clause of include/sel.h "Program validation".
"""

from __future__ import annotations

import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import ast_eval
from selgen import configs
from selgen.program import (Cmp, Between, In, InSet, And, Or, Not, Const, F32Bits, encode, encode_raw,
                            random_program, INT32, INT64, FLOAT32, DATE32, DICT8, DICT16, DICT32)

from helpers import random_table, np_mask, SqliteTable, random_bitmaps, make_bitmap

HERE = os.path.dirname(os.path.abspath(__file__))
ALL_TYPES = [INT32, INT64, FLOAT32, DATE32, DICT8, DICT16, DICT32]


def _ids(cols, types, node):
    c, ids, _ = oracle.pushdown(cols, types, encode(node, types))
    assert c == len(ids)
    return ids


# ---- P1: SQLite and NumPy ------------------------------------------------------------------

@pytest.mark.parametrize("types", [
    [INT32, DICT8, FLOAT32],
    [INT64, DATE32, DICT16],
    [DICT32, INT32, INT64, FLOAT32],
])
def test_p1_sqlite_numpy(types):
    rng = np.random.default_rng(sum(types) * 7919)
    n = 3000
    cols, pools = random_table(rng, types, n)
    sq = SqliteTable(cols, types)
    for trial in range(60):
        node = random_program(rng, types, pools, max_depth=3)
        prog = encode(node, types)
        got_count = oracle.count(cols, types, prog)
        ids = _ids(cols, types, node)
        want_np = np.flatnonzero(np_mask(node, cols, types, n))
        want_sql = np.asarray(sq.ids(node), dtype=np.int64)
        assert got_count == len(want_np) == len(want_sql), node
        np.testing.assert_array_equal(ids, want_np)
        np.testing.assert_array_equal(ids, want_sql)


@pytest.mark.parametrize("types", [
    [INT32, DICT8, INT64],
    [DICT16, DATE32, DICT32, FLOAT32],
])
def test_p1_inset_sqlite_numpy(types):
    """IN_BITMAP leaves: membership of the value in a registered key set is
    SQL `col IN (keys...)` and np.isin, under AND/OR/NOT with every other leaf kind."""
    rng = np.random.default_rng(sum(types) * 131)
    n = 3000
    cols, pools = random_table(rng, types, n)
    for c, t in enumerate(types):   # small non-negative values, so that the key sets hit rows
        if t != FLOAT32:
            small = rng.integers(0, 256 if t == DICT8 else 1100, n)
            cols[c] = np.where(rng.random(n) < 0.5, small.astype(cols[c].dtype), cols[c])
            pools[c] = list(pools[c]) + [int(v) for v in small[:20]]
    bms = random_bitmaps(rng, pools)
    sq = SqliteTable(cols, types)
    seen_nonempty = 0
    for trial in range(60):
        node = random_program(rng, types, pools, max_depth=3, n_bitmaps=len(bms))
        prog = encode(node, types)
        got = oracle.count(cols, types, prog, bitmaps=bms)
        c, ids, _ = oracle.pushdown(cols, types, prog, bitmaps=bms)
        want_np = np.flatnonzero(np_mask(node, cols, types, n, bms))
        want_sql = np.asarray(sq.ids(node, bms), dtype=np.int64)
        assert got == c == len(want_np) == len(want_sql), node
        np.testing.assert_array_equal(ids, want_np)
        np.testing.assert_array_equal(ids, want_sql)
        seen_nonempty += 0 < got < n
    assert seen_nonempty > 10


def test_p1_inset_edges():
    """v < nbits boundary, negative values never members (also under NOT), the empty set, and an
    id that is not among the supplied sets (SEL_E_ARG)."""
    x = np.array([-2**31, -1, 0, 1, 62, 63, 64, 65, 99, 100, 2**31 - 1], dtype=np.int32)
    bm = [make_bitmap([0, 63, 64, 99], 100), make_bitmap([], 1)]
    prog = encode(InSet(0, 0), [INT32])
    assert oracle.pushdown([x], [INT32], prog, bitmaps=bm)[1].tolist() == [2, 5, 6, 8]
    notp = encode(Not(InSet(0, 0)), [INT32])
    assert oracle.pushdown([x], [INT32], notp, bitmaps=bm)[1].tolist() == [0, 1, 3, 4, 7, 9, 10]
    assert oracle.count([x], [INT32], encode(InSet(0, 1), [INT32]), bitmaps=bm) == 0
    y = np.array([-1, 0, 99, 100, 2**40], dtype=np.int64)
    assert oracle.pushdown([y], [INT64], prog, bitmaps=bm)[1].tolist() == [1, 2]
    with pytest.raises(oracle.OracleError) as e:
        oracle.count([x], [INT32], encode(InSet(0, 2), [INT32]), bitmaps=bm)
    assert e.value.status == 1
    with pytest.raises(oracle.OracleError):
        oracle.count([x], [INT32], prog)


def test_p1_float_nan_and_signed_zero_numpy():
    """NaN compares false, NOT(x < c) is true for NaN, -0 == +0 (IEEE; SQLite has no NaN)."""
    rng = np.random.default_rng(11)
    types = [FLOAT32]
    cols, pools = random_table(rng, types, 2000, with_nan=True)
    assert np.isnan(cols[0]).any()
    for trial in range(150):
        node = random_program(rng, types, pools, max_depth=3)
        ids = _ids(cols, types, node)
        np.testing.assert_array_equal(ids, np.flatnonzero(np_mask(node, cols, types, 2000)))
    x = np.array([-0.0, 0.0, np.nan, 1.0, -np.inf, np.inf], dtype=np.float32)
    for node, want in [(Cmp("=", 0, 0.0), [0, 1]), (Cmp("=", 0, -0.0), [0, 1]),
                       (Not(Cmp("<", 0, 1.0)), [2, 3, 5]), (Cmp("<", 0, F32Bits(0x7FC00000)), []),
                       (Not(Cmp("=", 0, F32Bits(0x7FC00000))), [0, 1, 2, 3, 4, 5]),
                       (Cmp("<=", 0, -math.inf), [4]), (Cmp(">", 0, -0.0), [3, 5]),
                       (Between(0, -0.0, 0.0), [0, 1]), (In(0, (math.inf, -math.inf)), [4, 5])]:
        np.testing.assert_array_equal(_ids([x], [FLOAT32], node), want)


def test_p1_subnormals_not_flushed():
    tiny = np.array([1e-45, -1e-45, 0.0, 1.2e-38], dtype=np.float32)
    assert oracle.count([tiny], [FLOAT32], encode(Cmp(">", 0, 0.0), [FLOAT32])) == 2
    assert oracle.count([tiny], [FLOAT32], encode(Cmp("=", 0, 1e-45), [FLOAT32])) == 1
    assert oracle.count([tiny], [FLOAT32], encode(Cmp("<", 0, 0.0), [FLOAT32])) == 1


# ---- P2: brute force vs the recursive AST evaluator ------------------------------------------

def _all_leaves(ncols, consts):
    out = []
    for c in range(ncols):
        for op in ["=", "<", ">", "<=", ">="]:
            out += [Cmp(op, c, k) for k in consts]
        out += [Between(c, lo, hi) for lo in consts for hi in consts]
        for r in (1, 2, 3):
            out += [In(c, s) for s in itertools.combinations(consts, r)]
    return out + [Const(True), Const(False)]


def _check_rows(node, rows, types):
    cols = [np.array([r[c] for r in rows], dtype={INT32: np.int32, DICT8: np.uint8,
                                                   FLOAT32: np.float32}[t])
            for c, t in enumerate(types)]
    prog = encode(node, types)
    rows = list(zip(*[[x.item() for x in c] for c in cols]))     # values as stored (binary32)
    want = ast_eval.ids_rows(node, rows, types)
    assert oracle.count(cols, types, prog) == len(want), node
    got = oracle.pushdown(cols, types, prog)[1]
    np.testing.assert_array_equal(got, want)


def test_p2_bruteforce_int_domain():
    """Every row of {-1,0,1,2}^2, every leaf with constants {-2..3}, NOT of each leaf, AND/OR of
    leaf pairs, and random depth-3 trees."""
    types = [INT32, INT32]
    dom = [-1, 0, 1, 2]
    rows = [(a, b) for a in dom for b in dom]
    leaves = _all_leaves(2, [-2, -1, 0, 1, 2, 3])
    for lf in leaves:
        _check_rows(lf, rows, types)
        _check_rows(Not(lf), rows, types)
    rng = np.random.default_rng(2)
    pick = [leaves[i] for i in rng.choice(len(leaves), 40, replace=False)]
    for x in pick:
        for y in pick:
            _check_rows(And(x, y), rows, types)
            _check_rows(Or(x, y), rows, types)
    pools = [[-2, -1, 0, 1, 2, 3]] * 2
    for _ in range(1500):
        _check_rows(random_program(rng, types, pools, max_depth=4), rows, types)


def test_p2_bruteforce_float_dict_domain():
    types = [FLOAT32, DICT8]
    fdom = [-math.inf, -1.5, -0.0, 0.0, 1e-45, 2.0, math.inf, math.nan]
    ddom = [0, 1, 2, 255]
    rows = [(f, d) for f in fdom for d in ddom]
    rng = np.random.default_rng(3)
    pools = [fdom, ddom]
    for _ in range(2500):
        _check_rows(random_program(rng, types, pools, max_depth=4), rows, types)


def test_p2_tiny_tables_all_lengths():
    """Every table of N <= 2 rows over {-1..2}^2 and sampled N = 3 tables, N = 0 included."""
    types = [INT32, INT32]
    dom = [-1, 0, 1, 2]
    all_rows = [(a, b) for a in dom for b in dom]
    rng = np.random.default_rng(4)
    progs = [random_program(rng, types, [[-2, -1, 0, 1, 2, 3]] * 2, max_depth=3) for _ in range(12)]
    tables = [[]] + [[r] for r in all_rows] + [list(p) for p in itertools.product(all_rows, repeat=2)]
    tables += [[all_rows[i] for i in rng.integers(0, 16, 3)] for _ in range(100)]
    for rows in tables:
        for node in progs:
            if rows:
                _check_rows(node, rows, types)
            else:
                cols = [np.zeros(0, np.int32), np.zeros(0, np.int32)]
                assert oracle.count(cols, types, encode(node, types)) == 0


# ---- P3: closed-form tuple multiset (C2 generator, scaled) -------------------------------------

def _closed_form(table, node):
    ta, tb, tc, tm = table.meta["tuples"]
    n = table.n_total
    cols = [ta.astype(np.int32), tb.astype(np.int32), tc.astype(np.uint8)]
    hit = np_mask(node, cols, [INT32, INT32, DICT8], len(ta))
    count = int(tm[hit].sum())
    ends = np.cumsum(tm)
    starts = ends - tm
    a, b, _ = table.meta["affine"]
    j = np.concatenate([np.arange(s, e, dtype=np.int64) for s, e in zip(starts[hit], ends[hit])]
                       or [np.zeros(0, np.int64)])
    ids = np.sort((a * j + b) % n)
    return count, ids


def test_p3_tuple_multiset_closed_form():
    T = configs.gen_c2(600_000)
    cols = [c.numpy() for c in T.columns]
    types = T.types
    rng = np.random.default_rng(5)
    progs = list(configs.c2_probes().values())
    pools = [[0, 1, 2, 3, 4, 5], [0, 500, 501, 1000, 1001, 1002, 1999, 2000, 2001, 2499, 2500],
             list(range(8))]
    progs += [random_program(rng, types[:3], pools, max_depth=3) for _ in range(25)]
    for node in progs:
        want_count, want_ids = _closed_form(T, node)
        c, ids, _ = oracle.pushdown(cols, types, encode(node, types))
        assert c == want_count, node
        np.testing.assert_array_equal(ids, want_ids)


# ---- P4: closed-form affine threshold (C5 generator, scaled) -----------------------------------

@pytest.mark.parametrize("layout", ["scattered", "clustered"])
def test_p4_affine_threshold(layout):
    n = 1_000_000
    T = configs.gen_sweep(n, layout=layout)
    x = T.col("x").numpy()
    a, b, a_inv = T.meta["affine"]
    for s in configs.C5_SELECTIVITIES + [0.0]:
        t = configs.sweep_threshold(n, s)
        prog = encode(configs.sweep_probe(t), T.types)
        c, ids, (y,) = oracle.pushdown([x, T.col("y").numpy()], T.types, prog, proj=[1])
        assert c == t
        v = np.arange(t, dtype=np.int64)
        want = np.sort((a_inv * ((v - b) % n)) % n) if layout == "scattered" else v
        np.testing.assert_array_equal(ids, want)
        np.testing.assert_array_equal(y, T.col("y").numpy()[ids])


# ---- P5: the worked example ------------------------------------------------------------------

def test_p5_worked_example_numbers():
    g = json.load(open(os.path.join(HERE, "golden", "worked_example.json")))
    f = g["leaf_estimates"]["values"]
    prod = f[0] * f[1] * f[2] * f[3]
    assert abs(prod - g["independence_product"]["value"]) <= g["independence_product"]["tolerance"]
    R = g["relation_sizes"]["R"]
    assert abs(prod * R - g["estimated_cardinality"]["value"]) <= g["estimated_cardinality"]["tolerance"]
    assert round(g["actual_selectivity_factor"]["value"] * R) == g["actual_cardinality"]["value"]
    assert round(g["actual_cardinality"]["value"] / g["relation_sizes"]["S"]) == g["plan_gap"]["value"]
    # G7: the printed leaf estimates imply V(R,A) = 5 and V(R,C) = 7.
    assert abs(1 / g["v_R_A"]["value"] - f[0]) < 1e-12
    v = g["v_R_C"]["value"]
    assert round(2 / v - 1 / v ** 2, 2) == f[3]
    assert all(round(2 / d - 1 / d ** 2, 2) != f[3] for d in (5, 6, 8, 9))


def test_p5_worked_example_generator_exact():
    """C2 at 1/1000 scale: the oracle counts exactly 0.167 * N for Listing 3.1 in all three
    encodings, while the data keep V(R,A) = 5, P(A = x) = 0.2 and V(R,C) = 7."""
    g = json.load(open(os.path.join(HERE, "golden", "worked_example.json")))
    n = 600_000
    T = configs.gen_c2(n)
    cols = [c.numpy() for c in T.columns]
    want = g["actual_cardinality"]["value"] * n // g["relation_sizes"]["R"]
    for node in configs.c2_probes().values():
        assert oracle.count(cols, T.types, encode(node, T.types)) == want == 100_200
    assert oracle.count(cols, T.types, encode(Cmp("=", 0, 2), T.types)) == n // 5
    assert len(np.unique(cols[0])) == g["v_R_A"]["value"]
    assert len(np.unique(cols[2])) == g["v_R_C"]["value"]


# ---- P6: invariants --------------------------------------------------------------------------

def test_p6_invariants():
    rng = np.random.default_rng(6)
    types = [INT32, DICT8, INT64, FLOAT32, DICT16]
    n = 4000
    cols, pools = random_table(rng, types, n)
    cnt = lambda node: oracle.count(cols, types, encode(node, types))
    for _ in range(80):
        P = random_program(rng, types, pools, max_depth=3)
        Q = random_program(rng, types, pools, max_depth=3)
        cp, cq, cpq = cnt(P), cnt(Q), cnt(And(P, Q))
        assert cpq <= min(cp, cq)
        assert cp + cnt(Not(P)) == n
        assert cnt(Or(P, Q)) == cp + cq - cpq
        assert cnt(Not(And(P, Q))) == cnt(Or(Not(P), Not(Q)))
        assert cnt(Not(Or(P, Q))) == cnt(And(Not(P), Not(Q)))
        ip = _ids(cols, types, P)
        inp = _ids(cols, types, Not(P))
        assert np.all(np.diff(ip.astype(np.int64)) > 0)
        np.testing.assert_array_equal(np.sort(np.concatenate([ip, inp])), np.arange(n))
    for c, t in enumerate(types):
        if t == FLOAT32:
            continue
        vals = sorted(set(pools[c]))
        for _ in range(10):
            lo, hi = sorted(rng.choice(vals, 2))
            lo, hi = int(lo), int(hi)
            assert cnt(Between(c, lo, hi)) == cnt(Cmp("<=", c, hi)) - cnt(Cmp("<", c, lo))
            L = tuple(int(v) for v in rng.choice(vals, 4))
            assert cnt(In(c, L)) == sum(cnt(Cmp("=", c, v)) for v in set(L))


def test_p6_gather_and_capacity_gate():
    """gathered[k] = col[ids[k]]; with capacity c the first c ids are written and the full
    count returned (Algorithm 1 'count > maxSize'; strict '>' so capacity = count
    passes)."""
    rng = np.random.default_rng(7)
    types = [INT32, DICT8, INT64, FLOAT32, DICT16, DICT32, DATE32]
    n = 3000
    cols, pools = random_table(rng, types, n)
    for _ in range(30):
        P = random_program(rng, types, pools, max_depth=3)
        prog = encode(P, types)
        full, ids, outs = oracle.pushdown(cols, types, prog, proj=list(range(7)) + [0], row_offset=0)
        for j, c in enumerate(list(range(7)) + [0]):
            np.testing.assert_array_equal(outs[j], cols[c][ids])
        for cap in (0, 1, full // 2, full, full + 5):
            c2, ids2, outs2 = oracle.pushdown(cols, types, prog, proj=[2], capacity=cap)
            assert c2 == full
            np.testing.assert_array_equal(ids2, ids[:min(cap, full)])
        off, ids3, _ = oracle.pushdown(cols, types, prog, row_offset=1000)
        np.testing.assert_array_equal(ids3, ids + 1000)


# ---- P7: the paper's fixed points on orders-shaped data -----------------------------------------

def test_p7_orders_fixed_points():
    n = 1_500_000                                        # SF 1 orders
    T = configs.gen_orders(n)
    cols = [c.numpy() for c in T.columns]
    pr = configs.orders_probes()
    # o_orderkey = 1 selects 1 row; o_orderkey >= 1 selects all.
    assert oracle.count(cols, T.types, encode(pr["l5.1"], T.types)) == 1
    assert oracle.count(cols, T.types, encode(pr["l5.2"], T.types)) == n
    # a one-year o_orderdate range keeps ~15.2% (365/2406 = 0.1517).
    frac = oracle.count(cols, T.types, encode(pr["q5_orderdate"], T.types)) / n
    assert abs(frac - 365 / 2406) < 0.0015


# ---- validator: every clause of include/sel.h "Program validation" -------------------------

E_OK, E_TYPE, E_PROG = 0, 3, 4


def _leaf(op=0x10, col=0, a=0, b=0, res=0):
    return (op, col, a, b, res)


VALIDATOR_CASES = [
    # (name, program bytes, column types, expected)
    ("ok_eq", encode_raw([_leaf()], [5]), [INT32], E_OK),
    ("short", b"SELP\x01\x00", [INT32], E_PROG),
    ("magic", encode_raw([_leaf()], [5], magic=b"SELQ"), [INT32], E_PROG),
    ("version", encode_raw([_leaf()], [5], version=2), [INT32], E_PROG),
    ("n_instr0", encode_raw([], [5]), [INT32], E_PROG),
    ("n_instr129", encode_raw([(0x01, 0, 0, 0)] + [(0x01, 0, 0, 0), (0x40, 0, 0, 0)] * 64, []),
     [INT32], E_PROG),
    ("n_consts513", encode_raw([_leaf()], [0] * 513), [INT32], E_PROG),
    ("hdr_reserved", encode_raw([_leaf()], [5], reserved=1), [INT32], E_PROG),
    ("len_plus1", encode_raw([_leaf()], [5]) + b"\x00", [INT32], E_PROG),
    ("len_minus8", encode_raw([_leaf()], [5])[:-8], [INT32], E_PROG),
    ("ins_reserved", encode_raw([_leaf(res=1)], [5]), [INT32], E_PROG),
    ("bad_op", encode_raw([_leaf(op=0x15)], [5]), [INT32], E_PROG),
    ("true_col", encode_raw([(0x01, 1, 0, 0)], []), [INT32, INT32], E_PROG),
    ("and_a", encode_raw([(0x01, 0, 0, 0), (0x01, 0, 0, 0), (0x40, 0, 1, 0)], []), [INT32], E_PROG),
    ("not_b", encode_raw([(0x01, 0, 0, 0), (0x42, 0, 0, 1)], []), [INT32], E_PROG),
    ("col_oob", encode_raw([_leaf(col=1)], [5]), [INT32], E_PROG),
    ("eq_b", encode_raw([_leaf(b=1)], [5, 6]), [INT32], E_PROG),
    ("eq_a_oob", encode_raw([_leaf(a=1)], [5]), [INT32], E_PROG),
    ("between_b_oob", encode_raw([_leaf(op=0x20, a=0, b=1)], [5]), [INT32], E_PROG),
    ("between_ok", encode_raw([_leaf(op=0x20, a=0, b=1)], [5, 6]), [INT32], E_OK),
    ("in_b0", encode_raw([_leaf(op=0x30, a=0, b=0)], [5]), [INT32], E_PROG),
    ("in_b257", encode_raw([_leaf(op=0x30, a=0, b=257)], [1] * 300), [INT32], E_PROG),
    ("in_oob", encode_raw([_leaf(op=0x30, a=1, b=2)], [1, 2]), [INT32], E_PROG),
    ("in_256_ok", encode_raw([_leaf(op=0x30, a=0, b=256)], list(range(256))), [INT32], E_OK),
    ("underflow_and", encode_raw([(0x01, 0, 0, 0), (0x40, 0, 0, 0)], []), [INT32], E_PROG),
    ("underflow_not", encode_raw([(0x42, 0, 0, 0)], []), [INT32], E_PROG),
    ("depth17", encode_raw([(0x01, 0, 0, 0)] * 17 + [(0x40, 0, 0, 0)] * 16, []), [INT32], E_PROG),
    ("depth16_ok", encode_raw([(0x01, 0, 0, 0)] * 16 + [(0x40, 0, 0, 0)] * 15, []), [INT32], E_OK),
    ("final_depth2", encode_raw([(0x01, 0, 0, 0)] * 2, []), [INT32], E_PROG),
    ("i32_hi", encode_raw([_leaf()], [1 << 31]), [INT32], E_TYPE),
    ("i32_lo", encode_raw([_leaf()], [(-(1 << 31) - 1) & (2**64 - 1)]), [INT32], E_TYPE),
    ("i32_min_ok", encode_raw([_leaf()], [(-(1 << 31)) & (2**64 - 1)]), [INT32], E_OK),
    ("date_hi", encode_raw([_leaf()], [1 << 31]), [DATE32], E_TYPE),
    ("i64_any", encode_raw([_leaf()], [2**64 - 1]), [INT64], E_OK),
    ("f32_high", encode_raw([_leaf()], [1 << 32]), [FLOAT32], E_TYPE),
    ("d8_256", encode_raw([_leaf()], [256]), [DICT8], E_TYPE),
    ("d8_255", encode_raw([_leaf()], [255]), [DICT8], E_OK),
    ("d16_65536", encode_raw([_leaf()], [65536]), [DICT16], E_TYPE),
    ("d32_2p32", encode_raw([_leaf()], [1 << 32]), [DICT32], E_TYPE),
    ("between_hi_type", encode_raw([_leaf(op=0x20, a=0, b=1)], [1, 300]), [DICT8], E_TYPE),
    ("in_type", encode_raw([_leaf(op=0x30, a=0, b=3)], [1, 2, 300]), [DICT8], E_TYPE),
    # first failing check wins, in instruction order
    ("type_then_prog", encode_raw([_leaf(a=0), _leaf(op=0x15)], [300]), [DICT8], E_TYPE),
    ("prog_then_type", encode_raw([_leaf(op=0x15), _leaf(a=0)], [300]), [DICT8], E_PROG),
    ("depth_then_type", encode_raw([(0x40, 0, 0, 0), _leaf(a=0)], [300]), [DICT8], E_PROG),
    ("unknown_coltype", encode_raw([_leaf()], [5]), [9], E_TYPE),
    # IN_BITMAP (0x31): a = set id (checked by the probe, not the validator), b must be 0
    ("inbm_ok", encode_raw([(0x31, 0, 7, 0)], []), [INT32], E_OK),
    ("inbm_d8_ok", encode_raw([(0x31, 0, 65535, 0)], []), [DICT8], E_OK),
    ("inbm_i64_ok", encode_raw([(0x31, 0, 0, 0), (0x42, 0, 0, 0)], []), [INT64], E_OK),
    ("inbm_b", encode_raw([(0x31, 0, 0, 1)], []), [INT32], E_PROG),
    ("inbm_col", encode_raw([(0x31, 1, 0, 0)], []), [INT32], E_PROG),
    ("inbm_f32", encode_raw([(0x31, 0, 0, 0)], []), [FLOAT32], E_TYPE),
    ("inbm_f32_then_b", encode_raw([(0x31, 0, 0, 0), (0x31, 0, 0, 1), (0x40, 0, 0, 0)], []),
     [FLOAT32], E_TYPE),
    ("inbm_b_then_f32", encode_raw([(0x31, 0, 0, 1), (0x31, 0, 0, 0), (0x40, 0, 0, 0)], []),
     [FLOAT32], E_PROG),
]


@pytest.mark.parametrize("name,prog,types,want", VALIDATOR_CASES, ids=[c[0] for c in VALIDATOR_CASES])
def test_validator_spec(name, prog, types, want):
    assert oracle.check(prog, types) == want


def test_validator_max_size_program():
    """128 instructions and 512 constants (5,132 bytes, include/sel.h) is accepted."""
    instrs = [(0x30, 0, 0, 256), (0x30, 0, 256, 256), (0x41, 0, 0, 0)]
    while len(instrs) < 127:
        instrs += [(0x10, 0, 0, 0), (0x41, 0, 0, 0)]
    instrs.append((0x42, 0, 0, 0))
    prog = encode_raw(instrs, list(range(512)))
    assert len(prog) == 5132 and len(instrs) == 128
    assert oracle.check(prog, [INT32]) == E_OK
    x = np.arange(-5, 600, dtype=np.int32)
    assert oracle.count([x], [INT32], prog) == int(((x < 0) | (x > 511)).sum())


def test_count_mt_matches_count():
    """The threaded count bench.py times (oracle_count_mt[_bm]) is the same count: shards of any
    size (incl. empty ones), every thread count, with key sets, and errors propagate."""
    rng = np.random.default_rng(404)
    types = [INT32, DICT8, INT64, FLOAT32]
    cols, pools = random_table(rng, types, 1001)
    bms = random_bitmaps(rng, pools)
    for _ in range(20):
        prog = encode(random_program(rng, types, pools, max_depth=3, n_bitmaps=len(bms)), types)
        want = oracle.count(cols, types, prog, bitmaps=bms)
        for nt in (1, 3, 8, 2000):
            assert oracle.count_mt(cols, types, prog, nt, bitmaps=bms) == want
    with pytest.raises(oracle.OracleError) as e:
        oracle.count_mt(cols, types, encode(InSet(0, 9), types), 4, bitmaps=bms)
    assert e.value.status == 1


def test_pushdown_mt_matches_pushdown():
    """The row-sharded push-down (oracle_pushdown_mt_bm, used to check whole full-size tables in
    tests/test_gpu_fullsize.py) returns exactly oracle_pushdown's ids and gathered bytes: every
    thread count (incl. more threads than rows: empty shards), capacity cuts inside and between
    shards (Algorithm 1's gate), row offsets, key sets, every column type, and
    errors propagate."""
    rng = np.random.default_rng(405)
    types = [INT32, DICT8, INT64, FLOAT32, DICT16, DICT32, DATE32]
    n = 1777
    cols, pools = random_table(rng, types, n)
    bms = random_bitmaps(rng, pools)
    proj = list(range(7)) + [2]
    for i in range(25):
        prog = encode(random_program(rng, types, pools, max_depth=3, n_bitmaps=len(bms)), types)
        full, ids, outs = oracle.pushdown(cols, types, prog, proj=proj, bitmaps=bms,
                                          row_offset=123 * i)
        for nt in (1, 2, 7, 16) + ((2500,) if i < 3 else ()):   # 2500 > n: empty shards
            caps = (None, 0, 1, full // 3, full, full + 9) if nt in (7, 2500) else (None,)
            for cap in caps:
                c, ids2, outs2 = oracle.pushdown_mt(cols, types, prog, proj=proj, capacity=cap,
                                                    row_offset=123 * i, bitmaps=bms, nthreads=nt)
                k = full if cap is None else min(cap, full)
                assert c == full
                np.testing.assert_array_equal(ids2, ids[:k])
                for a, b in zip(outs2, outs):
                    assert a.tobytes() == b[:k].tobytes()
    with pytest.raises(oracle.OracleError) as e:
        oracle.pushdown_mt(cols, types, encode(InSet(0, 9), types), bitmaps=bms, nthreads=4)
    assert e.value.status == 1
    empty = [c[:0] for c in cols]
    c, ids0, outs0 = oracle.pushdown_mt(empty, types, encode(Cmp("<", 0, 5), types), proj=[1],
                                        nthreads=4)
    assert c == 0 and len(ids0) == 0 and len(outs0[0]) == 0


def test_pushdown_mt_closed_forms():
    """The sharded push-down against the closed forms, not only against oracle_pushdown: C2's
    tuple multiset (P3) and the affine threshold (P4) at 1/1000 scale, on 16 threads."""
    T = configs.gen_c2(600_000)
    cols = [c.numpy() for c in T.columns]
    for node in configs.c2_probes().values():
        want_count, want_ids = _closed_form(T, node)
        c, ids, (d,) = oracle.pushdown_mt(cols, T.types, encode(node, T.types), proj=[3],
                                          nthreads=16)
        assert c == want_count == 100_200
        np.testing.assert_array_equal(ids, want_ids)
        np.testing.assert_array_equal(d, cols[3][want_ids])
    n = 1_000_000
    S = configs.gen_sweep(n)
    x, y = S.col("x").numpy(), S.col("y").numpy()
    a, b, a_inv = S.meta["affine"]
    for s in (1e-4, 0.1, 0.5):
        t = configs.sweep_threshold(n, s)
        c, ids, (yy,) = oracle.pushdown_mt([x, y], S.types, encode(configs.sweep_probe(t), S.types),
                                           proj=[1], nthreads=16)
        v = np.arange(t, dtype=np.int64)
        assert c == t
        np.testing.assert_array_equal(ids, np.sort((a_inv * ((v - b) % n)) % n))
        np.testing.assert_array_equal(yy, y[ids])


# ---- oracle/synopsis.py: the equi-depth histogram baseline ----------------

def test_equi_depth_paper_example_49_3():
    """"if we try to estimate the selectivity where the attribute involved equals
    to 16, 30/2 + 30/1 + 30/7 = 49.3": three buckets of depth D = 30 hold 16, with 2, 1 and 7
    distinct values (DESIGN.md §2 reading: the per-bucket estimates D / V(b) add up)."""
    from oracle import synopsis
    values = np.array([10] * 15 + [16] * (15 + 30 + 24) + list(range(17, 23)), np.int32)
    h = synopsis.equi_depth(values, 3)
    assert h["rows"].tolist() == [30, 30, 30]
    assert h["distinct"].tolist() == [2, 1, 7]
    est = synopsis.estimate_eq(h, 16, len(values))
    assert round(est, 1) == 49.3 and abs(est - (30 / 2 + 30 / 1 + 30 / 7)) < 1e-12
    assert synopsis.estimate_eq(h, 11, len(values)) == 15.0       # inside bucket 0 only: D / 2
    assert synopsis.estimate_eq(h, 99, len(values)) == 0.0        # outside every bucket


def test_equi_depth_brute_force_small():
    from oracle import synopsis
    rng = np.random.default_rng(3)
    for _ in range(300):
        m = int(rng.integers(0, 60))
        B = int(rng.integers(1, 9))
        v = rng.integers(-5, 6, m).astype(np.int32)
        h = synopsis.equi_depth(v, B)
        s = sorted(v.tolist())
        assert int(h["rows"].sum()) == m
        for b in range(B):
            part = s[b * m // B:(b + 1) * m // B]
            assert int(h["rows"][b]) == len(part) in (m // B, -(-m // B))
            assert int(h["distinct"][b]) == len(set(part))
            if part:
                assert (h["lo"][b], h["hi"][b]) == (min(part), max(part))
        # uniform data with one value per bucket: the estimate is exact
    u = np.repeat(np.arange(8, dtype=np.int32), 5)
    h = synopsis.equi_depth(u, 8)
    assert all(synopsis.estimate_eq(h, x, 40) == 5.0 for x in range(8))


def test_block_sample_rows():
    from oracle import synopsis
    v = np.arange(5000)
    s = synopsis.block_sample(v, 3, 1)
    assert s.tolist() == list(range(1024, 2048)) + list(range(4096, 5000))
