"""The C-ABI boundary on CPU (no compute calls need a GPU here):
  * libsel.so loads and exports exactly the functions include/sel.h declares;
  * its validator (canon.cpp) agrees with the oracle's (oracle.c) on the spec cases and on
    fuzzed/mutated program bytes — two independent implementations of include/sel.h;
  * its canonical plan is exact: the packed device arithmetic ((v - lo) mod 2^W <= span per
    interval, AND/OR postfix), emulated here in NumPy, selects exactly the oracle's rows;
  * the Python predicate builder writes the same bytes as the input generator.
"""

import ctypes
import math
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_1806_08384_b200 as sel
from paper_1806_08384_b200 import _native, col
from selgen.program import (InSet, Cmp, Between, In, And, Or, Not, Const, encode, encode_raw,
                            random_program, INT32, INT64, FLOAT32, DATE32, DICT8, DICT16, DICT32)

from helpers import random_table
from test_oracle_pins import VALIDATOR_CASES

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    hdr = open(os.path.join(ROOT, "include", "sel.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(sel_[a-z_0-9]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    declared = _declared()
    assert declared == sorted(_native.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = sorted(set(re.findall(r" T (sel_[a-z_0-9]+)$", out, flags=re.M)))
    assert exported == declared
    for name in declared:
        assert hasattr(lib, name)
    assert lib.sel_abi_version() == 1


@pytest.mark.parametrize("name,prog,types,want", VALIDATOR_CASES, ids=[c[0] for c in VALIDATOR_CASES])
def test_validator_matches_spec(name, prog, types, want):
    assert sel.program_check(prog, types) == want


def test_validator_parity_fuzz():
    rng = np.random.default_rng(99)
    types = [INT32, DICT8, FLOAT32, INT64, DICT16]
    cols, pools = random_table(rng, types, 10)
    seeds = [encode(random_program(rng, types, pools, 3), types) for _ in range(200)]
    n = 0
    for base in seeds:
        for _ in range(25):
            b = bytearray(base)
            k = int(rng.integers(1, 4))
            for _ in range(k):
                r = rng.random()
                if r < 0.6 and len(b):
                    b[int(rng.integers(len(b)))] = int(rng.integers(256))
                elif r < 0.8:
                    b = b[: int(rng.integers(len(b) + 1))]
                else:
                    b += bytes(rng.integers(0, 256, int(rng.integers(1, 9)), dtype=np.uint8))
            b = bytes(b)
            assert sel.program_check(b, types) == oracle.check(b, types), b.hex()
            n += 1
    assert n == 5000


def test_error_message_thread_local_and_set():
    assert sel.program_check(b"nope", [INT32]) == 4
    assert "short" in _native.lib().sel_last_error_message().decode()
    assert _native.lib().sel_last_error() == 4
    assert sel.program_check(encode(Cmp("=", 0, 1), [INT32]), [INT32]) == 0
    assert _native.lib().sel_last_error() == 0


# ---- canonicaliser exactness (device arithmetic emulated in NumPy) ----------------------------

_U = {INT32: np.uint32, DATE32: np.uint32, FLOAT32: np.uint32, DICT32: np.uint32, INT64: np.uint64,
      DICT8: np.uint8, DICT16: np.uint16}


def emulate_plan(plan, cols, types, n, bitmaps=None):
    if plan["path"] == 2:
        return np.full(n, plan["const"])
    masks = []
    for L in plan["leaves"]:
        c = L["col"]
        raw = cols[c].view(_U[types[c]]).astype(np.uint64)
        if "bitmap" in L:   # raw unsigned value < nbits and its bit set (kernels.cu bitmap_test)
            words, nbits = bitmaps[L["bitmap"]]
            inr = raw < np.uint64(nbits)
            k = np.where(inr, raw, np.uint64(0)).astype(np.int64)
            bit = (words[k >> 6] >> (k & 63).astype(np.uint64)) & np.uint64(1)
            m = inr & (bit == 1)
            masks.append(~m if L["negate"] else m)
            continue
        if L["fkey"]:
            sign = (raw >> np.uint64(31)) & np.uint64(1)
            raw = raw ^ np.where(sign == 1, np.uint64(0xFFFFFFFF), np.uint64(0x80000000))
        W = 64 if L["wclass"] == 3 else 32
        mod = np.uint64((1 << 64) - 1) if W == 64 else np.uint64(0xFFFFFFFF)
        m = np.zeros(n, dtype=bool)
        for lo, sp in zip(L["lo"], L["span"]):
            m |= ((raw - np.uint64(lo)) & mod) <= np.uint64(sp)
        masks.append(m)
    st = []
    for op, arg in plan["ops"]:
        if op == 0:
            st.append(masks[arg])
        else:
            y, x = st.pop(), st.pop()
            st.append(x & y if op == 1 else x | y)
    assert len(st) == 1
    return st[0]


@pytest.mark.parametrize("types", [
    [INT32, DICT8, FLOAT32], [INT64, DATE32, DICT16], [DICT32, INT32, INT64, FLOAT32],
])
def test_plan_is_exact_vs_oracle(types):
    rng = np.random.default_rng(sum(types) + 5)
    n = 2000
    cols, pools = random_table(rng, types, n, with_nan=FLOAT32 in types)
    paths = set()
    with np.errstate(over="ignore"):
        for _ in range(300):
            node = random_program(rng, types, pools, max_depth=4)
            prog = encode(node, types)
            plan = sel.program_plan(prog, types)
            paths.add(plan["path"])
            got = np.flatnonzero(emulate_plan(plan, cols, types, n))
            _, want, _ = oracle.pushdown(cols, types, prog)
            np.testing.assert_array_equal(got, want, err_msg=str(node))
    assert paths == {0, 1, 2}


@pytest.mark.parametrize("types", [[INT32, DICT8, INT64], [DICT16, DATE32, DICT32, FLOAT32]])
def test_plan_inset_exact_vs_oracle(types):
    """IN_BITMAP leaves through the canonicaliser: NOT folds into the leaf's negate flag, the leaf
    is never merged with interval leaves, and the plan selects exactly the oracle's rows."""
    from helpers import random_bitmaps
    rng = np.random.default_rng(sum(types) + 17)
    n = 2000
    cols, pools = random_table(rng, types, n)
    for c, t in enumerate(types):
        if t != FLOAT32:
            small = rng.integers(0, 256 if t == DICT8 else 1100, n)
            cols[c] = np.where(rng.random(n) < 0.5, small.astype(cols[c].dtype), cols[c])
    bms = random_bitmaps(rng, pools)
    negated = 0
    with np.errstate(over="ignore"):
        for _ in range(300):
            node = random_program(rng, types, pools, max_depth=4, n_bitmaps=len(bms))
            prog = encode(node, types)
            plan = sel.program_plan(prog, types)
            negated += sum(1 for L in plan.get("leaves", []) if L.get("negate"))
            got = np.flatnonzero(emulate_plan(plan, cols, types, n, bms))
            _, want, _ = oracle.pushdown(cols, types, prog, bitmaps=bms)
            np.testing.assert_array_equal(got, want, err_msg=str(node))
    assert negated > 0


def test_plan_paths_of_the_paper_predicates():
    from selgen import configs
    for node in configs.c2_probes().values():
        assert sel.program_path(encode(node, [INT32, INT32, DICT8, INT32]), [INT32, INT32, DICT8, INT32]) == 1
    assert sel.program_path(encode(Or(Cmp("=", 0, 1), Cmp("=", 1, 2)), [INT32, INT32]), [INT32, INT32]) == 0
    assert sel.program_path(encode(Or(Cmp("<", 0, 5), Cmp(">=", 0, 5)), [INT32]), [INT32]) == 2
    # NOT(x < c) on floats keeps NaN rows: never rewritten as x >= c
    plan = sel.program_plan(encode(Not(Cmp("<", 0, 1.0)), [FLOAT32]), [FLOAT32])
    assert len(plan["leaves"][0]["lo"]) == 2


# ---- predicate builder ---------------------------------------------------------------------------

def test_builder_bytes_match_generator():
    schema = [("A", INT32, None), ("B", INT32, None), ("C", DICT8, ["a", "b", "c", "d", "e"])]
    types = [INT32, INT32, DICT8]
    cases = [
        ((col("A") == 2) & (col("B") < 2001) & (col("B") > 1000) & ((col("C") == 1) | (col("C") == 4)),
         And(And(And(Cmp("=", 0, 2), Cmp("<", 1, 2001)), Cmp(">", 1, 1000)), Or(Cmp("=", 2, 1), Cmp("=", 2, 4)))),
        (col("B").between(-5, 7) | ~col("C").isin([0, 3]), Or(Between(1, -5, 7), Not(In(2, (0, 3))))),
        (col("C").isin(["b", "e", "zz"]), In(2, (1, 4))),
        (col("C") == "zz", Const(False)),
        (col("C") < "c", Cmp("<", 2, 2)),
        (col("C") <= "bb", Cmp("<=", 2, 1)),
        (col("B").in_set(3) & ~col("C").in_set(0), And(InSet(1, 3), Not(InSet(2, 0)))),
    ]
    for expr, node in cases:
        assert sel.predicate.compile_predicate(expr, schema) == encode(node, types)


def test_builder_float32_constants_exact():
    """a FLOAT32 leaf compares the column with the EXACT constant (SQL semantics of a
    binary32 value against a literal): builder + oracle select exactly the rows Python's exact
    float/int comparison selects, for constants float32 cannot represent (0.7, 1e-46, 1e39,
    2**60 + 1) and ones it can (0.5, -0.0, inf), under every operator, BETWEEN and IN."""
    import operator
    import struct as st
    xs = [0.7, 0.69999999, 0.70000005, -0.7, 0.5, -0.0, 0.0, 1e-45, -1e-45, 3.4028234663852886e38,
          float("inf"), float("-inf"), float("nan"), 2.0 ** 60, 1.0, 1e30]
    x = np.array(xs + [float(np.nextafter(np.float32(v), np.float32(np.inf))) for v in xs[:5]]
                 + [float(np.nextafter(np.float32(v), np.float32(-np.inf))) for v in xs[:5]],
                 dtype=np.float32)
    vals = [float(v) for v in x]                        # the stored binary32 values, exactly
    schema = [("f", FLOAT32, None)]
    cmp = {"<": operator.lt, "<=": operator.le, ">": operator.gt, ">=": operator.ge, "=": operator.eq}
    ids = lambda e: oracle.pushdown([x], [FLOAT32], sel.predicate.compile_predicate(e, schema))[1]
    consts = [0.7, -0.7, 1e-46, 1e39, -1e39, 2 ** 60 + 1, 2 ** 60, 0.5, -0.0, float("inf"), 1e-45,
              0.1, 1 / 3]
    for c in consts:
        for op, f in cmp.items():
            e = {"<": col("f") < c, "<=": col("f") <= c, ">": col("f") > c, ">=": col("f") >= c,
                 "=": col("f") == c}[op]
            want = [i for i, v in enumerate(vals) if f(v, c)]
            np.testing.assert_array_equal(ids(e), want, err_msg=f"{op} {c!r}")
    for lo, hi in [(0.1, 0.7), (-0.7, 1 / 3), (1e-46, 1e39), (0.5, 0.5), (0.7, 0.7)]:
        want = [i for i, v in enumerate(vals) if lo <= v <= hi]
        np.testing.assert_array_equal(ids(col("f").between(lo, hi)), want, err_msg=f"{lo}..{hi}")
    want = [i for i, v in enumerate(vals) if v in (0.7, 0.5, 1e39) or v == 0.5]
    np.testing.assert_array_equal(ids(col("f").isin([0.7, 0.5, 1e39])), want)
    assert sel.predicate.compile_predicate(col("f").isin([0.7, 0.1]), schema) == encode(Const(False), [FLOAT32])
    # the constant carried is a float32 (bits), so exactly representable constants pass unchanged
    prog = sel.predicate.compile_predicate(col("f") < 0.5, schema)
    assert st.unpack("<Q", prog[-8:])[0] == st.unpack("<I", st.pack("<f", 0.5))[0]


def test_builder_full_dictionary_bounds_fold():
    """a string bound sorting after every entry of a FULL DICT8 / DICT16 dictionary
    folds to TRUE ('<') / FALSE ('>=') instead of failing to encode code 256 / 65536."""
    for t, size in ((DICT8, 256), (DICT16, 65536)):
        d = [f"s{i:06d}" for i in range(size)]
        schema = [("s", t, d)]
        cp = lambda e: sel.predicate.compile_predicate(e, schema)
        assert cp(col("s") < "zzz") == encode(Const(True), [t])
        assert cp(col("s") >= "zzz") == encode(Const(False), [t])
        assert cp(col("s") < "s000001") == encode(Cmp("<", 0, 1), [t])
        assert cp(col("s").between("a", "zzz")) == encode(Between(0, 0, size - 1), [t])


def test_output_capacity_never_exceeds_caller_buffers():
    """with caller buffers (out=) the capacity defaults to what they hold and an
    explicit larger capacity is refused, so no kernel writes past a user tensor."""
    import torch
    from paper_1806_08384_b200.api import _fit_capacity
    ids, cols = torch.empty(10, dtype=torch.int32), [torch.empty(7), torch.empty(12)]
    assert _fit_capacity(None, 100, (ids, cols)) == 7
    assert _fit_capacity(None, 5, (ids, cols)) == 5
    assert _fit_capacity(7, 100, (ids, cols)) == 7
    with pytest.raises(ValueError):
        _fit_capacity(8, 100, (ids, cols))
    assert _fit_capacity(None, 100, None) == 100 and _fit_capacity(3, 100, None) == 3


def test_synopsis_estimators_in_the_library():
    """The NEXT(4) estimators are C entry points (sel_sample_estimate, sel_equi_depth_estimate;
    host arithmetic, no GPU): the paper's printed 49.3 from the oracle's
    histogram of the paper's example, and agreement with oracle/synopsis.estimate_eq on random
    histograms; the sampling estimator |sigma(R')| |R| / |R'|."""
    from oracle import synopsis
    values = np.array([10] * 15 + [16] * (15 + 30 + 24) + list(range(17, 23)), np.int32)
    h = synopsis.equi_depth(values, 3)
    h["table_rows"] = len(values)
    assert round(sel.equi_depth_estimate(h, 16), 1) == 49.3
    assert sel.equi_depth_estimate(h, 11) == 15.0 and sel.equi_depth_estimate(h, 99) == 0.0
    rng = np.random.default_rng(12)
    for _ in range(200):
        v = rng.integers(-50, 50, int(rng.integers(1, 400))).astype(np.int32)
        B = int(rng.integers(1, 20))
        h = synopsis.equi_depth(v, B)
        h["table_rows"] = int(rng.integers(len(v), 10 * len(v) + 1))
        for x in rng.integers(-60, 60, 5):
            want = synopsis.estimate_eq(h, int(x), h["table_rows"])
            assert abs(sel.equi_depth_estimate(h, int(x)) - want) <= 1e-9 * max(1.0, want)
    L = _native.lib()
    assert L.sel_sample_estimate(7, 100, 1000) == 70.0 and L.sel_sample_estimate(5, 0, 10) == 0.0
    assert math.isnan(L.sel_equi_depth_estimate(None, None, None, 0, 10, 1))
