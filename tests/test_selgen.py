"""Input generators: determinism, shard/chunk invariance, and the workload shapes DESIGN.md's
input recipe states."""

import numpy as np
import torch

import selgen
from selgen import configs
from selgen.program import encode, Cmp, In, And, Not, Const, INT32, DICT8, DICT16, FLOAT32


def _cat(tables, name):
    return np.concatenate([t.col(name).numpy() for t in tables])


def test_hash_deterministic_and_exact():
    i = torch.arange(0, 1 << 20, dtype=torch.int64)
    a = selgen.h32(123, i)
    b = selgen.h32(123, i)
    assert torch.equal(a, b)
    assert int(a.min()) >= 0 and int(a.max()) < (1 << 32)
    # multiply-shift uniform ints cover the range evenly (chi-square, 10 bins, p ~ 1e-6 bound)
    u = selgen.uniform_int(7, i, 0, 9).numpy()
    obs = np.bincount(u, minlength=10)
    exp = len(u) / 10
    assert ((obs - exp) ** 2 / exp).sum() < 40


def test_shards_concatenate_to_full_table():
    n = 120_000
    full = configs.gen_c2(n, chunk=7777)
    parts = [configs.gen_c2(n, row_start=s, row_count=e - s, chunk=5000)
             for s, e in [(0, 40_000), (40_000, 40_001), (40_001, n)]]
    for c in "ABCD":
        np.testing.assert_array_equal(_cat(parts, c), full.col(c).numpy())
    L = configs.gen_lineitem(10_000)
    Lp = [configs.gen_lineitem(10_000, s, 5000) for s in (0, 5000)]
    for c in configs.LINEITEM_COLS:
        np.testing.assert_array_equal(_cat(Lp, c), L.col(c).numpy())


def test_c2_group_structure():
    n = 600_000
    T = configs.gen_c2(n)
    ta, tb, tc, tm = T.meta["tuples"]
    assert tm.sum() == n
    A, B, C = (T.col(c).numpy() for c in "ABC")
    # each A value holds exactly N/5 rows (V(R,A) = 5)
    np.testing.assert_array_equal(np.bincount(A), [n // 5] * 5)
    assert set(np.unique(C)) == set(range(7))
    # the multiset matches the tuple list exactly
    keys = A.astype(np.int64) * 10**7 + B.astype(np.int64) * 10 + C
    tk = ta * 10**7 + tb * 10 + tc
    u, cnt = np.unique(keys, return_counts=True)
    order = np.argsort(tk)
    np.testing.assert_array_equal(u, tk[order])
    np.testing.assert_array_equal(cnt, tm[order])


def test_lineitem_shape():
    T = configs.gen_lineitem(200_000)
    sd = T.col("l_shipdate").numpy()
    rd = T.col("l_receiptdate").numpy()
    rf = T.col("l_returnflag").numpy()
    assert sd.min() >= configs.ORDERDATE_LO + 1 and sd.max() <= configs.ORDERDATE_HI + 121
    assert (rd > sd).all() and (rd - sd <= 30).all()
    assert set(np.unique(rf[rd > configs.RETURN_CUTOFF])) == {1}         # 'N'
    assert set(np.unique(rf[rd <= configs.RETURN_CUTOFF])) == {0, 2}      # 'A' / 'R'
    assert set(np.unique(T.col("l_shipmode").numpy())) == set(range(7))


def test_lineorder_dates_are_yyyymmdd():
    T = configs.gen_lineorder(50_000)
    d = T.col("lo_orderdate").numpy()
    assert d.min() >= 19920101 and d.max() <= 19980802
    assert ((d % 100) >= 1).all() and ((d // 100 % 100) <= 12).all()


def test_program_encoding_layout():
    p = encode(And(Cmp("=", 0, -1), In(1, (3, 4))), [INT32, DICT8])
    assert p[:4] == b"SELP"
    assert len(p) == 12 + 8 * (3 + 3)
    assert p[12:20] == bytes([0x10, 0, 0, 0, 0, 0, 0, 0])
    assert p[20:28] == bytes([0x30, 1, 1, 0, 2, 0, 0, 0])
    assert p[36:44] == b"\xff" * 8                        # -1 sign-extended
    f = encode(Cmp("<", 0, -0.0), [FLOAT32])
    assert f[-8:] == bytes([0, 0, 0, 0x80, 0, 0, 0, 0])  # binary32 bits, high word zero


def test_inset_encoding_layout():
    """IN_BITMAP instruction: op 0x31, col, a = set id, b = 0, no constants (include/sel.h)."""
    from selgen.program import InSet
    b = encode(Not(InSet(1, 513)), [INT32, DICT16])
    assert b[:4] == b"SELP" and b[6:8] == b"\x02\x00" and b[8:10] == b"\x00\x00"
    assert b[12:20] == bytes([0x31, 1, 0x01, 0x02, 0, 0, 0, 0])
    assert b[20:28] == bytes([0x42, 0, 0, 0, 0, 0, 0, 0]) and len(b) == 28
