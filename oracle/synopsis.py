"""oracle/synopsis.py — TEST INFRASTRUCTURE ONLY (task rule ③): the equi-depth histogram and its
equality estimate written out from the paper, for parity with sel_histogram.

    equi_depth(values, B)      sort the values; bucket b holds sorted positions
                               [floor(b m / B), floor((b+1) m / B)); report lo, hi, rows and the
                               number of distinct values V(b) of each bucket.
    estimate_eq(h, x, T)       |sigma_{A=x}(R)| = D / V(b_x), D = T / B, summed
                               over the buckets whose [lo, hi] contains x (DESIGN.md §2 reading
                               of the paper's "30/2 + 30/1 + 30/7 = 49.3" example).
    block_sample(values, s, p) the rows of the 1024-row chunks c with c mod s == p.

Pinned by tests/test_oracle_pins.py (the paper's printed 49.3; brute-force distinct counts and
bucket sizes on tiny inputs)."""

from __future__ import annotations

import numpy as np


def block_sample(values: np.ndarray, stride: int, phase: int) -> np.ndarray:
    n = len(values)
    parts = [values[c * 1024:min(n, c * 1024 + 1024)]
             for c in range(phase, (n + 1023) // 1024, stride)]
    return np.concatenate(parts) if parts else values[:0]


def equi_depth(values: np.ndarray, buckets: int) -> dict:
    s = np.sort(np.asarray(values).astype(np.int64), kind="stable")
    m = len(s)
    lo, hi, rows, distinct = [], [], [], []
    for b in range(buckets):
        a, e = b * m // buckets, (b + 1) * m // buckets
        part = s[a:e]
        rows.append(e - a)
        distinct.append(len(set(part.tolist())))
        lo.append(int(part[0]) if e > a else 0)
        hi.append(int(part[-1]) if e > a else 0)
    return {"lo": np.array(lo, np.int64), "hi": np.array(hi, np.int64),
            "rows": np.array(rows, np.uint64), "distinct": np.array(distinct, np.uint64),
            "sample_rows": m}


def estimate_eq(hist: dict, x: int, table_rows: int) -> float:
    d = table_rows / len(hist["rows"])
    return float(sum(d / int(v) for lo, hi, v in zip(hist["lo"], hist["hi"], hist["distinct"])
                     if int(v) and lo <= x <= hi))
