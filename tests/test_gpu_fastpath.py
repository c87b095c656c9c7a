"""GPU parity of the count kernel's conjunctive fast path (sel_internal.h FastKind; SURVEY §8a
a2/a3 "template-specialised fast paths for conjunctive range/equality forms") against the CPU
oracle: random conjunctions of 1..4 leaves of every fast kind — point / interval / 2..4
intervals on 4-byte columns, an interval on an 8-byte column, 1..4 points on a 1-byte column
(SWAR) — in every leaf slot, on boundary-heavy tables of ragged sizes (full chunks take the fast
path, the tail chunk the interpreter), through the count, the sampled count and every push-down
path. Bit-exact."""


import numpy as np
import pytest

import oracle
import paper_1806_08384_b200 as sel
from selgen.program import (Cmp, Between, In, And, Not, encode, INT32, INT64, DATE32, DICT8,
                            DICT32)

from helpers import random_table
from test_gpu_parity import check_parity, register

TYPES = [INT32, DATE32, DICT32, INT64, DICT8, DICT8]


def _pick(rng, pool):
    return int(pool[int(rng.integers(len(pool)))])


def fast_leaf(rng, c, t, pool):
    r = rng.random()
    if t == DICT8:
        if r < 0.3:
            return Cmp("=", c, _pick(rng, pool))
        if r < 0.6:
            lo = _pick(rng, pool)
            return Between(c, lo, min(255, lo + int(rng.integers(0, 4))))
        return In(c, tuple(_pick(rng, pool) for _ in range(int(rng.integers(1, 5)))))
    if t == INT64:
        if r < 0.6:
            return Cmp(["=", "<", ">", "<=", ">="][int(rng.integers(5))], c, _pick(rng, pool))
        return Between(c, _pick(rng, pool), _pick(rng, pool))
    if r < 0.35:
        return Cmp(["=", "<", ">", "<=", ">="][int(rng.integers(5))], c, _pick(rng, pool))
    if r < 0.55:
        return Between(c, _pick(rng, pool), _pick(rng, pool))
    if r < 0.8:
        return In(c, tuple(_pick(rng, pool) for _ in range(int(rng.integers(2, 5)))))
    return Not(Cmp("=", c, _pick(rng, pool)))          # two intervals


def fast_conjunction(rng, pools):
    k = int(rng.integers(1, 5))
    cols = rng.choice(len(TYPES), size=k, replace=False)
    node = None
    for c in cols:
        leaf = fast_leaf(rng, int(c), TYPES[int(c)], pools[int(c)])
        node = leaf if node is None else And(node, leaf)
    return node


def fast_kinds(node):
    plan = sel.program_plan(encode(node, TYPES), TYPES)
    return plan.get("fast", [])


def test_plan_fast_classification():
    """Host-side: which programs take the fast path (no GPU)."""
    assert fast_kinds(And(Cmp("=", 0, 2), Between(1, 5, 9))) == [0, 1]
    assert fast_kinds(In(4, (1, 4))) == [4]
    assert fast_kinds(Between(4, 1, 4)) == [4]                # 4 points: SWAR
    assert fast_kinds(Between(4, 1, 5)) == []                 # 5 points: interpreter
    assert fast_kinds(Not(Cmp("=", 0, 3))) == [2]             # two intervals
    assert fast_kinds(Cmp("<", 3, 10)) == [3]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 1023, 1024, 1025, 8193, 65537, 250_003])
def test_fast_conjunctions_ragged(ctx, n):
    rng = np.random.default_rng(1000 + n)
    cols, pools = random_table(rng, TYPES, n)
    t = register(ctx, cols, TYPES)
    hits = 0
    for _ in range(30):
        node = fast_conjunction(rng, pools)
        hits += bool(fast_kinds(node))
        check_parity(t, cols, TYPES, node, proj=[0, 3, 4, 5])
    assert hits >= 20


@pytest.mark.gpu
def test_fast_sampled_count(ctx):
    """The block-sampled count (chunk stride/phase) through the fast kernel."""
    rng = np.random.default_rng(77)
    n = 200_003
    cols, pools = random_table(rng, TYPES, n)
    t = register(ctx, cols, TYPES)
    for _ in range(10):
        node = fast_conjunction(rng, pools)
        prog = encode(node, TYPES)
        for stride, phase in [(1, 0), (3, 1), (7, 6)]:
            got, rows, _ = t.count_sampled(prog, stride, phase)
            # oracle over exactly the sampled 1024-row chunks
            idx = np.concatenate([np.arange(c * 1024, min(n, c * 1024 + 1024))
                                  for c in range(phase, (n + 1023) // 1024, stride)])
            want = oracle.count([c[idx] for c in cols], TYPES, prog)
            assert (got, rows) == (want, len(idx)), (node, stride, phase)


@pytest.fixture(scope="module")
def ctx(cuda_device):
    c = sel.Context(cuda_device)
    yield c
    c.close()
