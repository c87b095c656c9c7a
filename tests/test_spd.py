"""Algorithm 1 host driver: structural properties on CPU with an oracle-backed
Execute (SPEC.md:632 acceptance 4: ratio 0 never pushes a non-empty selection, ratio 1.0 pushes
every qualifying non-probe selection, relations <= min size are never pushed, the largest relation
is never pushed), and the real GPU Execute on a desk-scale replica of the worked example."""

import numpy as np
import pytest

import oracle
from paper_1806_08384_b200.spd import Relation, evaluate_and_push_down, max_size_for
from selgen import configs, encode
from selgen.program import Cmp


def _oracle_execute(data):
    def execute(rel, max_size):
        cols, types = data[rel.name]
        prog = encode(rel.predicate, types)
        count = oracle.count(cols, types, prog)
        if count > max_size:                            # "throw"
            return count, False, None
        return count, True, oracle.pushdown(cols, types, prog, proj=list(rel.project))
    return execute


def _relations(rng, k):
    rels, data = [], {}
    for i in range(k):
        n = int(rng.integers(0, 5000))
        x = rng.integers(0, 100, n).astype(np.int32)
        t = int(rng.integers(0, 110))
        pred = None if rng.random() < 0.15 else Cmp("<", 0, t)
        rels.append(Relation(f"r{i:02d}", n, pred, [0]))
        data[f"r{i:02d}"] = ([x], [1])
    return rels, data


@pytest.mark.parametrize("seed", range(40))
def test_algorithm1_structure(seed):
    rng = np.random.default_rng(seed)
    rels, data = _relations(rng, int(rng.integers(1, 9)))
    min_size = int(rng.integers(0, 3000))
    for ratio in (0.0, 1.0, float(rng.random()), int(rng.integers(0, 3000))):
        dec = evaluate_and_push_down(rels, min_size, ratio, execute=_oracle_execute(data))
        by = {d.name: d for d in dec}
        assert sorted(by) == sorted(r.name for r in rels)
        big = [r for r in rels if r.size > min_size]
        if big:
            largest = sorted(big, key=lambda r: (-r.size, r.name))[0]
            assert by[largest.name].role == "probe" and not by[largest.name].pushed
        for r in rels:
            d = by[r.name]
            if r.size <= min_size:
                assert d.role == "too_small" and not d.pushed
            elif d.role == "evaluated":
                want = oracle.count(data[r.name][0], data[r.name][1], encode(r.predicate, [1]))
                assert d.count == want
                ms = max_size_for(r.size, ratio)
                assert d.pushed == (d.count <= ms)             # gate soundness
                if ratio == 0.0:
                    assert d.pushed == (d.count == 0)          # only empty selections pass ratio 0
                if ratio == 1.0:
                    assert d.pushed                            # every selection passes ratio 1.0
        # processing order: probe, then the queue by descending size (ties by name)
        ev = [d for d in dec if d.role in ("evaluated", "no_condition")]
        assert [d.size for d in ev] == sorted((d.size for d in ev), reverse=True)


def test_max_size_reading():
    assert max_size_for(600_000_000, 1.0) == 600_000_000
    assert max_size_for(75_000_000, 0.044) == 3_300_000            # orders crossover
    assert max_size_for(10, 0.0) == 0
    assert max_size_for(10, 7) == 7                                 # absolute form


@pytest.mark.gpu
def test_algorithm1_on_gpu_worked_example(cuda_device):
    """Desk-scale replica of the worked example (R 600k, S 5k, T 1k rows): R is the
    largest, so it is the probe side and never pushed; with R's predicate moved onto S and T's
    key ranges the exact counts drive the push-down decisions."""
    import paper_1806_08384_b200 as sel
    ctx = sel.Context(cuda_device)
    R = configs.gen_c2(600_000, device=cuda_device)
    S = configs.gen_c2(6_000, device=cuda_device)
    T = configs.gen_c2(12_000, device=cuda_device)
    tabs = {nm: sel.Table(ctx, list("ABCD"), X.types, [c.data for c in X.columns])
            for nm, X in (("R", R), ("S", S), ("T", T))}
    pred = configs.c2_probes()["listing"]
    prog = encode(pred, R.types)                                   # the pushed-down conditions
    rels = [Relation(nm, tabs[nm].global_rows, prog, ["A", "C", "D"], tabs[nm]) for nm in "RST"]
    dec = {d.name: d for d in evaluate_and_push_down(rels, 1_000, 1.0)}
    assert dec["R"].role == "probe"
    for nm, X in (("S", S), ("T", T)):
        host = [c.numpy() for c in X.columns]
        want_c, want_ids, _ = oracle.pushdown(host, X.types, encode(pred, X.types), proj=[0, 2, 3])
        assert dec[nm].count == want_c == X.n_rows * 167 // 1000 and dec[nm].pushed
        np.testing.assert_array_equal(dec[nm].result.rowids.cpu().numpy().view(np.uint32), want_ids)
    dec0 = {d.name: d for d in evaluate_and_push_down(rels, 1_000, 0.0)}
    assert not dec0["S"].pushed and not dec0["T"].pushed and dec0["S"].count == dec["S"].count
    ctx.close()
