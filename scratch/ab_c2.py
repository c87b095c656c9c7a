"""A/B kernel timings on C2 (600M rows) for the probe variants; run with SEL_PREFETCH=0/1."""
import os, sys, time, statistics
sys.path.insert(0, '.')
import torch
import paper_1806_08384_b200 as sel
from selgen import configs, encode

dev = torch.device('cuda:0')
ctx = sel.Context(dev)
ctx.enable_timing(True)
n = int(os.environ.get('ROWS', 600_000_000))
T = configs.gen_c2(n, device=dev)
t = sel.Table(ctx, list('ABCD'), T.types, [c.data for c in T.columns])
prog = encode(configs.c2_probes()['listing'], T.types)
proj = ['A', 'C', 'D']
cnt = t.count(prog)
ids = torch.empty(cnt, dtype=torch.int32, device=dev)
outs = [torch.empty(cnt, dtype=d, device=dev) for d in (torch.int32, torch.uint8, torch.int32)]


def med(f, k=15):
    xs = []
    for i in range(k + 3):
        v = f()
        if i >= 3:
            xs.append(v)
    return statistics.median(xs)


def plain():
    t.count(prog)
    return ctx.last_times()[0]


def keep_mask():
    t.count(prog, keep_selection=True)
    c = ctx.last_times()[0]
    t.pushdown(prog, project=proj, capacity=cnt, out=(ids, outs))
    return c, ctx.last_times()[1]


def keep_vals():
    t.count(prog, keep_selection=True, keep_columns=proj)
    c = ctx.last_times()[0]
    t.pushdown(prog, project=proj, capacity=cnt, out=(ids, outs))
    return c, ctx.last_times()[1]


def single():
    t.count(sel.predicate.compile_predicate(sel.TRUE, t.schema), keep_selection=True)
    t.pushdown(prog, project=proj, capacity=cnt, out=(ids, outs))
    return ctx.last_times()[1]


print('prefetch', os.environ.get('SEL_PREFETCH', 'auto'))
print('plain count        %.3f ms' % med(plain))
km = [keep_mask() for _ in range(12)][3:]
print('keep mask   count  %.3f  pushdown %.3f' % (statistics.median(x[0] for x in km), statistics.median(x[1] for x in km)))
kv = [keep_vals() for _ in range(12)][3:]
print('keep values count  %.3f  pushdown %.3f' % (statistics.median(x[0] for x in kv), statistics.median(x[1] for x in kv)))
print('single pass        %.3f' % med(single, 6))
