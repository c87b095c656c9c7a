import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle, paper_1806_08384_b200 as sel
from selgen.program import *
from selgen import configs
dev = torch.device('cuda:0'); ctx = sel.Context(dev)
for n in [6000, 60000, 600000, 6000000]:
    T = configs.gen_c2(n)
    cols = [c.numpy() for c in T.columns]
    t = sel.Table(ctx, list('ABCD'), T.types, [torch.from_numpy(c).to(dev) for c in cols])
    prog = encode(configs.c2_probes()['listing'], T.types)
    want = oracle.pushdown(cols, T.types, prog)[1]
    c = t.count(prog)
    r = t.pushdown(prog, capacity=n)
    got = r.rowids.cpu().numpy().view(np.uint32)
    print(n, 'count', c, 'oracle', len(want), 'pd count', r.count, 'local', r.local_count, 'nids', len(got))
    k = min(len(got), len(want))
    bad = np.flatnonzero(got[:k] != want[:k])
    print('   first bad', bad[:5], got[bad[:3]] if len(bad) else '', want[bad[:3]] if len(bad) else '')
