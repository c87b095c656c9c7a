import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle, paper_1806_08384_b200 as sel
from selgen.program import *
from selgen import configs
dev = torch.device('cuda:0'); ctx = sel.Context(dev)
n = 60000
T = configs.gen_c2(n)
cols = [c.numpy() for c in T.columns]
t = sel.Table(ctx, list('ABCD'), T.types, [torch.from_numpy(c).to(dev) for c in cols])
for name, node in [('listing', configs.c2_probes()['listing']), ('C in 1,4', In(2, (1, 4))), ('A=2', Cmp('=', 0, 2))]:
    prog = encode(node, T.types)
    for proj in ([], [3], [0], [2], [0, 2, 3]):
        cnt, ids, outs = oracle.pushdown(cols, T.types, prog, proj=proj)
        r = t.pushdown(prog, project=proj, capacity=n)
        ok = r.count == cnt and np.array_equal(r.rowids.cpu().numpy().view(np.uint32), ids)
        for j, c in enumerate(proj):
            ok = ok and np.array_equal(r.columns[c].cpu().numpy().view(outs[j].dtype), outs[j])
        print(f"{name:10s} proj={proj} oracle={cnt} pd={r.count} {'OK' if ok else 'BAD'}")
