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
tC = sel.Table(ctx, ['C'], [DICT8], [torch.from_numpy(cols[2]).to(dev)])
tB = sel.Table(ctx, ['B'], [INT32], [torch.from_numpy(cols[1]).to(dev)])
cases = {
 'C in 1,4': (t, In(2, (1, 4))), 'C in 1,4 (C only)': (tC, In(0, (1, 4))),
 'C=1': (t, Cmp('=', 2, 1)), 'C=4': (t, Cmp('=', 2, 4)),
 'B in 5,1500': (t, In(1, (5, 1500))), 'B in 5,1500 (B only)': (tB, In(0, (5, 1500))),
 'B between': (t, Between(1, 1001, 2000)), 'A=2': (t, Cmp('=', 0, 2)),
 'C in 0..3': (t, In(2, (0, 1, 2, 3))), 'B<100 or B>2100': (t, Or(Cmp('<', 1, 100), Cmp('>', 1, 2100))),
 'C in 1,4 or A=7': (t, Or(In(2, (1, 4)), Cmp('=', 0, 7))),
}
for name, (tab, node) in cases.items():
    types = tab.types
    prog = encode(node, types)
    hc = [cols[2]] if tab is tC else ([cols[1]] if tab is tB else cols)
    want = oracle.pushdown(hc, types, prog)[1]
    r = tab.pushdown(prog, capacity=n)
    print(f"{name:24s} path={sel.program_path(prog, types)} oracle={len(want)} count={tab.count(prog)} pd={r.count}")
