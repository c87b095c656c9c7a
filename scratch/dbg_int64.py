import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle, paper_1806_08384_b200 as sel
from selgen.program import *
from helpers import random_table
dev = torch.device('cuda:0'); ctx = sel.Context(dev)
for n in [31, 64, 128, 129, 256, 512, 1000, 1023, 1024, 2048]:
    rng = np.random.default_rng(n)
    x = rng.choice(np.array([2**63-1, -5, 7, -11612619170], dtype=np.int64), n)
    prog = encode(In(0, (2**63-1, -11612619170)), [INT64])
    t = sel.Table(ctx, ['x'], [INT64], [torch.from_numpy(x).to(dev)])
    want = oracle.pushdown([x], [INT64], prog)[1]
    got = t.pushdown(prog, capacity=n).rowids.cpu().numpy()
    miss = sorted(set(want) - set(got)); extra = sorted(set(got) - set(want))
    print(n, t.count(prog), len(want), 'miss', miss[:12], 'extra', extra[:12])
    prog2 = encode(Cmp('=', 0, -5), [INT64])
    print('   eq', t.count(prog2), int((x == -5).sum()))
