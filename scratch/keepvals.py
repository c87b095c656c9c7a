import os, sys
sys.path.insert(0, '.')
import torch
import paper_1806_08384_b200 as sel
from selgen import configs, encode
dev = torch.device('cuda:0'); ctx = sel.Context(dev)
T = configs.gen_c2(device=dev)
t = sel.Table(ctx, list('ABCD'), T.types, [c.data for c in T.columns])
prog = encode(configs.c2_probes()['listing'], T.types)
for _ in range(4):
    t.count(prog, keep_selection=True, keep_columns=['A', 'C', 'D'])
torch.cuda.synchronize()
