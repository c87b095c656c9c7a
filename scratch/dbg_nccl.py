import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1806_08384_b200 as sel
from selgen.program import *
from selgen import configs
def say(*a): print(*a, flush=True)
dev = torch.device('cuda:0')
c = sel.Context(dev); say('ctx')
uid = sel.Context.new_unique_id(); say('uid', len(uid))
c.set_comm(1, 0, uid); say('comm')
c.enable_timing(True); say('timing')
T = configs.gen_c2(600_000)
t = sel.Table(c, list('ABCD'), T.types, [x.data.to(dev) for x in T.columns]); say('table')
prog = encode(configs.c2_probes()['listing'], T.types)
say('count', t.count(prog)); say('ms', c.last_kernel_ms())
res = t.pushdown(prog, project=[3]); say('pd', res.count, res.offset)
res = t.pushdown(prog); say('pd2', res.count)
t.release(); say('released')
c.close(); say('closed')
