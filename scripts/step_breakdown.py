"""Kernels of one Execute at a given size (for an ncu launch list: run under
`ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.max`):
C2-shaped table, 5 warm executes then 5 measured ones (plain sel_execute, no graph)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08384_b200 as sel  # noqa: E402
from selgen import configs, encode  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 75_000_000
dev = torch.device("cuda:0")
ctx = sel.Context(dev)
T = configs.gen_c2(n, device=dev)
t = sel.Table(ctx, ["A", "B", "C", "D"], T.types, [c.data for c in T.columns])
prog = encode(configs.c2_probes()["listing"], T.types)
for _ in range(10):
    t.execute(prog, project=["A", "C", "D"], max_size=n)
torch.cuda.synchronize()
print("ok")
