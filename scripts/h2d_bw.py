"""Pinned host -> device copy bandwidth with 1, 2 and 4 streams (the e2e leg of bench.py)."""
import json
import torch

n = 1 << 30   # 1 GiB per buffer
dev = torch.device("cuda:0")
h = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(4)]
d = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(4)]
res = {}
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream(dev) for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(4):
            s = ss[i % ns]
            s.wait_event(a)
            with torch.cuda.stream(s):
                d[i].copy_(h[i], non_blocking=True)
        for s in ss:
            b.wait_stream(s) if hasattr(b, "wait_stream") else None
        torch.cuda.current_stream().wait_stream(ss[0])
        for s in ss[1:]:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        res[f"h2d_{ns}streams_gbs"] = round(4 * n / (a.elapsed_time(b) / 1000) / 1e9, 1)
# D2H
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(4):
    h[i].copy_(d[i], non_blocking=True)
b.record()
torch.cuda.synchronize()
res["d2h_gbs"] = round(4 * n / (a.elapsed_time(b) / 1000) / 1e9, 1)
print(json.dumps(res))
