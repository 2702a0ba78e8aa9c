#!/usr/bin/env python3
"""Pinned host -> device copy of the 102.4 MB gradient, as 1 copy or split
into K chunks on K streams (do several copy engines beat one?). One GPU."""
import json

import torch

n = 102_400_008
host = torch.empty(n, dtype=torch.uint8).pin_memory()
host.fill_(1)
dev = torch.device("cuda", 0)
d = torch.empty(n, dtype=torch.uint8, device=dev)
out = {}
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream(device=dev) for _ in range(k)]
    per = (n + k - 1) // k

    def once():
        for i, s in enumerate(streams):
            s.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s):
                d[i * per:(i + 1) * per].copy_(host[i * per:(i + 1) * per], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream(dev).wait_stream(s)

    for _ in range(3):
        once()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        once()
    e1.record()
    torch.cuda.synchronize(dev)
    out[f"k{k}_GBps"] = round(20 * n / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)
print(json.dumps(out))
