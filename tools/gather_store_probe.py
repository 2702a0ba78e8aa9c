#!/usr/bin/env python3
"""Bulk gather (8,192 random records) from a freshly generated shard vs the
same shard after a local shuffle (N = 1): does the record placement matter?"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1711_00705_b200 import dimd, run_ranks  # noqa: E402
from paper_1711_00705_b200.dimd import BatchRequest, BatchSlots, random_batch_device  # noqa: E402

REC = 224 * 224 * 3


def timed(store, slots, reps=5):
    random_batch_device(store, BatchRequest(8192, 1), REC, slots)
    dimd._gather_fixed(store, slots, 8192, REC)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dimd._gather_fixed(store, slots, 8192, REC)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"ms": ms, "GBps": 2 * 8192 * REC / (ms / 1e3) / 1e9}


def prog(ep):
    out = {}
    with torch.cuda.stream(ep.stream):
        st = dimd.synth_store(160_000, REC, 0, 1, 7, 0, 1, 0, device=ep.torch_device)
        slots = BatchSlots(8192, REC, ep.torch_device)
        out["fresh"] = timed(st, slots)
        st2 = dimd.shuffle_all(ep, st, seed=3)
        del st
        out["shuffled"] = timed(st2, slots)
        out["shuffled_again"] = timed(st2, slots)
    return out


print(json.dumps(run_ranks(1, "cuda", prog).results[0]))
