#!/usr/bin/env python3
"""Where does the fixed-size gather lose HBM bandwidth? Times md_gather of
8192 x 150528 B records for several pick patterns / shard sizes, both gather
kernels (TMA ring vs LDG), against a contiguous torch copy of the same bytes."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1711_00705_b200 import dimd  # noqa: E402

REC, B = 224 * 224 * 3, 8192
dev = torch.device("cuda", 0)
store = dimd.synth_store(160_000, REC, 0, 1, 5, 0, 1, 0, device=dev)
slots = dimd.BatchSlots(B, REC, dev)


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return round(ms, 4), round(2 * B * REC / ms / 1e6, 1)


res = {}
src = store.blob[: B * REC]
res["torch_copy"] = t(lambda: slots.records.view(-1).copy_(src))
g = torch.Generator(device="cpu").manual_seed(1)
pats = {
    "seq": torch.arange(B),
    "rand_in_1.2GB": torch.randint(0, B, (B,), generator=g),
    "rand_in_24GB": torch.randint(0, 160_000, (B,), generator=g),
    "strided_19": (torch.arange(B) * 19) % 160_000,
}
for kern in ("tma", "ldg"):
    if kern == "tma":
        os.environ["MD_GATHER_TMA"] = "1"
    for name, p in pats.items():
        slots.picks.copy_(p.to(dev))
        res[f"{kern}_{name}"] = t(lambda: dimd._gather_fixed(store, slots, B, REC))
    os.environ.pop("MD_GATHER_TMA", None)
print(json.dumps({"ms, GB/s (read+write)": res}))
