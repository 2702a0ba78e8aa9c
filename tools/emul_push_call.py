#!/usr/bin/env python3
"""Sharded C5 calls with N ranks emulated on ONE GPU (one cooperative launch
serves every rank), for an `ncu --set full` capture of the owner-push kernel's
HBM traffic: every "peer" access is then a local HBM access, so DRAM bytes
cover the kernel's whole data movement.

    ncu --set full -k regex:push -s 2 -c 1 python tools/emul_push_call.py [--n 2]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1711_00705_b200 import GradientBuffer, run_ranks  # noqa: E402
from paper_1711_00705_b200.collectives import SgdUpdate, allreduce  # noqa: E402
from paper_1711_00705_b200.sgd import comm_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2)
ap.add_argument("--calls", type=int, default=4)
a = ap.parse_args()
P = 25_600_000


def prog(ep):
    ts, _ = comm_plan(ep.n_ranks, "multicolor")
    buf = GradientBuffer.alloc(P + 2, ep)
    w, _ = ep.alloc(P)
    m = torch.zeros(P, device=ep.torch_device)
    upd = SgdUpdate(weights=w, c=1e-4, momentum=m, mu=0.9, wd_b=3.2e-3, update_len=P, sharded=True)
    for _ in range(a.calls):
        buf.data.fill_(1.0)
        allreduce(ep, buf, "multicolor", tree_set=ts, update=upd)
    return True


print(all(run_ranks(a.n, "cuda", prog, emulate=True).results))
