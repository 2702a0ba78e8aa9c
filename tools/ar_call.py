#!/usr/bin/env python3
"""A few allreduce calls on the default route, for profilers (ncu on one rank
of a torchrun job: tools/ncu_rank0.sh) -- eager launches, no CUDA graph.

    torchrun --nproc-per-node N tools/ar_call.py [--mb 102.4] [--update none|replicated|sharded]

Prints per-call CUDA-event times (rank 0) and the route md_allreduce took.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1711_00705_b200 import GradientBuffer, _lib  # noqa: E402
from paper_1711_00705_b200.collectives import SgdUpdate, allreduce  # noqa: E402
from paper_1711_00705_b200.sgd import comm_plan  # noqa: E402
from paper_1711_00705_b200.transport import init_from_env  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=25_600_002)
    ap.add_argument("--update", choices=["none", "replicated", "sharded"], default="replicated")
    ap.add_argument("--calls", type=int, default=6)
    ap.add_argument("--route", default="auto")
    a = ap.parse_args()
    ep = init_from_env()
    N, rank, dev = ep.n_ranks, ep.rank, ep.torch_device
    lib = _lib.load()
    ts, _ = comm_plan(N, "multicolor")
    n = a.elems
    P = n - 2 if a.update != "none" else 0
    sptr = _lib.stream_ptr(ep.stream)
    with torch.cuda.stream(ep.stream):
        buf = GradientBuffer.alloc(n, ep)
        upd = None
        if a.update != "none":
            w, _ = ep.alloc(P)
            m = torch.zeros(P, device=dev)
            upd = SgdUpdate(weights=w, c=1e-4, momentum=m, mu=0.9, wd_b=3.2e-3, update_len=P,
                            sharded=a.update == "sharded")
        ts_ms = []
        for _ in range(a.calls):
            _lib.check(lib.md_fill_rank_input(buf.data.data_ptr(), n, rank, N, sptr))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ep.stream)
            allreduce(ep, buf, "multicolor", tree_set=ts, update=upd, check=False, route=a.route)
            e1.record(ep.stream)
            ts_ms.append((e0, e1))
        ep.synchronize()
    route = _lib.last_route(ep.device)
    times = [round(e0.elapsed_time(e1) * 1e3, 1) for e0, e1 in ts_ms]
    rows = ep.all_gather({"rank": rank, "us": times, "route": route})
    if rank == 0:
        bus = [2 * n * 4 * (N - 1) / N / (max(r["us"][i] for r in rows) * 1e-6) / 1e9
               for i in range(a.calls)]
        print(json.dumps({"n": N, "elems": n, "update": a.update, "route": route,
                          "us_max_over_ranks": [max(r["us"][i] for r in rows)
                                                for i in range(a.calls)],
                          "bus_gbps": [round(b, 1) for b in bus], "rows": rows}), flush=True)
    np.zeros(1)


if __name__ == "__main__":
    main()
