#!/usr/bin/env python3
"""Diagnostics for the fused allreduce under torchrun: per-variant CUDA-event
times (per rank), to separate kernel cost from inter-rank skew.

    torchrun --nproc-per-node N tools/diag_ar.py
"""

from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch

    from paper_1711_00705_b200 import _lib
    from paper_1711_00705_b200.collectives import GradientBuffer, SgdUpdate, allreduce
    from paper_1711_00705_b200.sgd import comm_plan
    from paper_1711_00705_b200.transport import init_from_env

    ep = init_from_env()
    N, rank, dev = ep.n_ranks, ep.rank, ep.torch_device
    lib = _lib.load()
    P = 25_600_000
    ts, _ = comm_plan(N, "multicolor")
    grad = GradientBuffer.alloc(P + 2, ep)
    w = torch.zeros(P, device=dev)
    v = torch.zeros(P, device=dev)
    s = ep.stream
    sp = _lib.stream_ptr(s)

    def fill():
        lib.md_fill_rank_input(grad.data.data_ptr(), P + 2, rank, N, sp)

    variants = {
        "ar_plain": dict(),
        "ar_sgd": dict(update=SgdUpdate(weights=w, c=1e-4, update_len=P)),
        "ar_sgd_mom_wd": dict(update=SgdUpdate(weights=w, c=1e-4, momentum=v, mu=0.9,
                                               wd_b=0.0032, update_len=P)),
    }
    out = {}
    import os

    lags = [x for x in os.environ.get("DIAG_LAGS", "default").split(",")]
    with torch.cuda.stream(s):
        for name, kw in variants.items():
            modes = [("free", g) for g in lags] + [("sync", "default")]
            if os.environ.get("DIAG_NOSYNC"):
                modes = modes[:-1]
            for mode, lag in modes:
                if lag == "default":
                    os.environ.pop("MD_AR_LAG", None)
                else:
                    os.environ["MD_AR_LAG"] = lag
                mode = f"{mode}/lag{lag}"
                for seg in [int(x) for x in os.environ.get("DIAG_SEGS", "16384,65536,262144").split(",")]:
                    times = []
                    for i in range(12):
                        fill()
                        if mode == "sync":
                            torch.cuda.synchronize(dev)
                            ep.barrier()
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(s)
                        allreduce(ep, grad, "multicolor", tree_set=ts, segment_elems=seg,
                                  check=False, **kw)
                        e1.record(s)
                        times.append((e0, e1))
                    torch.cuda.synchronize(dev)
                    ep.take_error()
                    ms = [a.elapsed_time(b) for a, b in times[2:]]
                    out[f"{name}/{mode}/seg{seg}"] = (statistics.median(ms), min(ms), max(ms))
        # bench-like steps: gather + fill + fused allreduce (mom+wd)
        from paper_1711_00705_b200 import dimd
        from paper_1711_00705_b200.dimd import BatchRequest, BatchSlots, random_batch_device

        upd = variants["ar_sgd_mom_wd"]["update"]
        slots = BatchSlots(32, 150528, dev)
        for shard in (() if os.environ.get("DIAG_NOSTEP") else (2000, 160000)):
            store = dimd.synth_store(shard, 150528, rank, N, 1, 0, N, rank, device=dev)
            for clocks in (False, True):
                sampler = None
                if clocks and rank == 0:
                    sys.path.insert(0, str(ROOT))
                    from bench import Clocks

                    sampler = Clocks([0, 1])
                    sampler.start()
                steps, ars = [], []
                torch.cuda.synchronize(dev)
                ep.barrier()
                for i in range(12):
                    a0 = torch.cuda.Event(enable_timing=True)
                    a0.record(s)
                    random_batch_device(store, BatchRequest(32, 1000 + i), 150528, slots)
                    fill()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    allreduce(ep, grad, "multicolor", tree_set=ts, check=False, update=upd)
                    e1.record(s)
                    steps.append((a0, e1))
                    ars.append((e0, e1))
                torch.cuda.synchronize(dev)
                if sampler:
                    sampler.stop()
                st = [a.elapsed_time(b) for a, b in steps[2:]]
                ar = [a.elapsed_time(b) for a, b in ars[2:]]
                out[f"bench_step/shard{shard}/clocks{int(clocks)}"] = (
                    statistics.median(st), statistics.median(ar), max(ar))
            del store
    rows = ep.all_gather(out)
    if rank == 0:
        for key in rows[0]:
            print(json.dumps({"variant": key,
                              "per_rank_median_min_max_ms": [r[key] for r in rows]}))


if __name__ == "__main__":
    main()
