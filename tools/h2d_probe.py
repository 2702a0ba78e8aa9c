#!/usr/bin/env python3
"""Concurrent pinned-host -> device copy bandwidth per rank, with and without
binding the rank to its GPU's NUMA node before the pinned allocation.

    torchrun --nproc-per-node N tools/h2d_probe.py
"""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1711_00705_b200.transport.runner import bind_numa_local, gpu_numa_node  # noqa: E402


def run(tag, dev, nbytes=102_400_008):
    host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    host.fill_(1)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(host, non_blocking=True)
    torch.cuda.synchronize(dev)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        d.copy_(host, non_blocking=True)
    e1.record()
    torch.cuda.synchronize(dev)
    gbs = 20 * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9
    del host, d
    return {tag: round(gbs, 1)}


def main():
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    row = {"rank": rank, "gpu_numa": gpu_numa_node(dev.index), "cpus0": len(os.sched_getaffinity(0))}
    row.update(run("default", dev))
    row["bound_to"] = bind_numa_local(dev.index)
    row["cpus1"] = len(os.sched_getaffinity(0))
    row.update(run("numa_bound", dev))
    rows = [None] * dist.get_world_size()
    dist.all_gather_object(rows, row)
    if rank == 0:
        for r in rows:
            print(json.dumps(r))


if __name__ == "__main__":
    main()
