#!/usr/bin/env python3
"""Concurrent pinned host -> device bandwidth on every rank of one box, with the
pinned buffer placed (a) wherever the process happened to run and (b) on the
GPU's own NUMA node (CPU affinity set to the GPU's local_cpulist before the
cudaHostAlloc, so first-touch lands the pages there).

    torchrun --nproc-per-node N tools/h2d_numa_probe.py
"""
import json
import os

import torch
import torch.distributed as dist

N_BYTES = 102_400_008


def gpu_sysfs(dev: int) -> str:
    p = torch.cuda.get_device_properties(dev)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    return f"/sys/bus/pci/devices/{bus}"


def read(path: str) -> str:
    try:
        with open(path) as f:
            return f.read().strip()
    except OSError as e:
        return f"? ({e.__class__.__name__})"


def parse_cpulist(s: str) -> set[int]:
    out: set[int] = set()
    for part in s.split(","):
        if "-" in part:
            lo, hi = part.split("-")
            out.update(range(int(lo), int(hi) + 1))
        elif part:
            out.add(int(part))
    return out


def measure(dev: torch.device, host: torch.Tensor, d: torch.Tensor, k: int = 4) -> float:
    streams = [torch.cuda.Stream(device=dev) for _ in range(k)]
    per = (host.numel() + k - 1) // k

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
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        once()
    e1.record()
    torch.cuda.synchronize(dev)
    return round(20 * host.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)


def main() -> None:
    dist.init_process_group("gloo")
    rank, n = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sysfs = gpu_sysfs(local)
    info = {"rank": rank, "sysfs": sysfs, "numa_node": read(sysfs + "/numa_node"),
            "local_cpulist": read(sysfs + "/local_cpulist"),
            "affinity_before": len(os.sched_getaffinity(0))}
    d = torch.empty(N_BYTES, dtype=torch.uint8, device=dev)
    host = torch.empty(N_BYTES, dtype=torch.uint8).pin_memory()
    host.fill_(1)
    info["default_GBps"] = measure(dev, host, d)
    del host
    cpus = parse_cpulist(info["local_cpulist"]) if not info["local_cpulist"].startswith("?") else set()
    if cpus:
        os.sched_setaffinity(0, cpus)
        host = torch.empty(N_BYTES, dtype=torch.uint8).pin_memory()
        host.fill_(1)
        info["numa_local_GBps"] = measure(dev, host, d)
        # the same buffer, copied by a process running on the other node(s)
        del host
    rows = [None] * n
    dist.all_gather_object(rows, info)
    if rank == 0:
        print(json.dumps({"n": n, "nodes": read("/sys/devices/system/node/online"),
                          "rows": rows}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
