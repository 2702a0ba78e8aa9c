"""run_ranks: execute one program per rank (transport/runner.py:29-80 of the
reference) on the "cuda" backend, plus the torchrun entry for one process
per GPU.

In-process ("cuda"): one host thread per rank -- like the reference's
``threads`` backend and the paper's one host thread per GPU -- each driving
its own GPU when the box has at least ``n_ranks`` GPUs, else every rank is
emulated on GPU 0 (collectives launch once for all ranks).
"""

from __future__ import annotations

import os
import threading
import time
from dataclasses import dataclass

import torch

from paper_1711_00705_b200.errors import Closed, InvalidConfig
from paper_1711_00705_b200.transport.channel import Board, Rendezvous, ThreadChannel, TorchChannel
from paper_1711_00705_b200.transport.endpoint import (
    DEFAULT_MAX_SEGMENT,
    DEFAULT_PULL_TIMEOUT,
    CudaEndpoint,
)

BACKENDS = ("cuda", "torchrun")


@dataclass(frozen=True)
class RunResult:
    """Per-rank return values plus wall time (virtual_time is always None:
    there is no simulated clock on real hardware)."""

    results: list
    virtual_time: float | None
    wall_time: float


def plan_devices(n_ranks: int, emulate: bool | None = None) -> tuple[str, list[int]]:
    n_dev = torch.cuda.device_count()
    if n_dev == 0:
        raise InvalidConfig("the cuda backend needs a GPU (no CPU fallback)")
    if emulate is None:
        emulate = n_dev < n_ranks or n_ranks == 1
    if emulate:
        return "emulated", [0] * n_ranks
    return "p2p", list(range(n_ranks))


def run_ranks(
    n_ranks: int,
    backend: str,
    program,
    *,
    max_segment: int = DEFAULT_MAX_SEGMENT,
    pull_timeout: float = DEFAULT_PULL_TIMEOUT,
    emulate: bool | None = None,
    **unused,
) -> RunResult:
    """Run ``program(endpoint)`` once per rank and collect the results.

    ``"cuda"``: one host thread per rank in this process (one GPU per rank,
    or all ranks emulated on one GPU). ``"torchrun"``: this process is one
    rank of a job torchrun launched (one process per GPU, ``init_from_env``);
    it runs its own rank and every process gets every rank's result.
    The reference's ``network``/``rendezvous``/``inflight_budget`` knobs
    belong to its simulated and TCP transports and have no meaning here.
    """
    if backend not in BACKENDS:
        raise InvalidConfig(f"unknown backend {backend!r}, expected one of {BACKENDS}")
    if n_ranks < 1:
        raise InvalidConfig(f"need at least 1 rank, got {n_ranks}")
    for k, v in unused.items():
        if v is not None:
            raise InvalidConfig(f"{k} is not supported by the cuda backend")
    if backend == "torchrun":
        return _run_this_process(n_ranks, program, pull_timeout)
    mode, devices = plan_devices(n_ranks, emulate)
    board = Board(n_ranks)
    rdv = Rendezvous(n_ranks) if mode == "emulated" else None
    shared_stream = torch.cuda.Stream(device=devices[0]) if mode == "emulated" else None
    results: list = [None] * n_ranks
    errs: list = [None] * n_ranks
    eps: list = [None] * n_ranks

    def main(rank: int) -> None:
        torch.cuda.set_device(devices[rank])
        try:
            ep = CudaEndpoint(
                rank,
                n_ranks,
                devices[rank],
                ThreadChannel(board, rank),
                mode=mode,
                rendezvous=rdv,
                stream=shared_stream,
                max_segment=max_segment,
                pull_timeout=pull_timeout,
            )
            eps[rank] = ep
            with torch.cuda.stream(ep.stream):
                results[rank] = program(ep)
            ep.synchronize()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errs[rank] = e
            board.abort(e)
            if rdv is not None:
                rdv.abort(e)

    t0 = time.perf_counter()
    threads = [threading.Thread(target=main, args=(r,), daemon=True) for r in range(n_ranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    wall = time.perf_counter() - t0
    for ep in eps:
        if ep is not None:
            try:
                ep.close()
            except Exception:  # noqa: BLE001 - teardown after a failure
                pass
    primary = [e for e in errs if e is not None and not isinstance(e, Closed)]
    if primary:
        raise primary[0]
    if any(e is not None for e in errs):
        raise next(e for e in errs if e is not None)
    return RunResult(results, None, wall)


def _run_this_process(n_ranks: int, program, pull_timeout: float) -> RunResult:
    ep = init_from_env(pull_timeout)
    if ep.n_ranks != n_ranks:
        ep.close()
        raise InvalidConfig(f"torchrun launched {ep.n_ranks} processes, the job needs {n_ranks}")
    t0 = time.perf_counter()
    try:
        with torch.cuda.stream(ep.stream):
            res = program(ep)
        ep.synchronize()
        results = ep.all_gather(res)
    finally:
        ep.close()
    return RunResult(results, None, time.perf_counter() - t0)


def gpu_numa_node(device: int) -> int:
    """NUMA node of a GPU's PCIe attachment (sysfs), -1 if unknown."""
    try:
        props = torch.cuda.get_device_properties(device)
        bdf = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/numa_node") as f:
            return int(f.read().strip())
    except (OSError, ValueError, AttributeError):
        return -1


def _cpulist(text: str) -> set[int]:
    cpus: set[int] = set()
    for part in text.strip().split(","):
        if "-" in part:
            lo, hi = part.split("-")
            cpus.update(range(int(lo), int(hi) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


def bind_numa_local(device: int) -> int | None:
    """Pin this process to the CPUs of its GPU's NUMA node, so pinned host
    buffers it allocates afterwards (first touch) sit next to the GPU's PCIe
    root. Returns the node, or None when unknown / not permitted."""
    node = gpu_numa_node(device)
    if node < 0:
        return None
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            cpus = _cpulist(f.read()) & os.sched_getaffinity(0)
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
    except OSError:
        return None
    return node


def init_from_env(pull_timeout: float = DEFAULT_PULL_TIMEOUT) -> CudaEndpoint:
    """Endpoint for one process per GPU launched by torchrun (RANK, WORLD_SIZE,
    LOCAL_RANK, MASTER_ADDR/PORT in the environment). Peers are mapped with
    CUDA IPC; host metadata rides a gloo group."""
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("gloo", rank=rank, world_size=world)
    channel = TorchChannel() if world > 1 else _SoloChannel()
    return CudaEndpoint(
        rank, world, local, channel, mode="p2p", multiprocess=world > 1, pull_timeout=pull_timeout
    )


class _SoloChannel:
    rank = 0
    n_ranks = 1

    def all_gather(self, obj) -> list:
        return [obj]

    def barrier(self) -> None:
        return None
