#!/usr/bin/env python3
"""BASELINE config C2: allreduce message-size sweep (4 KiB .. 1 GiB) x colors
{1, 2, 4, 8} on N B200s, our multicolor kernel vs NCCL on the same buffers.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench_sweep.py [--max-mb 1024]

Every configuration is checked before it is timed (the reference's rule,
src/bench.py:258-268: the deterministic fill has a closed-form float64 sum,
max rel err <= 1e-5). Scenario "allreduce": device time per call -- G
back-to-back calls captured in one CUDA graph (ours and NCCL alike), CUDA
events around each of R replays, median / G, max over ranks. Scenario
"allreduce_eager": host-launched calls (fill, event, call, event), which add
each library's launch path (Python + ctypes / torch.distributed). Bus
bandwidth = 2 * bytes * (N-1)/N / t (src/bench.py:116-119).
Unconstructible (N, k, arity) triples are skipped like src/bench.py:224-232.

Every row names its DATA MOVEMENT (all of them produce the reference's bits):
  tree_k{k}_a{a}    the reference's schedule: reduce up + broadcast down each
                    color's own tree (route pinned to the pipelined tree kernel,
                    md_plan_set_route(MD_ROUTE_TREE)) -- the row whose speed
                    depends on k and the tree shapes;
  owner_k{k}_a{a}   owner-computes schedule on the same kernel (N >= 4, k < N;
                    md_plan_set_schedule): every element still folds in its
                    color's tree order;
  push              owner-push kernel (sizes from 1 MiB; independent of k: it
                    evaluates each element's color program, so one row, k = max);
  auto_k{k}_a{a}    what a caller gets by default (route picked by size);
                    the "route" column says which kernel md_allreduce ran
                    (md_last_route: ll / oneshot / tree / push);
  nccl_allreduce    NCCL 2.28 (torch.distributed) on the same buffer;
  cpu_port_k{k}     the reference algorithm on the host (the oracle's threaded
                    C port of the tree fold + broadcast, all host cores), sizes
                    up to --cpu-max-mb; `cores` column.
Writes the reference's CSV schema plus route/cores columns to
profiles/sweep_n{N}.csv and prints one JSON line per row.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

C1_BYTES = 25_600_000 * 4  # BASELINE config C1: 25.6M floats
CSV_HEADER = ("scenario,algorithm,n_ranks,payload_bytes,median_time_s,throughput_GBps,backend,"
              "route,cores")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-mb", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seg", type=int, default=0, help="segment_elems (0 = library default)")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--graph-calls", type=int, default=20, help="calls per captured graph")
    ap.add_argument("--eager", action="store_true", help="also host-launched (eager) rows")
    ap.add_argument("--cpu-max-mb", type=int, default=128,
                    help="largest payload of the CPU rows (0 = none)")
    ap.add_argument("--cpu-seconds", type=float, default=3.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_1711_00705_b200 import _lib
    from paper_1711_00705_b200.collectives import DEFAULT_SEGMENT_ELEMS, GradientBuffer, allreduce
    from paper_1711_00705_b200.errors import DisjointnessViolation, InvalidConfig
    from paper_1711_00705_b200.topology import build_multicolor_trees
    from paper_1711_00705_b200.transport import init_from_env

    ep = init_from_env()
    N, rank, dev = ep.n_ranks, ep.rank, ep.torch_device
    nccl = None
    if N > 1 and not a.no_nccl:
        nccl = dist.new_group(backend="nccl")
    lib = _lib.load()
    seg = a.seg or DEFAULT_SEGMENT_ELEMS
    sizes = [4 << 10]
    while sizes[-1] * 4 <= a.max_mb << 20:
        sizes.append(sizes[-1] * 4)
    if C1_BYTES <= a.max_mb << 20:  # the ResNet-50 gradient itself (C1 / C3 size)
        sizes = sorted(set(sizes + [C1_BYTES]))
    max_elems = max(sizes) // 4
    buf = GradientBuffer.alloc(max_elems, ep)  # one registered buffer, views per size
    plans = []
    for k in (1, 2, 4, 8):
        for arity in ((7,) if k == 8 else (4,)):
            try:
                plans.append((k, arity, build_multicolor_trees(N, k, arity) if N > 1 else None))
            except (InvalidConfig, DisjointnessViolation) as e:
                if rank == 0:
                    print(json.dumps({"skip": f"k={k} arity={arity} at N={N}: {e}"}), flush=True)
    rows = []
    stream = ep.stream
    total = sum((r + 1) * np.pi / N for r in range(N))

    def fill(n):
        _lib.check(lib.md_fill_rank_input(buf.data.data_ptr(), n, rank, N,
                                          _lib.stream_ptr(stream)))

    def timed(fn, n):
        """Host-launched calls: fill, event, call, event (includes the
        launch path of every call -- Python, ctypes / torch.distributed)."""
        ts = []
        for i in range(a.warmup + a.reps):
            fill(n)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(n)
            e1.record(stream)
            if i >= a.warmup:
                ts.append((e0, e1))
        torch.cuda.synchronize(dev)
        ep.take_error()
        med = statistics.median(e0.elapsed_time(e1) for e0, e1 in ts) / 1e3
        return max(ep.all_gather(med))

    def timed_graph(fn, n):
        """Device time per call: G back-to-back calls captured as ONE CUDA
        graph, replayed R times; events around each replay, median / G, max
        over ranks. (None if the call cannot be captured.)"""
        G = a.graph_calls
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
                for _ in range(G):
                    fn(n)
        except Exception as e:  # noqa: BLE001
            if rank == 0:
                print(json.dumps({"graph_capture_failed": repr(e)[:200]}), flush=True)
            ep.barrier()
            return None
        ep.barrier()
        g.replay()
        torch.cuda.synchronize(dev)
        ts = []
        for _ in range(a.reps):
            ep.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ts.append(e0.elapsed_time(e1) / G)
        ep.take_error()
        del g
        return max(ep.all_gather(statistics.median(ts) / 1e3))

    def check(n, name):
        idx = np.arange(0, n, max(1, n // 4096))
        got = buf.data[:n][torch.from_numpy(idx).to(dev)].cpu().numpy().astype(np.float64)
        want = (idx.astype(np.float64) % 997.0 + 1.0) * total
        rel = float(np.max(np.abs(got - want) / want)) if n else 0.0
        bad = max(ep.all_gather(rel))
        if bad > 1e-5:
            raise SystemExit(f"{name} n={n}: result check failed (max rel {bad:.3g})")

    def measure(label, fn, n, size):
        fill(n)
        fn(n)
        torch.cuda.synchronize(dev)
        ep.take_error()
        check(n, label)
        route = _lib.last_route(ep.device)
        rname = route[0] + ("_sharded" if route[2] else "")
        t = timed_graph(fn, n)
        if t is not None:
            rows.append(("allreduce", label, N, size, t, "b200", rname, ""))
        if a.eager:
            t = timed(fn, n)
            rows.append(("allreduce_eager", label, N, size, t, "b200", rname, ""))

    with torch.cuda.stream(stream):
        for size in sizes:
            n = size // 4
            view = GradientBuffer(buf.data[:n], peers=buf.peers)
            for k, arity, ts in plans:
                def call(n, ts=ts, view=view, **kw):
                    allreduce(ep, view, "multicolor", tree_set=ts, segment_elems=seg, check=False,
                              **kw)

                if N > 1:
                    measure(f"tree_k{k}_a{arity}", lambda n, c=call: c(n, route="tree"), n, size)
                if N >= 4 and k < N and size > (1 << 20):
                    measure(f"owner_k{k}_a{arity}",
                            lambda n, c=call: c(n, route="tree", schedule="owner"), n, size)
                measure(f"auto_k{k}_a{arity}", call, n, size)
            if N > 1 and size >= (1 << 20) and plans:
                k, arity, ts = plans[-1]
                measure("push", lambda n, ts=ts, view=view: allreduce(
                    ep, view, "multicolor", tree_set=ts, check=False, route="push"), n, size)
            if nccl is not None:
                def ref(n):
                    dist.all_reduce(buf.data[:n], group=nccl)

                fill(n)
                ref(n)
                torch.cuda.synchronize(dev)
                check(n, "nccl")
                t = timed_graph(ref, n)
                if t is not None:
                    rows.append(("allreduce", "nccl_allreduce", N, size, t, "nccl", "nccl", ""))
                if a.eager:
                    t = timed(ref, n)
                    rows.append(("allreduce_eager", "nccl_allreduce", N, size, t, "nccl", "nccl",
                                 ""))

    # the reference algorithm on the host CPU (rank 0; after the GPU rows)
    if rank == 0 and a.cpu_max_mb > 0 and N > 1:
        rows.extend(cpu_rows(N, [x for x in sizes if x <= a.cpu_max_mb << 20 or x == C1_BYTES],
                             plans, a.cpu_seconds))
    ep.barrier()

    if rank == 0:
        out = Path(a.out) if a.out else ROOT / "profiles" / f"sweep_n{N}.csv"
        out.parent.mkdir(exist_ok=True)
        lines = [CSV_HEADER]
        for sc, algo, n_r, size, t, be, route, cores in rows:
            bus = 2 * size * (n_r - 1) / n_r / t / 1e9 if n_r > 1 else 0.0
            lines.append(f"{sc},{algo},{n_r},{size},{t!r},{bus!r},{be},{route},{cores}")
            print(json.dumps({"scenario": sc, "algorithm": algo, "n": n_r, "bytes": size,
                              "us": t * 1e6, "bus_GBps": bus, "backend": be, "route": route,
                              "cores": cores}), flush=True)
        out.write_text("\n".join(lines) + "\n")
    ep.barrier()
    if dist.is_initialized():
        dist.destroy_process_group()


def cpu_rows(N, sizes, plans, seconds):
    """The reference's CPU allreduce (tree fold + broadcast per color) for N
    ranks on this host: the oracle's threaded C port (oracle/mdoracle.c
    mo_allreduce_threads), all host cores, bounded to ~`seconds` per row."""
    import time

    from oracle import oracle as O

    cores = len(os.sched_getaffinity(0))
    out = []
    for k, arity, _ in plans:
        tables = O.tables_from_trees(N, O.trees(N, k, arity))
        for size in sizes:
            n = size // 4
            bufs = [O.fill_rank_input(n, r, N) for r in range(N)]
            O.allreduce_threads(tables, bufs, threads=cores)  # warm
            t0, reps = time.perf_counter(), 0
            while reps < 3 or time.perf_counter() - t0 < seconds:
                O.allreduce_threads(tables, bufs, threads=cores)
                reps += 1
                if reps >= 1000:
                    break
            t = (time.perf_counter() - t0) / reps
            out.append(("allreduce", f"cpu_port_k{k}_a{arity}", N, size, t, "cpu", "host",
                        str(cores)))
    return out


if __name__ == "__main__":
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    main()
