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
At N >= 4, for k < N and sizes above the LL range, rows "..._owner" time the
owner-computes schedule (same fold order, same bits; md_plan_set_schedule).
Writes the reference's CSV schema to profiles/sweep_n{N}.csv (algorithm
column carries k and arity) and prints one JSON line per row.
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

CSV_HEADER = "scenario,algorithm,n_ranks,payload_bytes,median_time_s,throughput_GBps,backend"


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-mb", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seg", type=int, default=0, help="segment_elems (0 = library default)")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--graph-calls", type=int, default=20, help="calls per captured graph")
    ap.add_argument("--no-eager", action="store_true", help="graph-timed rows only")
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
    max_elems = sizes[-1] // 4
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

    with torch.cuda.stream(stream):
        for size in sizes:
            n = size // 4
            view = GradientBuffer(buf.data[:n], peers=buf.peers)
            for k, arity, ts in plans:
                def ours(n, ts=ts, view=view):
                    allreduce(ep, view, "multicolor", tree_set=ts, segment_elems=seg, check=False)

                fill(n)
                ours(n)
                torch.cuda.synchronize(dev)
                ep.take_error()
                check(n, f"multicolor k={k}")
                t = timed_graph(ours, n)
                if t is not None:
                    rows.append(("allreduce", f"multicolor_k{k}_a{arity}", N, size, t, "b200"))
                if not a.no_eager:
                    t = timed(ours, n)
                    rows.append(("allreduce_eager", f"multicolor_k{k}_a{arity}", N, size, t, "b200"))
                if N >= 4 and k < N and size > (1 << 20):
                    # owner-computes schedule: same fold order (same bits), balanced traffic
                    def owner(n, ts=ts, view=view):
                        allreduce(ep, view, "multicolor", tree_set=ts, segment_elems=seg,
                                  check=False, schedule="owner")

                    fill(n)
                    owner(n)
                    torch.cuda.synchronize(dev)
                    ep.take_error()
                    check(n, f"multicolor k={k} owner")
                    t = timed_graph(owner, n)
                    if t is not None:
                        rows.append(("allreduce", f"multicolor_k{k}_a{arity}_owner", N, size, t,
                                     "b200"))
            if nccl is not None:
                def ref(n):
                    dist.all_reduce(buf.data[:n], group=nccl)

                fill(n)
                ref(n)
                torch.cuda.synchronize(dev)
                check(n, "nccl")
                t = timed_graph(ref, n)
                if t is not None:
                    rows.append(("allreduce", "nccl_allreduce", N, size, t, "nccl"))
                if not a.no_eager:
                    t = timed(ref, n)
                    rows.append(("allreduce_eager", "nccl_allreduce", N, size, t, "nccl"))

    if rank == 0:
        out = Path(a.out) if a.out else ROOT / "profiles" / f"sweep_n{N}.csv"
        out.parent.mkdir(exist_ok=True)
        lines = [CSV_HEADER]
        for sc, algo, n_r, size, t, be in rows:
            bus = 2 * size * (n_r - 1) / n_r / t / 1e9 if n_r > 1 else 0.0
            lines.append(f"{sc},{algo},{n_r},{size},{t!r},{bus!r},{be}")
            print(json.dumps({"scenario": sc, "algorithm": algo, "n": n_r, "bytes": size,
                              "us": t * 1e6,
                              "bus_GBps": bus, "backend": be}), flush=True)
        out.write_text("\n".join(lines) + "\n")
    ep.barrier()
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    main()
