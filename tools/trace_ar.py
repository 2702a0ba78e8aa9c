#!/usr/bin/env python3
"""Trace one fused allreduce (MD_AR_TRACE=1) on every rank and summarise the
per-CTA timeline: kernel span, producer flag waits, first-chunk latency,
segment processing time and publish latency, grouped by task.

    MD_AR_TRACE=1 torchrun --nproc-per-node N tools/trace_ar.py [--seg 32768] [--plain]

(MD_AR_TRACE is read once per process, so every call of the run is traced.)
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
EV = {1: "WAIT0", 2: "WAIT1", 3: "ISSUED", 4: "FIRST", 5: "DONE", 6: "PUB", 7: "ENTRY", 8: "EXIT",
      9: "START", 10: "LEFT", 11: "X1", 12: "X2"}
DT = np.dtype([("t", "<u8"), ("cta", "<u4"), ("ev", "<u2"), ("seg", "<u2")])


def analyse(path: str, stamps=None) -> dict:
    rec = np.fromfile(path, dtype=DT)
    rec = rec[rec["ev"] != 0]
    t0 = int(rec["t"].min())
    by_cta = defaultdict(list)
    for r in rec:
        by_cta[int(r["cta"])].append((int(r["t"] - t0), EV[int(r["ev"])], int(r["seg"])))
    out = defaultdict(lambda: defaultdict(list))
    spans = []
    for cta, evs in by_cta.items():
        evs.sort()
        d = {(e, s): t for t, e, s in evs}
        task = next((s for t, e, s in evs if e == "ENTRY"), -1)
        entry = d.get(("ENTRY", task), 0)
        exit_ = d.get(("EXIT", task), 0)
        spans.append((entry, exit_))
        segs = sorted({s for t, e, s in evs if e == "WAIT0"})
        g = out[task]
        g["ctas"].append(cta)
        g["span_us"].append((exit_ - entry) / 1e3)
        for s in segs:
            if ("WAIT1", s) in d:
                g["wait_us"].append((d[("WAIT1", s)] - d[("WAIT0", s)]) / 1e3)
            if ("FIRST", s) in d and ("WAIT1", s) in d:
                g["first_us"].append((d[("FIRST", s)] - d[("WAIT1", s)]) / 1e3)
            if ("DONE", s) in d and ("FIRST", s) in d:
                g["proc_us"].append((d[("DONE", s)] - d[("FIRST", s)]) / 1e3)
            if ("PUB", s) in d and ("DONE", s) in d:
                g["pub_us"].append((d[("PUB", s)] - d[("DONE", s)]) / 1e3)
        g["first_wait0_us"].append((d.get(("WAIT0", segs[0]), entry) - entry) / 1e3 if segs else 0)
        g["idle_tail_us"].append(
            (exit_ - max((t for t, e, s in evs if e in ("DONE", "PUB", "ISSUED")), default=exit_)) / 1e3
        )
    # timeline: segments issued per 10 us bin, per task (is ingress busy end to end?)
    k0 = min(s for s, _ in spans)
    kend = max(e for _, e in spans)
    nb = int((kend - k0) // 10_000) + 1
    timeline = {}
    for cta, evs in by_cta.items():
        task = next((s for t, e, s in evs if e == "ENTRY"), -1)
        row = timeline.setdefault(f"task{task}", [0] * nb)
        for t, e, s in evs:
            if e == "ISSUED":  # producer finished issuing a segment's loads
                row[int((t - k0) // 10_000)] += 1
    kev = {e: [t for c in by_cta.values() for t, ee, _ in c if ee == e]
           for e in ("START", "ENTRY", "EXIT", "LEFT", "X1", "X2")}
    t_start = min(kev["START"]) if kev["START"] else k0
    summary = {"start_spread_us": (max(kev["START"]) - t_start) / 1e3 if kev["START"] else None,
               "start_to_first_entry_us": (k0 - t_start) / 1e3,
               "first_exit_to_last_left_us": ((max(kev["LEFT"]) - min(kev["EXIT"])) / 1e3
                                              if kev["LEFT"] else None),
               "last_exit_to_last_left_us": ((max(kev["LEFT"]) - max(kev["EXIT"])) / 1e3
                                             if kev["LEFT"] else None),
               "exit_phases_us": ([(kev["X1"][0] - max(kev["EXIT"])) / 1e3,
                                   (kev["X2"][0] - kev["X1"][0]) / 1e3,
                                   (max(kev["LEFT"]) - kev["X2"][0]) / 1e3] if kev["X2"] else None),
               "start_to_last_left_us": (max(kev["LEFT"]) - t_start) / 1e3 if kev["LEFT"] else None,
               "kernel_us": (max(e for _, e in spans) - min(s for s, _ in spans)) / 1e3,
               # stream stamps just before / after the call: launch latency and drain
               "stamp_to_start_us": (t_start + t0 - stamps[0]) / 1e3 if stamps else None,
               "left_to_stamp_us": ((stamps[1] - max(kev["LEFT"]) - t0) / 1e3
                                    if stamps and kev["LEFT"] else None),
               "stamp_to_stamp_us": (stamps[1] - stamps[0]) / 1e3 if stamps else None,
               "bare_kernel_gap_us": (stamps[2] - stamps[1]) / 1e3 if stamps else None,
               "timeline_10us": timeline,
               "entry_spread_us": (max(s for s, _ in spans) - min(s for s, _ in spans)) / 1e3,
               "first_entry_to_last_exit_us": (max(e for _, e in spans) - min(s for s, _ in spans)) / 1e3}
    for task, g in sorted(out.items()):
        summary[f"task{task}"] = {
            k: (round(float(np.mean(v)), 2), round(float(np.sum(v)), 1), len(v))
            for k, v in g.items() if k != "ctas"
        } | {"n_ctas": len(g["ctas"])}
    return summary


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--seg", type=int, default=0)
    ap.add_argument("--plain", action="store_true")
    ap.add_argument("--elems", type=int, default=25_600_000)
    ap.add_argument("--out", default="gpurun_out")
    a = ap.parse_args()
    import torch

    from paper_1711_00705_b200 import _lib
    from paper_1711_00705_b200.collectives import DEFAULT_SEGMENT_ELEMS, GradientBuffer, SgdUpdate, allreduce
    from paper_1711_00705_b200.sgd import comm_plan
    from paper_1711_00705_b200.transport import init_from_env

    ep = init_from_env()
    N, rank, dev = ep.n_ranks, ep.rank, ep.torch_device
    lib = _lib.load()
    P = a.elems
    ts, _ = comm_plan(N, "multicolor")
    grad = GradientBuffer.alloc(P + 2, ep)
    w = torch.zeros(P, device=dev)
    v = torch.zeros(P, device=dev)
    upd = None if a.plain else SgdUpdate(weights=w, c=1e-4, momentum=v, mu=0.9, wd_b=0.0032, update_len=P)
    seg = a.seg or DEFAULT_SEGMENT_ELEMS
    stamps = torch.zeros(4, dtype=torch.int64, device=dev)
    with torch.cuda.stream(ep.stream):
        for i in range(6):
            lib.md_fill_rank_input(grad.data.data_ptr(), P + 2, rank, N, _lib.stream_ptr(ep.stream))
            if i == 1:  # every later call overwrites the log: the last one is steady state
                torch.cuda.synchronize(dev)
                ep.barrier()
                pass  # MD_AR_TRACE is read once per process: set it before launch
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ep.stream)
            if i == 5:
                lib.md_stamp(stamps[0:].data_ptr(), _lib.stream_ptr(ep.stream))
            allreduce(ep, grad, "multicolor", tree_set=ts, segment_elems=seg, update=upd, check=False)
            if i == 5:
                lib.md_stamp(stamps[1:].data_ptr(), _lib.stream_ptr(ep.stream))
                lib.md_stamp(stamps[2:].data_ptr(), _lib.stream_ptr(ep.stream))  # bare gap
            e1.record(ep.stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
        plain_ms = []
        for _ in range(5):  # untraced calls on the same stream, for comparison
            lib.md_fill_rank_input(grad.data.data_ptr(), P + 2, rank, N, _lib.stream_ptr(ep.stream))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ep.stream)
            allreduce(ep, grad, "multicolor", tree_set=ts, segment_elems=seg, update=upd, check=False)
            e1.record(ep.stream)
            torch.cuda.synchronize(dev)
            plain_ms.append(round(e0.elapsed_time(e1), 4))
    path = f"{a.out}/trace_n{N}_r{rank}.bin"
    _lib.check(lib.md_trace_dump(ep.device, path.encode()))
    summ = analyse(path, [int(x) for x in stamps.cpu()])
    summ["event_ms"] = ms
    summ["untraced_event_ms"] = plain_ms
    rows = ep.all_gather(summ)
    if rank == 0:
        for r, s in enumerate(rows):
            print(json.dumps({"rank": r, **s}))


if __name__ == "__main__":
    main()
