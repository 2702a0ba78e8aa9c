#!/usr/bin/env python3
"""Where the fixed cost of an owner-push call goes: %globaltimer events of
every CTA (MD_AR_TRACE=1 is read once per process, so set it on the command
line) around one sharded C5 call, plus stream-ordered md_stamp kernels just
before and after it.

    MD_AR_TRACE=1 torchrun --nproc-per-node N tools/trace_push.py [--update sharded|none]

Per rank (us from the stamp before the call): first CTA start, last CTA past
the entry barrier, first tile folded (median over CTAs), last bulk store
issued, last store landed (wait_group 0), the exit barrier's done flags out /
every peer's seen, and the stamp after the call.
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import tempfile
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1711_00705_b200 import GradientBuffer, _lib  # noqa: E402
from paper_1711_00705_b200.collectives import SgdUpdate, allreduce  # noqa: E402
from paper_1711_00705_b200.sgd import comm_plan  # noqa: E402
from paper_1711_00705_b200.transport import init_from_env  # noqa: E402

EV = {1: "WAIT0", 2: "WAIT1", 3: "ISSUED", 4: "FIRST", 5: "DONE", 6: "PUB", 7: "ENTRY",
      8: "EXIT", 9: "START", 10: "LEFT", 11: "X1", 12: "X2", 13: "X3"}
HALF = 512  # kTraceHalf


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=25_600_002)
    ap.add_argument("--update", choices=["sharded", "none"], default="sharded")
    ap.add_argument("--calls", type=int, default=5)
    a = ap.parse_args()
    ep = init_from_env()
    N, rank, dev = ep.n_ranks, ep.rank, ep.torch_device
    lib = _lib.load()
    ts, _ = comm_plan(N, "multicolor")
    n = a.elems
    sptr = _lib.stream_ptr(ep.stream)
    stamps = torch.zeros(2, dtype=torch.int64, device=dev)
    with torch.cuda.stream(ep.stream):
        buf = GradientBuffer.alloc(n, ep)
        upd = None
        if a.update == "sharded":
            w, _ = ep.alloc(n - 2)
            upd = SgdUpdate(weights=w, c=1e-4, momentum=torch.zeros(n - 2, device=dev), mu=0.9,
                            wd_b=3.2e-3, update_len=n - 2, sharded=True)
        for i in range(a.calls):
            _lib.check(lib.md_fill_rank_input(buf.data.data_ptr(), n, rank, N, sptr))
            if i == a.calls - 1:
                _lib.check(lib.md_stamp(stamps[0:].data_ptr(), sptr))
            allreduce(ep, buf, "multicolor", tree_set=ts, update=upd, check=False)
            if i == a.calls - 1:
                _lib.check(lib.md_stamp(stamps[1:].data_ptr(), sptr))
        ep.synchronize()
    route = _lib.last_route(ep.device)
    path = Path(tempfile.mkdtemp()) / f"trace_r{rank}.bin"
    _lib.check(lib.md_trace_dump(ep.device, str(path).encode()))
    rec = np.fromfile(path, dtype=np.dtype([("t", "<u8"), ("cta", "<u4"), ("ev", "<u2"),
                                             ("seg", "<u2")]))
    rec = rec.reshape(-1, 3, HALF)
    t0 = int(stamps[0])
    ev = {}
    for cta in range(rec.shape[0]):
        for role in range(3):
            for e in rec[cta, role]:
                if e["t"]:
                    ev.setdefault(EV.get(int(e["ev"]), str(e["ev"])), []).append(
                        (int(e["t"]) - t0) / 1e3)
    def spread(name):
        x = sorted(ev.get(name, []))
        return [round(x[0], 2), round(statistics.median(x), 2), round(x[-1], 2)] if x else None

    row = {"rank": rank, "route": route,
           "start_min_med_max": spread("START"), "entry_min_med_max": spread("ENTRY"),
           "first_fold_min_med_max": spread("FIRST"), "issued_min_med_max": spread("ISSUED"),
           "stamp_after_us": (int(stamps[1]) - t0) / 1e3,
           "first_start_us": min(ev.get("START", [float("nan")])),
           "last_entry_us": max(ev.get("ENTRY", [float("nan")])),
           "first_tile_folded_median_us": statistics.median(ev["FIRST"]) if "FIRST" in ev else None,
           "last_store_issued_us": max(ev.get("ISSUED", [float("nan")])),
           "last_store_landed_us": max(ev.get("DONE", [float("nan")])),
           "done_flags_out_us": max(ev.get("X2", [float("nan")])),
           "peers_done_seen_us": max(ev.get("X3", [float("nan")]))}
    rows = ep.all_gather(row)
    if rank == 0:
        print(json.dumps({"n": N, "elems": n, "update": a.update, "rows": rows}), flush=True)


if __name__ == "__main__":
    main()
