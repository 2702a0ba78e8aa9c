#!/usr/bin/env python3
"""Stress test of the cross-GPU flag protocol on real NVLink: thousands of
graph-replayed fused C5 calls (25.6M + 2 floats, momentum 0.9 + weight decay)
with a random per-rank start skew before every call, every call's weights
checked against the oracle.

    torchrun --nproc-per-node N tools/stress_fused.py [--calls 2000] [--sharded]
    MD_AR_SYS_FENCE=1 torchrun ...    (system-scope release on every flag)

Per call, inside ONE captured CUDA graph of --per-graph calls (replayed until
--calls calls ran): a spin kernel of a random length (0..~40 us, drawn per
rank and call at capture time) skews the ranks' starts; the gradient buffer is
refilled (the reference bench fill, src/bench.py:188-195); the fused allreduce
+ update runs on md_allreduce's default route; then on the device
  * diff[i]  = number of weight words that differ from a shadow copy updated
               by md_sgd_update with the oracle-checked sum g (same math);
  * gdiff[i] = number of differing sum words (own slice when sharded);
  * sum[i]   = sum of the weights' int32 bit patterns (a checksum).
Rank 0's host meanwhile chains the oracle's C update (oracle/mdoracle.c
mo_sgd_update) from the same start and the same oracle-folded g, and the
checksum of every call is compared with it. The first call's g is checked
bit for bit against the oracle fold (oracle/mdoracle.c mo_fold_range).
Prints one JSON line per rank-0 run.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1711_00705_b200 import GradientBuffer, _lib  # noqa: E402
from paper_1711_00705_b200.collectives import SgdUpdate, allreduce  # noqa: E402
from paper_1711_00705_b200.sgd import comm_plan  # noqa: E402
from paper_1711_00705_b200.transport import init_from_env  # noqa: E402

P = 25_600_000
L = P + 2
MU, WD, LR = 0.9, 1e-4, 0.1


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=2000)
    ap.add_argument("--per-graph", type=int, default=100)
    ap.add_argument("--max-skew-us", type=float, default=40.0)
    ap.add_argument("--sharded", action="store_true")
    ap.add_argument("--route", default="auto", help="pin md_allreduce's kernel (tree, stream, ...)")
    a = ap.parse_args()
    ep = init_from_env()
    N, rank, dev = ep.n_ranks, ep.rank, ep.torch_device
    lib = _lib.load()
    ts, _ = comm_plan(N, "multicolor")
    tables = O.tables_from_trees(N, O.trees(N, ts.k, ts.arity))
    B = 32 * N
    c, wd_b = float(np.float32(LR / B)), float(np.float32(WD * B))
    sptr = _lib.stream_ptr(ep.stream)
    rng = np.random.default_rng(1234)
    w0 = (rng.standard_normal(P, dtype=np.float32) * np.float32(0.01)).astype(np.float32)
    # the oracle's sum of the bench fill, every rank's input recomputed here
    g_want = O.fold_c(tables, [O.fill_rank_input(L, r, N) for r in range(N)])

    with torch.cuda.stream(ep.stream):
        w, _ = ep.alloc(P)
        w.copy_(torch.from_numpy(w0))
        m = torch.zeros(P, device=dev)
        w_ref = w.clone()
        m_ref = torch.zeros(P, device=dev)
        grad = GradientBuffer.alloc(L, ep)
        g_ref = torch.from_numpy(g_want).to(dev)
        upd = SgdUpdate(weights=w, c=c, momentum=m, mu=MU, wd_b=wd_b, update_len=P,
                        sharded=a.sharded)
        lo, hi = 0, L
        if a.sharded:  # the sum is defined on the own slice (md_allreduce_ex)
            n4 = L & ~3
            per = ((n4 // 4 + N - 1) // N) * 4
            lo, hi = min(n4, rank * per), min(n4, (rank + 1) * per)
        calls = a.per_graph * max(1, (a.calls + a.per_graph - 1) // a.per_graph)
        diff = torch.zeros(calls, dtype=torch.int64, device=dev)
        gdiff = torch.zeros(calls, dtype=torch.int64, device=dev)
        csum = torch.zeros(calls, dtype=torch.int64, device=dev)
        skew = np.random.default_rng(99 + 7 * rank).uniform(0, a.max_skew_us, a.per_graph)
        cycles = (skew * 1.9e3).astype(np.int64)  # ~1.9 GHz SM clock
        slot = torch.zeros(1, dtype=torch.int64, device=dev)  # device call counter

        def one_call(i_static: int | None):
            if cycles[i_static % a.per_graph] > 0:
                torch.cuda._sleep(int(cycles[i_static % a.per_graph]))
            _lib.check(lib.md_fill_rank_input(grad.data.data_ptr(), L, rank, N, sptr))
            allreduce(ep, grad, "multicolor", tree_set=ts, update=upd, check=False, route=a.route)
            _lib.check(lib.md_sgd_update(w_ref.data_ptr(), g_ref.data_ptr(), m_ref.data_ptr(), P,
                                         c, MU, wd_b, sptr))
            idx = slot
            diff.index_copy_(0, idx, (w.view(torch.int32) != w_ref.view(torch.int32))
                             .sum().reshape(1))
            gdiff.index_copy_(0, idx, (grad.data[lo:hi].view(torch.int32)
                                       != g_ref[lo:hi].view(torch.int32)).sum().reshape(1))
            csum.index_copy_(0, idx, w.view(torch.int32).sum(dtype=torch.int64).reshape(1))
            slot.add_(1)

        # call 0, eager: the sum bit for bit against the oracle fold
        _lib.check(lib.md_fill_rank_input(grad.data.data_ptr(), L, rank, N, sptr))
        allreduce(ep, grad, "multicolor", tree_set=ts, check=True)
        first_ok = bool(torch.equal(grad.data[lo:hi].view(torch.int32),
                                    g_ref[lo:hi].view(torch.int32)))
        route = _lib.last_route(ep.device)
        # one fused call eagerly (warm-up of the update route), shadow in step
        one_call(0)
        ep.synchronize()
        slot.zero_()
        diff.zero_()
        gdiff.zero_()
        csum.zero_()
        w.copy_(torch.from_numpy(w0))
        m.zero_()
        w_ref.copy_(w)
        m_ref.zero_()
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=ep.stream, capture_error_mode="thread_local"):
            for i in range(a.per_graph):
                one_call(i)
        fused_route = _lib.last_route(ep.device)

    # rank 0: the oracle chain on the host, concurrently with the replays
    want_sums = []
    if rank == 0:
        def chain():
            ww, mm = w0.copy(), np.zeros(P, np.float32)
            L_ = O.lib()
            for _ in range(calls):
                L_.mo_sgd_update(O._f32p(ww), O._f32p(g_want), O._f32p(mm), P, c, MU, wd_b)
                want_sums.append(int(ww.view(np.int32).astype(np.int64).sum()))
        th = threading.Thread(target=chain)
        th.start()
    ep.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(calls // a.per_graph):
        graph.replay()
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - t0
    err = None
    try:
        ep.take_error()
    except Exception as e:  # noqa: BLE001
        err = repr(e)
    row = {"rank": rank, "route": fused_route, "first_sum_ok": first_ok, "plain_route": route,
           "calls": calls, "bad_calls_w": int((diff != 0).sum()),
           "bad_calls_g": int((gdiff != 0).sum()), "max_bad_words": int(diff.max()),
           "sums": csum.cpu().tolist(), "wall_s": wall, "error": err}
    rows = ep.all_gather(row)
    if rank == 0:
        th.join()
        sums_ok = all(r["sums"] == want_sums for r in rows)
        out = {"n": N, "sharded": a.sharded,
               "sys_fence": bool(os.environ.get("MD_AR_SYS_FENCE")),
               "calls": calls, "per_graph": a.per_graph, "max_skew_us": a.max_skew_us,
               "route": rows[0]["route"],
               "ok": sums_ok and all(r["bad_calls_w"] == 0 and r["bad_calls_g"] == 0
                                     and r["first_sum_ok"] and r["error"] is None for r in rows),
               "oracle_checksums_match": sums_ok,
               "per_rank": [{k: v for k, v in r.items() if k != "sums"} for r in rows]}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
