#!/usr/bin/env python3
"""BASELINE config C4: the DIMD store on B200 -- per-epoch shuffle (partition
exchange over NVLink) and minibatch gather, with bit-exact indices.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench_dimd.py [--records 160000]

Every rank holds a shard of `--records` synthetic 224x224x3 uint8 records
(24.08 GB at 160,000; C4 puts 1.28M records on 8 GPUs = 160,000 each),
striped by the reference rule (dimd.py:192). `--epochs` successive
`shuffle_all` epochs (keys _mix64(seed, "shuf", epoch); m_segments =
default_segments(shard bytes), as the reference computes it) are timed (wall,
max over ranks; steady state = median of epochs >= 3). After every epoch each
record is verified against the generator; after the first, every slot's
source index is compared with the CPU oracle's plan (numpy-Philox semantics)
-- bit-exact indices. Then the training loop's 32-record batches (CUDA-graph
replays of BatchStream.next()) and one bulk gather are timed. Prints one JSON line.
Roofline: the exchange must move (S-1)/S of the shard bytes over NVLink
(pull) and write every byte once into HBM.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
REC = 224 * 224 * 3


def _hbm_peak():
    try:
        from bench import hbm_peak
        return hbm_peak()
    except Exception:
        return None


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", type=int, default=160_000)
    ap.add_argument("--gathers", type=int, default=1000)
    ap.add_argument("--bulk", type=int, default=8192, help="records in the bulk-gather probe")
    ap.add_argument("--seed", type=int, default=2017)
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--epochs", type=int, default=5)
    ap.add_argument("--exchange", choices=["push", "pull"], default="push",
                    help="shuffle data movement (dimd.EXCHANGE)")
    ap.add_argument("--no-prefetch-plan", dest="prefetch_plan", action="store_false",
                    help="do not pass next_seed (plan every epoch inside its own shuffle)")
    ap.add_argument("--cpu-records", type=int, default=1024,
                    help="records per member of the host (CPU reference) shuffle row; 0 = none")
    a = ap.parse_args()

    import torch

    from oracle import oracle as O
    from paper_1711_00705_b200 import dimd
    from paper_1711_00705_b200.dimd import BatchRequest, BatchSlots, random_batch_device
    from paper_1711_00705_b200.sgd import SAMPLE_ROLE
    from paper_1711_00705_b200.transport import init_from_env

    ep = init_from_env()
    N, rank, dev = ep.n_ranks, ep.rank, ep.torch_device
    dimd.EXCHANGE = a.exchange
    S, n = N, a.records
    # epoch keys _mix64(seed, "shuf", epoch), sgd.py:503-506
    with torch.cuda.stream(ep.stream):
        store = dimd.synth_store(n, REC, rank, S, a.seed, 0, S, rank, device=dev)
        torch.cuda.synchronize(dev)
        m_seg = dimd.default_segments(store.nbytes)
        walls, evs, phases_all = [], [], []
        bad, exact = 0, None
        for epoch in range(a.epochs):
            key = O.mix64(a.seed, O.SHUF_ROLE, epoch)
            ep.barrier()
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ep.stream)
            nxt = O.mix64(a.seed, O.SHUF_ROLE, epoch + 1) if a.prefetch_plan else None
            out = dimd.shuffle_all(ep, store, m_segments=m_seg, seed=key, next_seed=nxt)
            e1.record(ep.stream)
            torch.cuda.synchronize(dev)
            walls.append(time.perf_counter() - t0)
            evs.append(e0.elapsed_time(e1))
            phases_all.append(dict(dimd.LAST_SHUFFLE_PHASES))
            if not a.no_verify:
                b, gids = dimd.synth_verify(out, a.seed)
                bad += b
                if epoch == 0:  # indices: every slot's source vs the oracle's plan
                    mem, rec = O.shuffle_plan_c(key, 0, S, rank, rank, m_seg, [n] * S)
                    exact = bool(np.array_equal(gids.cpu().numpy(), mem + S * rec))
            store = out
        # steady state: the first epochs pay one-time CUDA IPC mappings of the
        # peers' shard allocations (cached afterwards, dimd._ShardArena)
        wall, ev_ms = float(np.median(walls[2:] if len(walls) > 2 else walls)), evs[-1]
        n_out = out.n_records
        # minibatch gathers from the new shard. (1) the training loop's
        # 32-record batches: BatchStream.next() (device-keyed picks + gather)
        # captured 100x into one CUDA graph, replayed -- device time per batch,
        # no host work in between; (2) one bulk gather of --bulk records for
        # the kernel's HBM roofline (read + write of every record byte).
        bs = dimd.BatchStream(out, 32, REC, a.seed, SAMPLE_ROLE, rank)
        for _ in range(5):
            bs.next()
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=ep.stream, capture_error_mode="thread_local"):
            for _ in range(100):
                bs.next()
        graph.replay()
        torch.cuda.synchronize(dev)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, a.gathers // 100)
        g0.record(ep.stream)
        for _ in range(reps):
            graph.replay()
        g1.record(ep.stream)
        torch.cuda.synchronize(dev)
        bs.slots.check()
        gather_ms = g0.elapsed_time(g1) / (100 * reps)
        bulk = BatchSlots(a.bulk, REC, dev)
        random_batch_device(out, BatchRequest(a.bulk, 1), REC, bulk)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(ep.stream)
        for i in range(5):
            random_batch_device(out, BatchRequest(a.bulk, 2 + i), REC, bulk)
        b1.record(ep.stream)
        torch.cuda.synchronize(dev)
        bulk.check()
        bulk_ms = b0.elapsed_time(b1) / 5
        # the gather kernel alone (picks already drawn): its HBM roofline
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(ep.stream)
        for i in range(5):
            dimd._gather_fixed(out, bulk, a.bulk, REC)
        k1.record(ep.stream)
        torch.cuda.synchronize(dev)
        bulk.check()
        gather_only_ms = k0.elapsed_time(k1) / 5
        del bulk
    rows = ep.all_gather((wall, ev_ms, n_out, bad, exact, gather_ms, phases_all, walls, bulk_ms,
                          gather_only_ms))
    if rank == 0:
        wall = max(r[0] for r in rows)
        total = sum(r[2] for r in rows)
        nvlink_bytes = n * REC * (S - 1) / S  # expected pulled bytes per GPU
        line = {
            "metric": "DIMD shuffle records/s (whole job) and minibatch gather records/s per GPU",
            "n_gpus": N, "records_per_gpu": n, "record_bytes": REC, "m_segments": m_seg,
            "epochs": a.epochs,
            "shuffle_s_per_epoch": [max(r[7][e] for r in rows) for e in range(a.epochs)],
            "shuffle_s": wall, "shuffle_s_is": "median over epochs >= 3 (steady state)",
            "shuffle_records_per_s": total / wall,
            "shuffle_GBps_per_gpu": n * REC / wall / 1e9,
            "nvlink_GBps_per_gpu": nvlink_bytes / wall / 1e9 if S > 1 else None,
            "hbm_GBps_per_gpu": 2 * n * REC / wall / 1e9,
            "shuffle_event_ms_max": max(r[1] for r in rows),
            "records_out": [r[2] for r in rows],
            "corrupt_records": sum(max(0, r[3]) for r in rows),
            "indices_bit_exact_vs_oracle": all(r[4] for r in rows) if not a.no_verify else None,
            "batch32_ms": max(r[5] for r in rows),
            "batch32_is": "BatchStream.next() (picks + gather), 100 per CUDA graph, device time",
            "batch32_records_per_s_per_gpu": 32 / (max(r[5] for r in rows) / 1e3),
            "exchange": a.exchange,
            "plan_prefetch": a.prefetch_plan,
            "bulk_gather_records": a.bulk,
            "bulk_gather_is": "random_batch_device: Philox picks of --bulk records + gather kernel",
            "bulk_gather_ms": max(r[8] for r in rows),
            "gather_kernel_ms": max(r[9] for r in rows),
            "gather_kernel_is": "md_gather alone on the same picks (2 x record bytes per record)",
            "gather_kernel_hbm_GBps": 2 * a.bulk * REC / (max(r[9] for r in rows) / 1e3) / 1e9,
            "bulk_gather_records_per_s_per_gpu": a.bulk / (max(r[8] for r in rows) / 1e3),
            "bulk_gather_hbm_GBps": 2 * a.bulk * REC / (max(r[8] for r in rows) / 1e3) / 1e9,
        }
        peak = _hbm_peak()
        if peak:
            line["bulk_gather_hbm_frac"] = line["bulk_gather_hbm_GBps"] / peak[0]
            line["gather_kernel_hbm_frac"] = line["gather_kernel_hbm_GBps"] / peak[0]
            line["hbm_peak"] = {"GBps": peak[0], "source": peak[1]}
        if rows[0][6] and rows[0][6][-1]:
            line["phases_s_per_rank"] = [r[6] for r in rows]
        if a.cpu_records > 0:
            line["cpu_baseline"] = cpu_shuffle(S, a.cpu_records, a.seed)
        print(json.dumps(line), flush=True)
    ep.barrier()


def cpu_shuffle(S: int, n_local: int, seed: int, seconds: float = 5.0) -> dict:
    """The reference algorithm of one shuffle epoch on the host, for a scaled
    corpus (S members x n_local records of 224x224x3 bytes): every receiver's
    plan with the oracle's C port of dimd.py:281-350 (numpy-Philox dest draws,
    receive order, permutation), then the bytes moved into each receiver's new
    blob (numpy take). Single thread. The reference itself (Python over its
    threads transport) measured 2,337 records/s for 8,192 records at N = 8 in
    the build container."""
    import os

    from oracle import oracle as O

    rng = np.random.default_rng(seed)
    blobs = [rng.integers(0, 256, size=(n_local, REC), dtype=np.uint8) for _ in range(S)]
    m_seg = 4
    key = O.mix64(seed, O.SHUF_ROLE, 0)
    t0, reps = time.perf_counter(), 0
    while reps < 2 or time.perf_counter() - t0 < seconds:
        for r in range(S):
            mem, rec = O.shuffle_plan_c(key, 0, S, r, r, m_seg, [n_local] * S)
            out = np.empty((len(mem), REC), np.uint8)
            for q in range(S):
                sel = mem == q
                out[sel] = np.take(blobs[q], rec[sel], axis=0)
        reps += 1
    dt = (time.perf_counter() - t0) / reps
    return {"value": S * n_local / dt, "unit": "records/s (whole job)", "cores": 1,
            "kind": "port", "affinity_cores": len(os.sched_getaffinity(0)),
            "sample": f"one epoch of {S} x {n_local} records (150,528 B) on the host, "
                      f"oracle C plan + numpy byte moves, {reps} repetitions"}


if __name__ == "__main__":
    main()
