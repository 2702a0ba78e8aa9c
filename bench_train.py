#!/usr/bin/env python3
"""The reference's training benchmark on B200: ``bench_train``
(/root/reference/pkg/src/minidist/bench.py:379-422) -- median per-epoch time
of ``run_training`` per (algorithm, rank count) for the reference's own model
(ToyModel 16 -> hidden -> 4 on make_synthetic_corpus records; defaults =
the reference's BenchSpec: 4,096 records, 2 workers x 8 samples per rank,
hidden 2048, 3 epochs, bench.py:71-75).

Everything runs on the GPUs: the DIMD store and its per-epoch shuffle, the
ToyModel gradients (md_toy_grad), the fused fold + allreduce + update and the
replica check. One thread per rank, one GPU per rank when the box has enough
GPUs (else ranks are emulated on one GPU; the line says which).

    python bench_train.py [--ranks 1 2 4] [--algorithms multicolor ring reduce_bcast]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench_train.py --backend torchrun

Prints the reference's CSV rows (bench.py:41) and one JSON summary line. The
reference's own numbers for the same spec on the build container's CPU come
from tools/ref_cpu_bench.py (threads backend).
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CSV_HEADER = "scenario,algorithm,n_ranks,payload_bytes,median_time_s,throughput_GBps,backend"


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--algorithms", nargs="+", default=["multicolor", "ring", "reduce_bcast"])
    ap.add_argument("--records", type=int, default=4096)
    ap.add_argument("--workers", type=int, default=2)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--hidden", type=int, default=2048)
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--backend", choices=["cuda", "torchrun"], default="cuda",
                    help="cuda: one thread per rank in this process; torchrun: run under "
                         "torchrun, one process per GPU (ranks = WORLD_SIZE)")
    a = ap.parse_args()
    if a.backend == "torchrun":
        import os

        a.ranks = [int(os.environ.get("WORLD_SIZE", "1"))]

    import torch

    from paper_1711_00705_b200 import TrainConfig, make_synthetic_corpus, run_training
    from paper_1711_00705_b200.errors import MinidistError

    corpus = make_synthetic_corpus(a.records, seed=a.seed)
    n_gpus = torch.cuda.device_count()
    rows, out = [CSV_HEADER], []
    for algo in a.algorithms:
        for n in a.ranks:
            cfg = TrainConfig(n_nodes=n, workers_per_node=a.workers, per_worker_batch=a.batch,
                              epochs=a.epochs, seed=a.seed, hidden=a.hidden)
            emulate = n > n_gpus and a.backend == "cuda"
            t0 = time.perf_counter()
            try:
                if a.backend == "torchrun":
                    res = run_training(cfg, corpus, algo, backend="torchrun")
                else:
                    res = run_training(cfg, corpus, algo, emulate=emulate)
            except MinidistError as e:
                print(f"skipping train {algo} n={n}: {e}", file=sys.stderr)
                continue
            wall = time.perf_counter() - t0
            med = statistics.median(h.time_s for h in res.history)
            grad_bytes = (len(res.weights) + 2) * 4
            rows.append(f"train,{algo},{n},{grad_bytes},{med!r},0.0,cuda")
            steps = max(1, len(corpus) // cfg.effective_batch)
            out.append({"algorithm": algo, "n_ranks": n, "median_epoch_s": med,
                        "steps_per_epoch": steps, "ms_per_step": 1e3 * med / steps,
                        "epoch_s": [h.time_s for h in res.history], "final_acc": res.final_acc,
                        "final_loss": res.history[-1].loss, "wall_s": wall,
                        "ranks": ("one process per GPU" if a.backend == "torchrun" else
                                  "emulated on one GPU" if emulate else
                                  "one GPU per rank (threads)")})
    import os

    if int(os.environ.get("RANK", "0")) != 0:
        return
    print("\n".join(rows))
    print(json.dumps({"metric": "bench_train median epoch time (reference bench.py:379-422)",
                      "unit": "s", "spec": {"records": a.records, "workers": a.workers,
                                            "batch": a.batch, "hidden": a.hidden,
                                            "epochs": a.epochs, "seed": a.seed},
                      "gpus": n_gpus, "rows": out}), flush=True)


if __name__ == "__main__":
    main()
