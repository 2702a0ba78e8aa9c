#!/usr/bin/env python3
"""Time the REAL reference's training benchmark (minidist.bench.bench_train,
bench.py:379-422) on this container's CPU cores, threads backend, with the
spec bench_train.py uses on the GPU (the reference's BenchSpec defaults:
4,096 records, 2 workers x 8 samples, hidden 2048, 3 epochs). Runs only where
/root/reference exists (the build container).

    python tools/ref_train_bench.py > profiles/r02_ref_train_container.json
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests" / "golden"))

from make_golden import import_reference  # noqa: E402


def main() -> None:
    import_reference()
    from minidist.bench import BenchSpec, bench_train

    out = {"host": "build container (no GPU)", "cores": len(os.sched_getaffinity(0)),
           "backend": "threads", "rows": []}
    t0 = time.time()
    for n in (1, 2, 4):
        spec = BenchSpec(scenario="train", algorithms=("multicolor", "ring", "reduce_bcast"),
                         rank_sweep=(n,), backend="threads")
        rows, _ = bench_train(spec)
        for r in rows:
            out["rows"].append({"algorithm": r.algorithm, "n_ranks": r.n_ranks,
                                "payload_bytes": r.payload_bytes,
                                "median_epoch_s": r.median_time_s})
    out["spec"] = {"records": spec.train_records, "workers": spec.train_workers,
                   "batch": spec.train_batch, "hidden": spec.train_hidden,
                   "epochs": spec.train_epochs}
    out["wall_s"] = time.time() - t0
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
