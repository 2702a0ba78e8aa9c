#!/usr/bin/env python3
"""Time the REAL reference (minidist, /root/reference) on this container's
CPU cores through its own benchmark API (minidist.bench.bench_allreduce /
bench_shuffle, threads backend) -- the reference-side rows of the C1/C2 and
C4 tables. Runs only where /root/reference exists (the build container; the
GPU box times the oracle's C port instead, bench.py / bench_sweep.py).

    python tools/ref_cpu_bench.py > profiles/r02_ref_cpu_container.json
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))

from make_golden import import_reference  # noqa: E402


def main() -> None:
    import_reference()
    from minidist import _kernels
    from minidist.bench import BenchSpec, bench_allreduce, bench_shuffle

    cores = len(os.sched_getaffinity(0))
    out = {"host": "build container (no GPU)", "cores": cores,
           "kernels_backend": getattr(_kernels, "BACKEND", "?"), "rows": []}
    t0 = time.time()
    # C1 (N = 4, k = 4, 25.6M floats) and a C2-style size sweep at N = 2 / 4
    for n, ks in ((2, (1, 2)), (4, (1, 2, 4))):
        for k in ks:
            spec = BenchSpec(scenario="allreduce", algorithms=("multicolor",), rank_sweep=(n,),
                             k_colors=k, arity=4, backend="threads", repetitions=3,
                             payload_bytes=(4 << 10, 1 << 20, 16 << 20, 102_400_000))
            for r in bench_allreduce(spec):
                out["rows"].append({"scenario": r.scenario, "algorithm": f"multicolor_k{k}_a4",
                                    "n_ranks": r.n_ranks, "payload_bytes": r.payload_bytes,
                                    "median_time_s": r.median_time_s,
                                    "bus_GBps": r.throughput_GBps, "backend": r.backend})
    # C4-style shuffle, scaled corpus (the reference keeps it in host RAM)
    for n in (2, 4, 8):
        spec = BenchSpec(scenario="shuffle", rank_sweep=(n,), groups=(1,), backend="threads",
                         repetitions=3, corpus_records=8192, record_bytes=REC_BYTES)
        for r in bench_shuffle(spec):
            out["rows"].append({"scenario": r.scenario, "algorithm": r.algorithm,
                                "n_ranks": r.n_ranks, "corpus_records": 8192,
                                "record_bytes": REC_BYTES, "median_time_s": r.median_time_s,
                                "records_per_s": 8192 / r.median_time_s,
                                "backend": r.backend})
    out["wall_s"] = time.time() - t0
    print(json.dumps(out, indent=1))


REC_BYTES = 224 * 224 * 3

if __name__ == "__main__":
    main()
