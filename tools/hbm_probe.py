#!/usr/bin/env python3
"""HBM streaming probe on one GPU: torch copy (the MEASURED_PEAKS method),
md_sgd_update (standalone grid-stride kernel) and the fused allreduce kernel at
N = 1 (lone-root momentum/wd update), 25.6M floats, CUDA-event medians."""

from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch

    from paper_1711_00705_b200 import _kernels, run_ranks
    from paper_1711_00705_b200.collectives import GradientBuffer, SgdUpdate, allreduce

    P = 25_600_000
    dev = torch.device("cuda", 0)

    def timeit(fn, reps=20):
        ts = []
        for i in range(reps + 3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    src = torch.randn(P * 4, device=dev)
    dst = torch.empty_like(src)
    t = timeit(lambda: dst.copy_(src))
    out = {"torch_copy_GBps": 2 * src.numel() * 4 / t / 1e6}
    w = torch.randn(P, device=dev)
    g = torch.randn(P, device=dev)
    v = torch.randn(P, device=dev)
    t = timeit(lambda: _kernels.sgd_update(w, g, v, c=1e-4, mu=0.9, wd_b=0.0032))
    out["md_sgd_update_mom_wd_GBps"] = 20 * P / t / 1e6
    t = timeit(lambda: _kernels.sub_scaled_f32(w, g, 1e-4))
    out["md_sub_scaled_GBps"] = 12 * P / t / 1e6

    def prog(ep):
        buf = GradientBuffer.alloc(P, ep)
        upd = SgdUpdate(weights=w, c=1e-4, momentum=v, mu=0.9, wd_b=0.0032)
        with torch.cuda.stream(torch.cuda.current_stream()):
            return timeit(lambda: allreduce(ep, buf, "multicolor", update=upd, check=False))

    t = run_ranks(1, "cuda", prog).results[0]
    out["fused_allreduce_n1_GBps"] = 20 * P / t / 1e6
    print(json.dumps({k: round(x, 1) for k, x in out.items()}))


if __name__ == "__main__":
    main()
