#!/usr/bin/env python3
"""N=1: the fused allreduce kernel's lone-root SGD update vs the standalone
md_sgd_update kernel on the C5 buffers (fill first, as in the step)."""
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_1711_00705_b200 import _lib
    from paper_1711_00705_b200.collectives import GradientBuffer, SgdUpdate, allreduce
    from paper_1711_00705_b200.transport import init_from_env

    ep = init_from_env()
    dev = ep.torch_device
    lib = _lib.load()
    P = 25_600_000
    grad = GradientBuffer.alloc(P + 2, ep)
    w = torch.randn(P, device=dev) * 0.01
    m = torch.zeros(P, device=dev)
    s = ep.stream
    sp = _lib.stream_ptr(s)
    upd = SgdUpdate(weights=w, c=1e-4, momentum=m, mu=0.9, wd_b=0.0032, update_len=P)
    out = {}

    def fill():
        lib.md_fill_rank_input(grad.data.data_ptr(), P + 2, 0, 1, sp)

    variants = {
        "fused_allreduce": lambda: allreduce(ep, grad, "multicolor", update=upd, check=False),
        "md_sgd_update": lambda: _lib.check(lib.md_sgd_update(w.data_ptr(), grad.data.data_ptr(),
                                                              m.data_ptr(), P, 1e-4, 0.9, 0.0032, sp)),
    }
    with torch.cuda.stream(s):
        for name, fn in variants.items():
            ts = []
            for i in range(25):
                fill()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                fn()
                e1.record(s)
                ts.append((e0, e1))
            torch.cuda.synchronize(dev)
            v = [a.elapsed_time(b) * 1e3 for a, b in ts[5:]]
            out[name] = (round(statistics.median(v), 2), round(min(v), 2))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
