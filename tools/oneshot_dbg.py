#!/usr/bin/env python3
"""Debug: one-shot allreduce under eager calls and CUDA-graph replays (torchrun)."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    from paper_1711_00705_b200 import _lib
    from paper_1711_00705_b200.collectives import GradientBuffer, allreduce
    from paper_1711_00705_b200.sgd import comm_plan
    from paper_1711_00705_b200.transport import init_from_env

    ep = init_from_env(pull_timeout=3.0)
    N, rank, dev = ep.n_ranks, ep.rank, ep.torch_device
    lib = _lib.load()
    ts, _ = comm_plan(N, "multicolor")
    n = int(os.environ.get("DBG_N", "1024"))
    buf = GradientBuffer.alloc(n, ep)
    s = ep.stream
    log = []
    with torch.cuda.stream(s):
        for mode in ("eager", "graph"):
            try:
                if mode == "eager":
                    for i in range(50):
                        buf.data.fill_(1.0)
                        allreduce(ep, buf, "multicolor", tree_set=ts, check=False)
                    torch.cuda.synchronize(dev)
                    ep.take_error()
                    log.append((mode, float(buf.data[0])))
                else:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                        for _ in range(20):
                            allreduce(ep, buf, "multicolor", tree_set=ts, check=False)
                    for r in range(3):
                        ep.barrier()
                        buf.data.fill_(1.0)
                        g.replay()
                        torch.cuda.synchronize(dev)
                        ep.take_error()
                        log.append((mode, r, float(buf.data[0])))
            except Exception as e:  # noqa: BLE001
                torch.cuda.synchronize(dev)
                ctrl = ctypes_ctrl(lib, ep)
                log.append((mode, "FAIL", repr(e)[:200], ctrl))
                break
    print(json.dumps({"rank": rank, "log": log}), flush=True)


def ctypes_ctrl(lib, ep):
    import ctypes

    import torch
    p = ctypes.c_void_p()
    lib.md_comm_ctrl_ptr(ep.comm, ctypes.byref(p))
    words = torch.empty(64, dtype=torch.int32, device=ep.torch_device)
    torch.cuda.synchronize()
    cud = ctypes.CDLL("libcudart.so")
    host = (ctypes.c_uint32 * 96)()
    cud.cudaMemcpy(host, p, 96 * 4, 2)
    return list(host)


if __name__ == "__main__":
    main()
