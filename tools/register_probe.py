#!/usr/bin/env python3
"""Cost of the shuffle's registration step, piece by piece: IPC export of a
shard's arrays, the host all_gather, the (cached) imports.

    torchrun --nproc-per-node N tools/register_probe.py
"""
import ctypes as C
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1711_00705_b200 import _lib, dimd  # noqa: E402
from paper_1711_00705_b200.transport import init_from_env  # noqa: E402


def main():
    ep = init_from_env()
    dev = ep.torch_device
    store = dimd.synth_store(160_000, 224 * 224 * 3, ep.rank, ep.n_ranks, 1, 0, ep.n_ranks, ep.rank,
                             device=dev)
    arrays = [store.blob, store.off, store.length, store.label]
    torch.cuda.synchronize(dev)
    lib = _lib.load()
    out = {"rank": ep.rank}
    for rep in range(4):
        ep.barrier()
        t0 = time.perf_counter()
        for t in arrays:
            h = C.create_string_buffer(_lib.IPC_BYTES)
            off = C.c_uint64()
            _lib.check(lib.md_mem_export(C.c_void_p(t.data_ptr()), h, C.byref(off)))
        t1 = time.perf_counter()
        ep.all_gather((1, 2, b"x" * 256))
        t2 = time.perf_counter()
        ep.register_varlen_many(arrays, (1, 2))
        t3 = time.perf_counter()
        out[f"rep{rep}"] = {"export4_ms": round((t1 - t0) * 1e3, 3),
                            "all_gather_ms": round((t2 - t1) * 1e3, 3),
                            "register_many_ms": round((t3 - t2) * 1e3, 3)}
    # as the shuffle does: fresh index arrays every epoch, the previous ones alive
    prev = None
    for rep in range(4):
        fresh = [torch.empty(160_000 + rep, dtype=torch.int64, device=dev),
                 torch.empty(160_000 + rep, dtype=torch.int32, device=dev),
                 torch.empty(160_000 + rep, dtype=torch.int32, device=dev)]
        torch.cuda.synchronize(dev)
        ep.barrier()
        t0 = time.perf_counter()
        ep.register_varlen_many([store.blob] + fresh, (1, 2))
        out[f"fresh{rep}_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
        prev, fresh = fresh, None  # noqa: F841
    rows = ep.all_gather(out)
    if ep.rank == 0:
        for r in rows:
            print(json.dumps(r))


if __name__ == "__main__":
    main()
