"""One fused N = 2 allreduce + SGD(momentum, wd) call of the C5 size with both
ranks emulated on ONE GPU (one cooperative launch of allreduce_stream_kernel,
peer reads are local HBM) -- the single-GPU form of the N = 2 kernel that ncu
can replay. Used only for the ncu capture in profiles/ (a multi-rank command
must not run under ncu)."""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_00705_b200 import (GradientBuffer, SgdUpdate, allreduce,  # noqa: E402
                                   build_multicolor_trees, run_ranks)


L, P = 25_600_002, 25_600_000
ts = build_multicolor_trees(2, 2, 4)


def prog(ep):
    dev = ep.torch_device
    g = torch.randn(L, device=dev)
    w = torch.randn(P, device=dev)
    m = torch.zeros(P, device=dev)
    for _ in range(3):
        buf = GradientBuffer(g.clone())
        allreduce(ep, buf, "multicolor", tree_set=ts,
                  update=SgdUpdate(weights=w, c=1e-3, momentum=m, mu=0.9, wd_b=3.2e-3, update_len=P))
    torch.cuda.synchronize(dev)
    return True


print(run_ranks(2, "cuda", prog, emulate=True).results)
