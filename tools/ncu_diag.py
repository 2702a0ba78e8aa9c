"""Minimal torchrun rank for diagnosing ncu on one rank: rendezvous, one IPC
registration, one tiny allreduce. Prints the step it reached."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
print("start", flush=True)
import torch  # noqa: E402
from paper_1711_00705_b200 import GradientBuffer, allreduce  # noqa: E402
from paper_1711_00705_b200.transport import init_from_env  # noqa: E402
ep = init_from_env()
print("rendezvous ok", ep.rank, flush=True)
buf = GradientBuffer.alloc(1 << 20, ep)
print("ipc ok", flush=True)
buf.data.fill_(1.0)
allreduce(ep, buf, "multicolor")
print("allreduce ok", float(buf.data[0]), flush=True)
