"""The multi-process path (torchrun, one process per GPU, CUDA IPC): the
allreduce + fused update bitwise vs the oracle, back-to-back calls, the DIMD
shuffle (indices vs the oracle's plan, bytes vs the generator) and alltoallv,
all through init_from_env exactly as bench.py runs them."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

from tests.conftest import need_gpus

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = Path(__file__).resolve().parents[1]


def _torchrun(n: int, port: int) -> dict:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(ROOT / "tests" / "_mp_worker.py")]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [x for x in p.stdout.splitlines() if x.startswith("{")][-1]
    return json.loads(line)


@need_gpus(2)
def test_torchrun_two_processes():
    res = _torchrun(2, 29851)
    assert res["ok"], res["rows"]


@need_gpus(4)
def test_torchrun_four_processes():
    res = _torchrun(4, 29852)
    assert res["ok"], res["rows"]
