import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

try:
    from hypothesis import settings

    settings.register_profile("md", deadline=None, max_examples=40)
    settings.load_profile("md")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs on one box")


@pytest.fixture(scope="session")
def golden():
    # eager dict: the lazy NpzFile is not safe to read from rank threads
    with np.load(ROOT / "tests" / "golden" / "golden.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.lib()  # builds the C restatement if needed
    return o


def n_gpus() -> int:
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


def need_gpus(n: int):
    return pytest.mark.skipif(n_gpus() < n, reason=f"needs {n} GPUs on one box")


os.environ.setdefault("PYTHONHASHSEED", "0")
