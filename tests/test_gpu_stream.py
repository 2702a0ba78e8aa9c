"""The stream (all-pull, tiled) kernel as the DEFAULT route of replicated
fused N = 2 calls at the C5 size (25.6M + 2 floats, momentum + weight decay):
no route pinned, balanced tiles chosen by md_allreduce (and the test checks
that the stream kernel is what ran). Same bits as the oracle's fold + float32
update (the reference order: at N = 2 every color folds root + child, and the
update is the oracle's sgd_np)."""

import numpy as np
import pytest
import torch

from paper_1711_00705_b200 import GradientBuffer, _lib, build_multicolor_trees, run_ranks
from paper_1711_00705_b200.collectives import SgdUpdate, allreduce
from tests.conftest import need_gpus

pytestmark = pytest.mark.gpu

L = 25_600_002
P = L - 2


@pytest.fixture(autouse=True)
def default_route(monkeypatch):
    from paper_1711_00705_b200 import collectives

    monkeypatch.setattr(collectives, "_DEFAULT_ROUTE", "auto")


def _case(oracle, k, seed):
    rng = np.random.default_rng(seed)
    arrays = [rng.standard_normal(L).astype(np.float32) for _ in range(2)]
    w0 = rng.standard_normal(P).astype(np.float32)
    m0 = rng.standard_normal(P).astype(np.float32)
    tables = oracle.tables_from_trees(2, oracle.trees(2, k, 4))
    want = oracle.fold_c(tables, arrays)
    want_w, want_m = oracle.sgd_np(w0, want[:P], m0.copy(), 1e-3, 0.9, 3.2e-3)
    return arrays, w0, m0, want, want_w, want_m


def _prog(arrays, w0, m0, ts, steps=1):
    def prog(ep):
        dev = ep.torch_device
        w = torch.from_numpy(w0.copy()).to(dev)
        m = torch.from_numpy(m0.copy()).to(dev)
        for _ in range(steps):
            buf = GradientBuffer(torch.from_numpy(arrays[ep.rank].copy()).to(dev))
            upd = SgdUpdate(weights=w, c=1e-3, momentum=m, mu=0.9, wd_b=3.2e-3, update_len=P)
            allreduce(ep, buf, "multicolor", tree_set=ts, update=upd)
        route = _lib.last_route(ep.device)
        return buf.data.cpu().numpy(), w.cpu().numpy(), m.cpu().numpy(), route

    return prog


@pytest.mark.parametrize("k", [1, 2])
def test_c5_size_fused_emulated(oracle, k):
    arrays, w0, m0, want, want_w, want_m = _case(oracle, k, 11 + k)
    ts = build_multicolor_trees(2, k, 4)
    for g, w, m, route in run_ranks(2, "cuda", _prog(arrays, w0, m0, ts), emulate=True).results:
        assert route[0] == "stream"
        assert np.array_equal(g, want)
        assert np.array_equal(w, want_w)
        assert np.array_equal(m, want_m)


@need_gpus(2)
def test_c5_size_fused_two_gpus_back_to_back(oracle):
    """One process, two GPUs over NVLink; two calls in a row (the second
    reuses the per-tile read flags with the next epoch)."""
    arrays, w0, m0, want, _, _ = _case(oracle, 2, 5)
    w1, m1 = oracle.sgd_np(w0, want[:P], m0.copy(), 1e-3, 0.9, 3.2e-3)
    w2, m2 = oracle.sgd_np(w1, want[:P], m1.copy(), 1e-3, 0.9, 3.2e-3)
    ts = build_multicolor_trees(2, 2, 4)
    for g, w, m, route in run_ranks(2, "cuda", _prog(arrays, w0, m0, ts, steps=2),
                                    emulate=False).results:
        assert route[0] == "stream"
        assert np.array_equal(g, want)
        assert np.array_equal(w, w2)
        assert np.array_equal(m, m2)
