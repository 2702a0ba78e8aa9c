"""The owner-computes schedule (md_plan_set_schedule(MD_SCHED_OWNER),
``schedule="owner"``): every golden case of the reference, bitwise, through
the channelized tree kernel over the owner plan (the latency paths are
switched off here so the owner plan is what runs).

Ranks are emulated on one GPU (one cooperative launch serves all ranks); the
last test repeats a case with one GPU per rank when the box has them.
"""

import numpy as np
import pytest
import torch

from paper_1711_00705_b200 import (
    GradientBuffer,
    SgdUpdate,
    allreduce,
    build_multicolor_trees,
    build_ring,
    errors,
    run_ranks,
)
from tests.conftest import need_gpus
from tests.test_oracle import GOLD_MC

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _owner_plan_only(monkeypatch):
    """The owner plan runs on the channelized tree kernel: pin that route."""
    from paper_1711_00705_b200 import collectives

    monkeypatch.setattr(collectives, "_DEFAULT_ROUTE", "tree")


def run(n, arrays, algo, emulate=True, **kw):
    def prog(ep):
        buf = GradientBuffer(torch.from_numpy(arrays[ep.rank].copy()).to(ep.torch_device))
        return allreduce(ep, buf, algo, schedule="owner", **kw).data.cpu().numpy()

    return run_ranks(n, "cuda", prog, emulate=emulate).results


@pytest.mark.parametrize("n,L,k,arity", GOLD_MC)
@pytest.mark.parametrize("seg", [64, 16384])
def test_owner_multicolor_matches_reference(golden, n, L, k, arity, seg):
    inp = golden[f"mc_{n}_{L}_{k}_{arity}_in"]
    want = golden[f"mc_{n}_{L}_{k}_{arity}_out"]
    ts = build_multicolor_trees(n, k, arity)
    for r in run(n, list(inp), "multicolor", tree_set=ts, segment_elems=seg):
        assert np.array_equal(r, want)


@pytest.mark.parametrize("n,L", [(8, 1000), (5, 333), (2, 4), (4, 4099)])
def test_owner_ring_matches_reference(golden, n, L):
    out = run(n, list(golden[f"ring_{n}_{L}_in"]), "ring", ring=build_ring(n), segment_elems=100)
    for r in out:
        assert np.array_equal(r, golden[f"ring_{n}_{L}_out"])


@pytest.mark.parametrize("n,L,root", [(8, 513, 0), (4, 4099, 3)])
def test_owner_reduce_bcast_matches_reference(golden, n, L, root):
    for r in run(n, list(golden[f"rb_{n}_{L}_{root}_in"]), "reduce_bcast", root=root):
        assert np.array_equal(r, golden[f"rb_{n}_{L}_{root}_out"])


@pytest.mark.parametrize("n,k,arity", [(4, 1, 4), (4, 2, 4), (8, 4, 4), (8, 8, 7)])
def test_owner_large_unaligned_slices_with_fused_update(oracle, n, k, arity):
    """A 2.5M + 3 float buffer: slice and color boundaries fall inside float4
    groups (scalar edges, mixed-color groups); fused momentum/wd epilogue."""
    rng = np.random.default_rng(n * 10 + k)
    L = 2_500_003
    P = L - 2
    arrays = [rng.standard_normal(L).astype(np.float32) for _ in range(n)]
    w0 = rng.standard_normal(P).astype(np.float32)
    tables = oracle.tables_from_trees(n, oracle.trees(n, k, arity))
    want = oracle.fold_c(tables, arrays)
    want_w, want_m = oracle.sgd_np(w0, want[:P], np.zeros(P, np.float32), 1e-3, 0.9, 3.2e-3)
    ts = build_multicolor_trees(n, k, arity)

    def prog(ep):
        dev = ep.torch_device
        buf = GradientBuffer(torch.from_numpy(arrays[ep.rank].copy()).to(dev))
        w = torch.from_numpy(w0.copy()).to(dev)
        m = torch.zeros(P, device=dev)
        upd = SgdUpdate(weights=w, c=1e-3, momentum=m, mu=0.9, wd_b=3.2e-3, update_len=P)
        allreduce(ep, buf, "multicolor", tree_set=ts, update=upd, schedule="owner")
        return buf.data.cpu().numpy(), w.cpu().numpy(), m.cpu().numpy()

    for g, w, m in run_ranks(n, "cuda", prog, emulate=True).results:
        assert np.array_equal(g, want)
        assert np.array_equal(w, want_w)
        assert np.array_equal(m, want_m)


def test_owner_with_worker_fold_keeps_the_tree_schedule(oracle):
    """Worker folds run on the tree schedule (the owner plan would read the
    peers' unfolded buffers); the call still succeeds with the same bits."""
    n, P = 4, 10_007
    rng = np.random.default_rng(3)
    workers = [[rng.standard_normal(P).astype(np.float32) for _ in range(2)] for _ in range(n)]
    tables = oracle.tables_from_trees(n, oracle.trees(n, 4, 4))
    want = oracle.fold_c(tables, [w[0] + w[1] for w in workers])

    def prog(ep):
        dev = ep.torch_device
        buf = GradientBuffer.zeros(P, device=dev)
        allreduce(ep, buf, "multicolor", schedule="owner",
                  workers=[torch.from_numpy(x).to(dev) for x in workers[ep.rank]])
        return buf.data.cpu().numpy()

    for r in run_ranks(n, "cuda", prog, emulate=True).results:
        assert np.array_equal(r, want)


def test_bad_schedule_name_raises():
    def prog(ep):
        with pytest.raises(errors.InvalidConfig):
            allreduce(ep, GradientBuffer.zeros(8, device=ep.torch_device), "multicolor",
                      schedule="butterfly")

    run_ranks(2, "cuda", prog, emulate=True)


@pytest.mark.multigpu
@need_gpus(4)
@pytest.mark.parametrize("case", ["mc_4_4099_1_4", "mc_4_10007_4_4"])
def test_owner_p2p_four_gpus_match_reference(golden, case):
    inp = golden[case + "_in"]
    n, _, k, arity = (int(x) for x in case.split("_")[1:])
    ts = build_multicolor_trees(n, k, arity)
    for r in run(n, list(inp), "multicolor", emulate=False, tree_set=ts):
        assert np.array_equal(r, golden[case + "_out"])
