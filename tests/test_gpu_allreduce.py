"""Allreduce parity on the GPU: every golden case of the reference, bitwise.

Ranks are emulated on one GPU (run_ranks(..., emulate=True): one cooperative
launch serves all ranks) so this runs on a 1-GPU box; the multigpu tests at
the bottom repeat the cases with one GPU per rank over NVLink.
"""

import numpy as np
import pytest
import torch

from paper_1711_00705_b200 import (
    GradientBuffer,
    SgdUpdate,
    allreduce,
    allreduce_multicolor,
    build_multicolor_trees,
    build_ring,
    errors,
    run_ranks,
)
from tests.conftest import need_gpus
from tests.test_oracle import GOLD_MC

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["tree", "oneshot", "ll", "stream", "push"])
def ar_path(request, monkeypatch):
    """Every test runs on each kernel route (md_plan_set_route): the pipelined
    tree schedule (allreduce_channels_kernel / the work-queue kernel), the
    one-shot pull kernel, the LL push kernel, the tiled all-pull stream kernel
    and the owner-push kernel -- all but the tree evaluate the same fold
    programs locally, so the bits must not change. (Calls a route cannot take
    -- worker folds, sizes beyond its range, replicated updates on the push
    route -- fall back to the tree schedule.)"""
    from paper_1711_00705_b200 import collectives

    monkeypatch.setattr(collectives, "_DEFAULT_ROUTE", request.param)
    return request.param


def run(n, arrays, algo, emulate=True, **kw):
    def prog(ep):
        buf = GradientBuffer(torch.from_numpy(arrays[ep.rank].copy()).to(ep.torch_device))
        return allreduce(ep, buf, algo, **kw).data.cpu().numpy()

    return run_ranks(n, "cuda", prog, emulate=emulate).results


@pytest.mark.parametrize("n,L,k,arity", GOLD_MC)
@pytest.mark.parametrize("seg", [64, 16384])
def test_multicolor_matches_reference(golden, n, L, k, arity, seg):
    inp = golden[f"mc_{n}_{L}_{k}_{arity}_in"]
    want = golden[f"mc_{n}_{L}_{k}_{arity}_out"]
    ts = build_multicolor_trees(n, k, arity)
    for r in run(n, list(inp), "multicolor", tree_set=ts, segment_elems=seg):
        assert np.array_equal(r, want)


@pytest.mark.parametrize("n,L", [(8, 1000), (5, 333), (2, 4), (4, 4099)])
def test_ring_matches_reference(golden, n, L):
    out = run(n, list(golden[f"ring_{n}_{L}_in"]), "ring", ring=build_ring(n), segment_elems=100)
    for r in out:
        assert np.array_equal(r, golden[f"ring_{n}_{L}_out"])


@pytest.mark.parametrize("n,L,root", [(8, 513, 0), (4, 100, 2), (4, 4099, 3)])
def test_reduce_bcast_matches_reference(golden, n, L, root):
    for r in run(n, list(golden[f"rb_{n}_{L}_{root}_in"]), "reduce_bcast", root=root):
        assert np.array_equal(r, golden[f"rb_{n}_{L}_{root}_out"])


def test_exact_small_values():
    out = run(2, [np.array([1, 2], np.float32), np.array([10, 20], np.float32)], "multicolor",
              tree_set=build_multicolor_trees(2, 1, 4))
    assert [o.tolist() for o in out] == [[11.0, 22.0], [11.0, 22.0]]
    out = run(8, [np.full(10, r, np.float32) for r in range(8)], "multicolor")
    assert all((o == 28).all() for o in out)


def test_segmentation_does_not_change_bits(golden):
    inp = list(golden["mc_8_10007_4_4_in"])
    ts = build_multicolor_trees(8, 4, 4)
    outs = [run(8, inp, "multicolor", tree_set=ts, segment_elems=s)[3] for s in (1, 17, 250, 1 << 20)]
    for o in outs:
        assert np.array_equal(o, golden["mc_8_10007_4_4_out"])


def test_back_to_back_calls_reuse_flags_safely():
    ts = build_multicolor_trees(4, 4)

    def prog(ep):
        a = allreduce_multicolor(ep, GradientBuffer.of([float(ep.rank)], device=ep.torch_device), ts)
        first = float(a.data[0])
        b = allreduce_multicolor(ep, GradientBuffer.of([first], device=ep.torch_device), ts)
        return float(b.data[0])

    assert run_ranks(4, "cuda", prog, emulate=True).results == [24.0] * 4


def test_oneshot_and_tree_calls_interleave(oracle, monkeypatch):
    """Default thresholds: a 16 KB buffer takes the LL kernel, a 4.8 MB one
    the owner-push kernel (N = 4); alternating them on one communicator keeps
    the epoch protocol (arrival / done flags) consistent and the bits exact."""
    from paper_1711_00705_b200 import collectives

    monkeypatch.setattr(collectives, "_DEFAULT_ROUTE", "auto")
    n = 4
    ts = build_multicolor_trees(n, 4, 4)
    tables = oracle.tables_from_trees(n, oracle.trees(n, 4, 4))
    rng = np.random.default_rng(5)
    small = [rng.standard_normal(4099).astype(np.float32) for _ in range(n)]
    big = [rng.standard_normal(1_200_001).astype(np.float32) for _ in range(n)]
    want_s, want_b = oracle.fold_c(tables, small), oracle.fold_c(tables, big)

    def prog(ep):
        dev = ep.torch_device
        ok = []
        for i in range(5):
            src = small if i % 2 == 0 else big
            buf = GradientBuffer(torch.from_numpy(src[ep.rank].copy()).to(dev))
            allreduce_multicolor(ep, buf, ts)
            ok.append(np.array_equal(buf.data.cpu().numpy(), want_s if i % 2 == 0 else want_b))
        return ok

    for r in run_ranks(n, "cuda", prog, emulate=True).results:
        assert all(r)


@pytest.mark.parametrize("n,k,arity", [(2, 2, 4), (4, 4, 4), (8, 4, 4)])
@pytest.mark.parametrize("tail_in_update", [False, True])
def test_fused_update_without_workers(oracle, n, k, arity, tail_in_update):
    """Allreduce + momentum/wd update, no worker fold: the fused path of every
    kernel (tree epilogue, owner-push own slice + receiver CTAs). A 2.5M + 2
    float buffer; the update covers everything but the 2-element tail, or the
    tail too (then owner-push must hand the call to the tree)."""
    rng = np.random.default_rng(n * 7 + k + int(tail_in_update))
    L = 2_500_002
    P = L - 1 if tail_in_update else L - 2
    arrays = [rng.standard_normal(L).astype(np.float32) for _ in range(n)]
    w0 = rng.standard_normal(P).astype(np.float32)
    m0 = rng.standard_normal(P).astype(np.float32)
    tables = oracle.tables_from_trees(n, oracle.trees(n, k, arity))
    want = oracle.fold_c(tables, arrays)
    want_w, want_m = oracle.sgd_np(w0, want[:P], m0.copy(), 1e-3, 0.9, 3.2e-3)
    ts = build_multicolor_trees(n, k, arity)

    def prog(ep):
        dev = ep.torch_device
        buf = GradientBuffer(torch.from_numpy(arrays[ep.rank].copy()).to(dev))
        w = torch.from_numpy(w0.copy()).to(dev)
        m = torch.from_numpy(m0.copy()).to(dev)
        upd = SgdUpdate(weights=w, c=1e-3, momentum=m, mu=0.9, wd_b=3.2e-3, update_len=P)
        allreduce(ep, buf, "multicolor", tree_set=ts, update=upd)
        return buf.data.cpu().numpy(), w.cpu().numpy(), m.cpu().numpy()

    for g, w, m in run_ranks(n, "cuda", prog, emulate=True).results:
        assert np.array_equal(g, want)
        assert np.array_equal(w, want_w)
        assert np.array_equal(m, want_m)


def test_host_numpy_buffers_are_a_drop_in(golden):
    """Reference callers pass numpy arrays; the result lands back in them."""
    inp = golden["mc_8_997_4_4_in"]
    ts = build_multicolor_trees(8, 4, 4)

    def prog(ep):
        host = inp[ep.rank].copy()
        buf = GradientBuffer(host)
        allreduce_multicolor(ep, buf, ts, segment_elems=64)
        return host

    for r in run_ranks(8, "cuda", prog, emulate=True).results:
        assert np.array_equal(r, golden["mc_8_997_4_4_out"])


def test_mismatched_lengths_raise():
    def prog(ep):
        allreduce(ep, GradientBuffer.zeros(4 if ep.rank else 5, device=ep.torch_device), "ring")

    with pytest.raises(errors.LengthMismatch):
        run_ranks(2, "cuda", prog, emulate=True)


def test_one_rank_identity_and_bad_args():
    res = run_ranks(1, "cuda", lambda ep: allreduce(
        ep, GradientBuffer.of([3.5, 4.5], device=ep.torch_device), "multicolor").data.tolist()).results
    assert res == [[3.5, 4.5]]

    def prog(ep):
        with pytest.raises(errors.InvalidConfig):
            allreduce(ep, GradientBuffer.zeros(4, device=ep.torch_device), "butterfly")
        with pytest.raises(errors.InvalidConfig):
            allreduce_multicolor(ep, GradientBuffer.zeros(4, device=ep.torch_device),
                                 build_multicolor_trees(8, 4))

    run_ranks(4, "cuda", prog, emulate=True)


@pytest.mark.parametrize("n,k,arity", [(4, 4, 4), (8, 4, 4), (8, 8, 7), (2, 1, 4)])
@pytest.mark.parametrize("mu,wd", [(0.0, 0.0), (0.9, 1e-4)])
def test_fused_accumulation_allreduce_and_update(oracle, n, k, arity, mu, wd):
    """Worker fold -> tree fold -> SGD epilogue in ONE launch == the unfused
    reference pipeline (node_gradient, allreduce, sub_scaled_f32 [+ momentum])."""
    rng = np.random.default_rng(n * 100 + k + int(mu * 10))
    P, m = 100_003, 3
    workers = [[rng.standard_normal(P).astype(np.float32) for _ in range(m)] for _ in range(n)]
    w0 = rng.standard_normal(P - 2).astype(np.float32)
    v0 = rng.standard_normal(P - 2).astype(np.float32)
    c, wd_b = 0.1 / 128, float(np.float32(wd * 128))
    tables = oracle.tables_from_trees(n, oracle.trees(n, k, arity))
    folded = []
    for r in range(n):
        acc = workers[r][0].copy()
        for j in range(1, m):
            acc += workers[r][j]
        folded.append(acc)
    g = oracle.fold_c(tables, folded)
    want_w, want_v = oracle.sgd_np(w0, g[: P - 2], v0.copy() if mu else None, c, mu, wd_b)
    ts = build_multicolor_trees(n, k, arity)

    def prog(ep):
        dev = ep.torch_device
        buf = GradientBuffer.alloc(P, ep)
        wk = [torch.from_numpy(x).to(dev) for x in workers[ep.rank]]
        w = torch.from_numpy(w0.copy()).to(dev)
        v = torch.from_numpy(v0.copy()).to(dev)
        upd = SgdUpdate(weights=w, c=c, momentum=v, mu=mu, wd_b=wd_b, update_len=P - 2)
        allreduce(ep, buf, "multicolor", tree_set=ts, workers=wk, update=upd)
        return buf.data.cpu().numpy(), w.cpu().numpy(), v.cpu().numpy()

    for gb, w, v in run_ranks(n, "cuda", prog, emulate=True).results:
        assert np.array_equal(gb, g)
        assert np.array_equal(w, want_w)
        if mu:
            assert np.array_equal(v, want_v)


@pytest.mark.parametrize("case", ["mc_8_10007_4_4", "mc_4_4099_2_4", "mc_16_250_4_4"])
def test_work_queue_kernel_matches_reference(golden, monkeypatch, case):
    """The work-queue kernel (fallback when the channel allotment does not
    fit) folds identically; the "queue" route forces it."""
    from paper_1711_00705_b200 import collectives

    monkeypatch.setattr(collectives, "_DEFAULT_ROUTE", "queue")
    n, _, k, arity = (int(x) for x in case.split("_")[1:])
    ts = build_multicolor_trees(n, k, arity)
    for r in run(n, list(golden[case + "_in"]), "multicolor", tree_set=ts, segment_elems=512):
        assert np.array_equal(r, golden[case + "_out"])


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_unaligned_buffers_take_the_scalar_path(oracle, offset):
    """Buffers that are not 16-byte aligned run the work-queue kernel's scalar
    path (no TMA); bits must not change."""
    n, P = 4, 10_007
    rng = np.random.default_rng(offset)
    arrays = [rng.standard_normal(P).astype(np.float32) for _ in range(n)]
    w0 = rng.standard_normal(P).astype(np.float32)
    tables = oracle.tables_from_trees(n, oracle.trees(n, 4, 4))
    g = oracle.fold_c(tables, arrays)
    want_w, _ = oracle.sgd_np(w0, g, None, 1e-3, 0.0, 0.0)
    ts = build_multicolor_trees(n, 4, 4)

    def prog(ep):
        dev = ep.torch_device
        base = torch.zeros(P + offset, device=dev)
        view = base[offset:]
        view.copy_(torch.from_numpy(arrays[ep.rank]))
        wb = torch.zeros(P + offset, device=dev)
        w = wb[offset:]
        w.copy_(torch.from_numpy(w0))
        allreduce(ep, GradientBuffer(view), "multicolor", tree_set=ts, segment_elems=1000,
                  update=SgdUpdate(weights=w, c=1e-3))
        return view.cpu().numpy(), w.cpu().numpy()

    for gb, w in run_ranks(n, "cuda", prog, emulate=True).results:
        assert np.array_equal(gb, g)
        assert np.array_equal(w, want_w)


@pytest.mark.parametrize("workers", [0, 2])
@pytest.mark.parametrize("mu,wd", [(0.0, 0.0), (0.9, 1e-4)])
def test_single_rank_fused_update(oracle, workers, mu, wd):
    """N = 1: the collective is the identity but the fused epilogue (and the
    worker fold) must still run -- the bench's one-GPU configuration."""
    rng = np.random.default_rng(17)
    P = 1_000_003
    g0 = rng.standard_normal(P).astype(np.float32)
    wk = [rng.standard_normal(P).astype(np.float32) for _ in range(workers)]
    w0 = rng.standard_normal(P - 2).astype(np.float32)
    v0 = rng.standard_normal(P - 2).astype(np.float32)
    c, wd_b = 0.1 / 32, float(np.float32(wd * 32))
    g = g0 if not workers else (wk[0] + wk[1])
    want_w, want_v = oracle.sgd_np(w0, g[: P - 2], v0.copy() if mu else None, c, mu, wd_b)

    def prog(ep):
        dev = ep.torch_device
        buf = GradientBuffer.alloc(P, ep)
        buf.data.copy_(torch.from_numpy(g0))
        w = torch.from_numpy(w0.copy()).to(dev)
        v = torch.from_numpy(v0.copy()).to(dev)
        allreduce(ep, buf, "multicolor",
                  workers=[torch.from_numpy(x).to(dev) for x in wk] or None,
                  update=SgdUpdate(weights=w, c=c, momentum=v, mu=mu, wd_b=wd_b, update_len=P - 2))
        return buf.data.cpu().numpy(), w.cpu().numpy(), v.cpu().numpy()

    gb, w, v = run_ranks(1, "cuda", prog).results[0]
    assert np.array_equal(gb, g)
    assert np.array_equal(w, want_w)
    if mu:
        assert np.array_equal(v, want_v)


@pytest.mark.parametrize("n,k,arity", [(4, 4, 4), (8, 4, 4)])
def test_full_resnet50_size_bitwise(oracle, n, k, arity):
    """25.6M floats (BASELINE config C1 at N=4; C3 tree at N=8), bit-exact."""
    P = 25_600_000
    rng = np.random.default_rng(99)
    arrays = [rng.standard_normal(P, dtype=np.float32) for _ in range(n)]
    want = oracle.fold_c(oracle.tables_from_trees(n, oracle.trees(n, k, arity)), arrays)
    ts = build_multicolor_trees(n, k, arity)

    def prog(ep):
        buf = GradientBuffer.alloc(P, ep)
        buf.data.copy_(torch.from_numpy(arrays[ep.rank]))
        allreduce(ep, buf, "multicolor", tree_set=ts)
        return bool(torch.equal(buf.data.cpu(), torch.from_numpy(want)))

    assert all(run_ranks(n, "cuda", prog, emulate=True).results)


def test_closed_form_check_of_reference_bench_fill(oracle):
    """bench.py's deterministic fill has a closed-form f64 sum: rel err <= 1e-5."""
    import ctypes as C  # noqa: F401

    from paper_1711_00705_b200 import _lib

    P, n = 4_000_000, 8

    def prog(ep):
        buf = GradientBuffer.alloc(P, ep)
        _lib.check(_lib.load().md_fill_rank_input(buf.data.data_ptr(), P, ep.rank, n,
                                                  _lib.stream_ptr(ep.stream)))
        allreduce(ep, buf, "multicolor")
        idx = np.arange(0, P, 997 * 13)
        got = buf.data.cpu().numpy()[idx].astype(np.float64)
        return float(np.max(np.abs(got - oracle.expected_fill_sum(idx, n)) / oracle.expected_fill_sum(idx, n)))

    assert max(run_ranks(n, "cuda", prog, emulate=True).results) <= 1e-5


# -- one GPU per rank (NVLink P2P) --------------------------------------------------------------


@pytest.mark.multigpu
@need_gpus(2)
def test_lost_peer_surfaces_as_not_exposed():
    """A rank that never enters the collective must not hang its peer: the
    device watchdog ends the wait (transport/base.py:28 semantics) and the
    waiting rank raises NotExposed."""
    import time

    from paper_1711_00705_b200.transport import PeerView

    def prog(ep):
        if ep.rank == 1:
            return None  # never enters the collective
        buf = GradientBuffer(torch.ones(1024, device=ep.torch_device))
        # pre-registered view, so the host-side registration (which would fail
        # fast) is skipped and the DEVICE wait is what must time out
        buf.peers = (ep, PeerView([buf.data.data_ptr()] * ep.n_ranks, 4096, buf.data))
        t0 = time.perf_counter()
        try:
            allreduce(ep, buf, "multicolor", tree_set=build_multicolor_trees(2, 1, 4))
        except errors.NotExposed:
            return time.perf_counter() - t0
        return -1.0

    waited = run_ranks(2, "cuda", prog, emulate=False, pull_timeout=2.0).results[0]
    assert waited is not None and 1.5 < waited < 20.0, waited


@pytest.mark.multigpu
@need_gpus(2)
@pytest.mark.parametrize("n,L,k,arity", [(2, 4099, 1, 4), (2, 4099, 2, 4), (2, 0, 2, 4)])
def test_p2p_two_gpus_match_reference(golden, n, L, k, arity):
    inp = golden[f"mc_{n}_{L}_{k}_{arity}_in"]
    ts = build_multicolor_trees(n, k, arity)
    for r in run(n, list(inp), "multicolor", emulate=False, tree_set=ts, segment_elems=64):
        assert np.array_equal(r, golden[f"mc_{n}_{L}_{k}_{arity}_out"])


@pytest.mark.multigpu
@need_gpus(4)
@pytest.mark.parametrize("case", ["mc_4_4099_4_4", "mc_4_10007_4_4", "mc_4_4099_1_4", "mc_4_7_4_4"])
def test_p2p_four_gpus_match_reference(golden, case):
    inp = golden[case + "_in"]
    n, _, k, arity = (int(x) for x in case.split("_")[1:])
    ts = build_multicolor_trees(n, k, arity)
    for r in run(n, list(inp), "multicolor", emulate=False, tree_set=ts):
        assert np.array_equal(r, golden[case + "_out"])
    out = run(4, list(golden["ring_4_4099_in"]), "ring", emulate=False)
    assert all(np.array_equal(o, golden["ring_4_4099_out"]) for o in out)


@pytest.mark.multigpu
@need_gpus(2)
def test_ranks_on_different_routes_fail_together():
    """Two ranks that take different kernels (here pinned: the tree and the
    one-shot pull) must not exchange differently shaped flags: the entry
    barrier compares their route words and both raise InvalidConfig."""
    def prog(ep):
        buf = GradientBuffer.alloc(100_000, ep)
        try:
            allreduce(ep, buf, "multicolor", tree_set=build_multicolor_trees(2, 1, 4),
                      route="tree" if ep.rank == 0 else "oneshot")
        except errors.InvalidConfig:
            return "InvalidConfig"
        return "ok"

    assert run_ranks(2, "cuda", prog, emulate=False, pull_timeout=5.0).results == \
        ["InvalidConfig", "InvalidConfig"]
