"""C3/C5-size fused parity: the 25.6M-float ResNet-50 gradient (+2 metric
slots, ref sgd.py:345-348) through ONE fused allreduce + SGD momentum 0.9 /
weight decay 1e-4 update, bitwise against the oracle (its C fold in the
reference's per-color order, ref collectives.py:271-296, and its float32
update restatement), on the route md_allreduce picks by default -- which the
tests assert through md_last_route:

* replicated update: N = 4 -> the channelized tree kernel (k = 4); N = 8
  emulated -> the tree kernel with k = 4 / arity 4 (the paper's Fig. 2 trees)
  and k = 8 / arity 7; two calls back to back, so the second reuses every flag
  at the next epoch;
* sharded update (SgdUpdate(sharded=True), md_allreduce_ex): the owner-push
  kernel; the weights must be bitwise the replicated ones on EVERY rank, the
  momentum and the sum on each rank's own slice.

Ranks are emulated on one GPU here; the multigpu tests repeat N = 4 with one
GPU per rank (threads, NVLink P2P).
"""

import numpy as np
import pytest
import torch

from paper_1711_00705_b200 import GradientBuffer, _lib, build_multicolor_trees, run_ranks
from paper_1711_00705_b200.collectives import SgdUpdate, allreduce
from tests.conftest import need_gpus

pytestmark = pytest.mark.gpu

P = 25_600_000
L = P + 2
MU, WD, LR = 0.9, 1e-4, 0.1


def _push_slice(n_elems: int, n: int, j: int) -> tuple[int, int]:
    """push_slice (csrc/md_allreduce.cuh): 16-byte aligned owner slice j."""
    n4 = n_elems & ~3
    per = ((n4 // 4 + n - 1) // n) * 4
    return min(n4, j * per), min(n4, (j + 1) * per)


@pytest.fixture(autouse=True)
def _auto_route(monkeypatch):
    from paper_1711_00705_b200 import collectives

    monkeypatch.setattr(collectives, "_DEFAULT_ROUTE", "auto")


def _case(oracle, n, k, arity, seed, steps):
    rng = np.random.default_rng(seed)
    arrays = [rng.standard_normal(L, dtype=np.float32) for _ in range(n)]
    w0 = (rng.standard_normal(P, dtype=np.float32) * np.float32(0.01)).astype(np.float32)
    m0 = np.zeros(P, np.float32)
    B = 32 * n
    c = float(np.float32(LR / B))
    wd_b = float(np.float32(WD * B))
    g = oracle.fold_c(oracle.tables_from_trees(n, oracle.trees(n, k, arity)), arrays)
    w, m = w0, m0
    for _ in range(steps):
        w, m = oracle.sgd_np(w, g[:P], m.copy(), c, MU, wd_b)
    return arrays, w0, c, wd_b, g, w, m


def _prog(arrays, w0, c, wd_b, ts, steps, sharded):
    def prog(ep):
        dev = ep.torch_device
        if sharded:  # peer-registered weights (ep.view_of would do it on first use too)
            w, _ = ep.alloc(P)
            w.copy_(torch.from_numpy(w0))
        else:
            w = torch.from_numpy(w0).to(dev)
        m = torch.zeros(P, device=dev)
        buf = GradientBuffer.alloc(L, ep)
        for _ in range(steps):
            buf.data.copy_(torch.from_numpy(arrays[ep.rank]))
            upd = SgdUpdate(weights=w, c=c, momentum=m, mu=MU, wd_b=wd_b, update_len=P,
                            sharded=sharded)
            allreduce(ep, buf, "multicolor", tree_set=ts, update=upd)
        route = _lib.last_route(ep.device)
        return buf.data.cpu().numpy(), w.cpu().numpy(), m.cpu().numpy(), route

    return prog


def _check(results, n, g, want_w, want_m, sharded, route):
    for r, (gb, w, m, got_route) in enumerate(results):
        assert got_route[0] == route and got_route[2] == sharded, got_route
        assert np.array_equal(w, want_w), f"rank {r}: weights differ"
        if sharded:
            lo, hi = _push_slice(L, n, r)
            assert np.array_equal(m[lo:min(hi, P)], want_m[lo:min(hi, P)]), f"rank {r}: momentum"
            assert np.array_equal(gb[lo:hi], g[lo:hi]), f"rank {r}: own slice of the sum"
            assert np.array_equal(gb[P:], g[P:]), f"rank {r}: metric slots"
        else:
            assert np.array_equal(m, want_m), f"rank {r}: momentum differs"
            assert np.array_equal(gb, g), f"rank {r}: sum differs"


@pytest.mark.parametrize("n,k,arity,sharded,route", [
    (4, 4, 4, False, "tree"),
    (4, 4, 4, True, "push"),
    (8, 4, 4, False, "tree"),
    (8, 8, 7, False, "tree"),
    (8, 4, 4, True, "push"),
    (2, 2, 4, True, "push"),
])
def test_c5_fused_emulated(oracle, n, k, arity, sharded, route):
    arrays, w0, c, wd_b, g, want_w, want_m = _case(oracle, n, k, arity, 100 + n + k, steps=2)
    ts = build_multicolor_trees(n, k, arity)
    res = run_ranks(n, "cuda", _prog(arrays, w0, c, wd_b, ts, 2, sharded), emulate=True).results
    _check(res, n, g, want_w, want_m, sharded, route)


def test_sharded_falls_back_to_replicated_when_unaligned(oracle):
    """update_len % 4 != 0: the sharded request runs replicated (a superset:
    same weights, full momentum, full sum) -- md_allreduce_ex's contract."""
    n, Pn = 4, 1_000_003
    rng = np.random.default_rng(3)
    arrays = [rng.standard_normal(Pn + 2).astype(np.float32) for _ in range(n)]
    w0 = rng.standard_normal(Pn).astype(np.float32)
    g = oracle.fold_c(oracle.tables_from_trees(n, oracle.trees(n, 4, 4)), arrays)
    want_w, want_m = oracle.sgd_np(w0, g[:Pn], np.zeros(Pn, np.float32), 1e-3, MU, 3.2e-3)
    ts = build_multicolor_trees(n, 4, 4)

    def prog(ep):
        w, _ = ep.alloc(Pn)
        w.copy_(torch.from_numpy(w0))
        m = torch.zeros(Pn, device=ep.torch_device)
        buf = GradientBuffer(torch.from_numpy(arrays[ep.rank]).to(ep.torch_device))
        allreduce(ep, buf, "multicolor", tree_set=ts,
                  update=SgdUpdate(weights=w, c=1e-3, momentum=m, mu=MU, wd_b=3.2e-3,
                                   update_len=Pn, sharded=True))
        return buf.data.cpu().numpy(), w.cpu().numpy(), m.cpu().numpy(), _lib.last_route(ep.device)

    for gb, w, m, route in run_ranks(n, "cuda", prog, emulate=True).results:
        assert not route[2]
        assert np.array_equal(gb, g) and np.array_equal(w, want_w) and np.array_equal(m, want_m)


@pytest.mark.multigpu
@need_gpus(4)
@pytest.mark.parametrize("sharded,route", [(False, "tree"), (True, "push")])
def test_c5_fused_four_gpus(oracle, sharded, route):
    """One GPU per rank over NVLink (threads of one process), the C5 call
    twice back to back."""
    arrays, w0, c, wd_b, g, want_w, want_m = _case(oracle, 4, 4, 4, 7, steps=2)
    ts = build_multicolor_trees(4, 4, 4)
    res = run_ranks(4, "cuda", _prog(arrays, w0, c, wd_b, ts, 2, sharded), emulate=False).results
    _check(res, 4, g, want_w, want_m, sharded, route)


@pytest.mark.multigpu
@need_gpus(2)
def test_c5_sharded_two_gpus(oracle):
    arrays, w0, c, wd_b, g, want_w, want_m = _case(oracle, 2, 2, 4, 9, steps=2)
    ts = build_multicolor_trees(2, 2, 4)
    res = run_ranks(2, "cuda", _prog(arrays, w0, c, wd_b, ts, 2, True), emulate=False).results
    _check(res, 2, g, want_w, want_m, True, "push")


@pytest.mark.parametrize("n,L,ulen,algo", [
    (2, 4099, 4096, "multicolor"),      # update covers all but the unaligned tail
    (4, 100_003, 50_000, "multicolor"),  # half the buffer past the update range
    (4, 100_004, 0, "multicolor"),      # empty update range: a plain push
    (3, 65_537, 32_768, "ring"),        # ring fold programs, odd world size
    (8, 200_002, 199_996, "reduce_bcast"),
])
def test_sharded_update_edges(oracle, n, L, ulen, algo):
    """Sharded update where the update range ends inside the push slices: W'
    is pushed for [0, ulen), the plain sum for [ulen, n) -- on every rank --
    and each rank's own slice of the sum and of the momentum is exact."""
    from paper_1711_00705_b200.topology import build_ring

    rng = np.random.default_rng(n * 1000 + L)
    arrays = [rng.standard_normal(L).astype(np.float32) for _ in range(n)]
    w0 = rng.standard_normal(max(ulen, 1)).astype(np.float32)
    m0 = rng.standard_normal(max(ulen, 1)).astype(np.float32)
    if algo == "multicolor":
        tables = oracle.tables_from_trees(n, oracle.trees(n, min(n, 4), 4))
        kw = {"tree_set": build_multicolor_trees(n, min(n, 4), 4)}
    elif algo == "ring":
        tables = oracle.ring_tables(list(range(n)))
        kw = {"ring": build_ring(n)}
    else:
        tables = oracle.star_tables(n, 0)
        kw = {"root": 0}
    g = oracle.fold_c(tables, arrays)

    def prog(ep):
        dev = ep.torch_device
        w, _ = ep.alloc(max(ulen, 1))
        w.copy_(torch.from_numpy(w0))
        m = torch.from_numpy(m0.copy()).to(dev)
        buf = GradientBuffer(torch.from_numpy(arrays[ep.rank]).to(dev))
        allreduce(ep, buf, algo, update=SgdUpdate(weights=w, c=1e-3, momentum=m, mu=MU,
                                                  wd_b=3.2e-3, update_len=ulen, sharded=True),
                  **kw)
        return buf.data.cpu().numpy(), w.cpu().numpy(), m.cpu().numpy(), _lib.last_route(ep.device)

    res = run_ranks(n, "cuda", prog, emulate=True).results
    want_w, want_m = oracle.sgd_np(w0[:ulen], g[:ulen], m0[:ulen].copy(), 1e-3, MU, 3.2e-3)
    for r, (gb, w, m, route) in enumerate(res):
        assert route[0] == "push" and route[2], route
        assert np.array_equal(w[:ulen], want_w), f"rank {r}: weights"
        assert np.array_equal(gb[ulen:], g[ulen:]), f"rank {r}: sum past the update range"
        lo, hi = _push_slice(L, n, r)
        assert np.array_equal(gb[lo:hi], g[lo:hi]), f"rank {r}: own slice of the sum"
        a, b = lo, min(hi, ulen)
        if b > a:
            assert np.array_equal(m[a:b], want_m[a:b]), f"rank {r}: own momentum"


@pytest.mark.parametrize("seed", range(6))
def test_sharded_update_random_shapes(oracle, seed):
    """Random world sizes, color counts, buffer lengths (ragged tails) and
    update ranges: the sharded owner-push update gives the oracle's weights
    on every rank, and each rank's own slices of the sum and the momentum."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 7))
    ks = [k for k in (1, 2, 4, 8) if k <= n]
    k = int(rng.choice(ks))
    arity = 7 if k == 8 else 4
    try:
        ts = build_multicolor_trees(n, k, arity)
    except Exception:  # noqa: BLE001  (unconstructible shape: fall back to one color)
        k, ts = 1, build_multicolor_trees(n, 1, 4)
    L = int(rng.integers(1_000, 400_000))
    ulen = int(rng.integers(0, L + 1)) & ~3
    arrays = [rng.standard_normal(L).astype(np.float32) for _ in range(n)]
    w0 = rng.standard_normal(max(ulen, 1)).astype(np.float32)
    m0 = rng.standard_normal(max(ulen, 1)).astype(np.float32)
    g = oracle.fold_c(oracle.tables_from_trees(n, oracle.trees(n, k, arity if k > 1 else 4)),
                      arrays)
    want_w, want_m = oracle.sgd_np(w0[:ulen], g[:ulen], m0[:ulen].copy(), 1e-3, MU, 3.2e-3)

    def prog(ep):
        w, _ = ep.alloc(max(ulen, 1))
        w.copy_(torch.from_numpy(w0))
        m = torch.from_numpy(m0.copy()).to(ep.torch_device)
        buf = GradientBuffer(torch.from_numpy(arrays[ep.rank]).to(ep.torch_device))
        allreduce(ep, buf, "multicolor", tree_set=ts,
                  update=SgdUpdate(weights=w, c=1e-3, momentum=m, mu=MU, wd_b=3.2e-3,
                                   update_len=ulen, sharded=True))
        return buf.data.cpu().numpy(), w.cpu().numpy(), m.cpu().numpy(), _lib.last_route(ep.device)

    for r, (gb, w, m, route) in enumerate(run_ranks(n, "cuda", prog, emulate=True).results):
        assert route[0] == "push" and route[2], (n, k, L, ulen, route)
        assert np.array_equal(w[:ulen], want_w), (n, k, L, ulen, r)
        assert np.array_equal(gb[ulen:], g[ulen:]), (n, k, L, ulen, r)
        lo, hi = _push_slice(L, n, r)
        assert np.array_equal(gb[lo:hi], g[lo:hi]), (n, k, L, ulen, r)
        if min(hi, ulen) > lo:
            assert np.array_equal(m[lo:min(hi, ulen)], want_m[lo:min(hi, ulen)])
