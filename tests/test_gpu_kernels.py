"""Operator seam on the GPU vs the reference's outputs and the oracle (bit-exact)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_1711_00705_b200 import _kernels

    assert _kernels.BACKEND == "cuda"
    return _kernels


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_add_matches_reference(golden, K):
    d, s = cuda(golden["kern_a"]), cuda(golden["kern_b"])
    K.add_f32(d, s)
    assert np.array_equal(d.cpu().numpy(), golden["kern_add"])


def test_sub_scaled_matches_reference(golden, K):
    for c, want in zip(golden["kern_c"], golden["kern_sub"]):
        d = cuda(golden["kern_a"])
        K.sub_scaled_f32(d, cuda(golden["kern_b"]), float(c))
        assert np.array_equal(d.cpu().numpy(), want), c


@pytest.mark.parametrize("off_d,off_s", [(0, 0), (1, 1), (3, 3), (1, 2), (0, 3)])
def test_unaligned_views_and_tails(K, off_d, off_s):
    rng = np.random.default_rng(off_d * 7 + off_s)
    n = 100_003
    a = rng.standard_normal(n + 8).astype(np.float32)
    b = rng.standard_normal(n + 8).astype(np.float32)
    da, db = cuda(a), cuda(b)
    dv, sv = da[off_d : off_d + n], db[off_s : off_s + n]
    K.add_f32(dv, sv)
    want = a.copy()
    want[off_d : off_d + n] = a[off_d : off_d + n] + b[off_s : off_s + n]
    assert np.array_equal(da.cpu().numpy(), want)
    K.sub_scaled_f32(dv, sv, 0.0123)
    want[off_d : off_d + n] = want[off_d : off_d + n] - np.float32(0.0123) * b[off_s : off_s + n]
    assert np.array_equal(da.cpu().numpy(), want)


def test_full_size_update_bitwise(K):
    """25.6M floats: the ResNet-50 gradient size of BASELINE.json."""
    rng = np.random.default_rng(11)
    n = 25_600_000
    w = rng.standard_normal(n, dtype=np.float32)
    g = rng.standard_normal(n, dtype=np.float32)
    dw = cuda(w)
    K.sub_scaled_f32(dw, cuda(g), 0.1 / 256)
    assert np.array_equal(dw.cpu().numpy(), w - np.float32(0.1 / 256) * g)


def test_length_mismatch_and_empty(K):
    with pytest.raises(ValueError):
        K.add_f32(torch.zeros(3, device="cuda"), torch.zeros(4, device="cuda"))
    with pytest.raises(ValueError):
        K.sub_scaled_f32(torch.zeros(4, device="cuda"), torch.zeros(3, device="cuda"), 1.0)
    e = torch.zeros(0, device="cuda")
    K.add_f32(e, e)
    K.sub_scaled_f32(e, e, 2.0)


def test_no_cpu_fallback(K):
    with pytest.raises(TypeError):
        K.add_f32(np.zeros(4, np.float32), np.zeros(4, np.float32))


@pytest.mark.parametrize("mu,wd", [(0.9, 0.0), (0.9, 1e-4), (0.0, 1e-4), (0.0, 0.0)])
def test_sgd_momentum_weight_decay_matches_oracle(K, oracle, mu, wd):
    rng = np.random.default_rng(5)
    n = 1_000_003
    w = rng.standard_normal(n, dtype=np.float32)
    g = rng.standard_normal(n, dtype=np.float32)
    v = rng.standard_normal(n, dtype=np.float32)
    c, wd_b = 0.1 / 256, float(np.float32(wd * 256))
    want_w, want_v = oracle.sgd_np(w, g, v.copy() if mu else None, c, mu, wd_b)
    dw, dv = cuda(w), cuda(v)
    K.sgd_update(dw, cuda(g), dv, c=c, mu=mu, wd_b=wd_b)
    assert np.array_equal(dw.cpu().numpy(), want_w)
    if mu:
        assert np.array_equal(dv.cpu().numpy(), want_v)


def test_fill_rank_input_matches_reference_bench(oracle):
    import ctypes as C

    from paper_1711_00705_b200 import _lib

    for rank, n_ranks in [(0, 1), (3, 8), (1, 4)]:
        t = torch.empty(1_000_000, dtype=torch.float32, device="cuda")
        _lib.check(_lib.load().md_fill_rank_input(t.data_ptr(), t.numel(), rank, n_ranks, None))
        assert np.array_equal(t.cpu().numpy(), oracle.fill_rank_input(t.numel(), rank, n_ranks))
    assert C  # keep import
