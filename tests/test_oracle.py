"""The oracle is pinned against the reference's own outputs (tests/golden)
before anything is checked against it. CPU only."""

import numpy as np
import pytest

GOLD_MC = [(8, 1000, 4, 4), (8, 997, 4, 4), (4, 7, 4, 4), (3, 1, 3, 4), (2, 0, 2, 4),
           (16, 250, 4, 4), (2, 4099, 1, 4), (2, 4099, 2, 4), (4, 4099, 1, 4), (4, 4099, 2, 4),
           (4, 4099, 4, 4), (8, 4099, 1, 4), (8, 4099, 2, 4), (8, 4099, 8, 7),
           (8, 10007, 4, 4), (4, 10007, 4, 4)]


@pytest.mark.parametrize("n,L,k,arity", GOLD_MC)
def test_multicolor_fold_matches_reference(golden, oracle, n, L, k, arity):
    inp = golden[f"mc_{n}_{L}_{k}_{arity}_in"]
    want = golden[f"mc_{n}_{L}_{k}_{arity}_out"]
    tables = oracle.tables_from_trees(n, oracle.trees(n, k, arity))
    arrays = [inp[r] for r in range(n)]
    assert np.array_equal(oracle.fold_numpy(tables, arrays), want)
    assert np.array_equal(oracle.fold_c(tables, arrays), want)


@pytest.mark.parametrize("n,L", [(8, 1000), (5, 333), (2, 4), (4, 4099)])
def test_ring_fold_matches_reference(golden, oracle, n, L):
    inp = golden[f"ring_{n}_{L}_in"]
    tables = oracle.ring_tables(list(range(n)))
    got = oracle.fold_c(tables, [inp[r] for r in range(n)])
    assert np.array_equal(got, golden[f"ring_{n}_{L}_out"])


@pytest.mark.parametrize("n,L,root", [(8, 513, 0), (4, 100, 2), (4, 4099, 3)])
def test_rank_order_fold_matches_reference(golden, oracle, n, L, root):
    inp = golden[f"rb_{n}_{L}_{root}_in"]
    tables = oracle.star_tables(n, root)
    arrays = [inp[r] for r in range(n)]
    assert np.array_equal(oracle.fold_numpy(tables, arrays), golden[f"rb_{n}_{L}_{root}_out"])
    assert np.array_equal(oracle.fold_c(tables, arrays), golden[f"rb_{n}_{L}_{root}_out"])


def test_float_kernels_match_reference(golden, oracle):
    a, b = golden["kern_a"], golden["kern_b"]
    d = a.copy()
    oracle.lib().mo_add_f32(oracle._f32p(d), oracle._f32p(b), len(d))
    assert np.array_equal(d, golden["kern_add"])
    for c, want in zip(golden["kern_c"], golden["kern_sub"]):
        assert np.array_equal(oracle.sub_scaled_np(a, b, c), want)
        d = a.copy()
        oracle.lib().mo_sub_scaled_f32(oracle._f32p(d), oracle._f32p(b), len(d), float(c))
        assert np.array_equal(d, want)


def test_reference_compiled_kernels_agree(golden, oracle):
    acc = oracle.ref_accel()
    if acc is None:
        pytest.skip("oracle/_ref not built (reference tree absent when it was built)")
    a, b = golden["kern_a"], golden["kern_b"]
    for c, want in zip(golden["kern_c"], golden["kern_sub"]):
        d = a.copy()
        acc.sub_scaled_f32(d, b, float(c))
        assert np.array_equal(d, want)


def test_sgd_extension_reduces_to_reference_update(golden, oracle):
    a, b = golden["kern_a"], golden["kern_b"]
    for c, want in zip(golden["kern_c"], golden["kern_sub"]):
        w, _ = oracle.sgd_np(a, b, None, c, 0.0, 0.0)
        assert np.array_equal(w, want)
        w2 = a.copy()
        oracle.lib().mo_sgd_update(oracle._f32p(w2), oracle._f32p(b), None, len(w2), float(np.float32(c)), 0.0, 0.0)
        assert np.array_equal(w2, want)


def test_sgd_momentum_c_matches_numpy(oracle):
    rng = np.random.default_rng(3)
    w = rng.standard_normal(5000).astype(np.float32)
    g = rng.standard_normal(5000).astype(np.float32)
    v = rng.standard_normal(5000).astype(np.float32)
    for mu, wd in [(0.9, 0.0), (0.9, 1e-4 * 256), (0.0, 1e-4 * 256)]:
        want_w, want_v = oracle.sgd_np(w, g, v.copy() if mu else None, 0.01, mu, wd)
        w2, v2 = w.copy(), v.copy()
        oracle.lib().mo_sgd_update(oracle._f32p(w2), oracle._f32p(g),
                                   oracle._f32p(v2) if mu else None, len(w2), 0.01, mu,
                                   float(np.float32(wd)))
        assert np.array_equal(w2, want_w)
        if mu:
            assert np.array_equal(v2, want_v)


def test_mix64_matches_reference(golden, oracle):
    for parts, n, want in zip(golden["mix64_parts"], golden["mix64_n"], golden["mix64_out"]):
        assert oracle.mix64(*[int(x) for x in parts[:n]]) == int(want)


@pytest.mark.parametrize("n", [1, 2, 3, 7, 8, 1000, 160000, (1 << 31) + 5, (1 << 32) - 1])
def test_integers_c_restatement_matches_numpy(oracle, n):
    for key in (0, 1, 0xDEADBEEF, (1 << 64) - 1):
        assert np.array_equal(oracle.integers_c(key, n, 300), oracle.integers_np(key, n, 300))


@pytest.mark.parametrize("n", [0, 1, 2, 5, 100, 4097, 65537])
def test_permutation_c_restatement_matches_numpy(oracle, n):
    for key in (3, 77, (1 << 63) + 11):
        assert np.array_equal(oracle.permutation_c(key, n), oracle.permutation_np(key, n))


def test_random_batch_picks_match_reference(golden, oracle):
    from paper_1711_00705_b200.dimd import _parse_table

    table = _parse_table(golden["rb_index"].tobytes())
    pos = 0
    for seed, size in zip(golden["rb_seeds"], golden["rb_sizes"]):
        want = golden["rb_picks"][pos : pos + size]
        pos += size
        assert np.array_equal(oracle.random_batch_picks(int(seed), len(table), int(size)), want)
        assert np.array_equal(oracle.integers_c(int(seed), len(table), int(size)), want)


SHUFFLES = ["sh_a", "sh_b", "sh_c", "sh_d", "sh_e", "sh_f", "sh_g"]


@pytest.mark.parametrize("name", SHUFFLES)
def test_shuffle_plan_matches_reference(golden, oracle, name):
    nrec, nr, gs, m, seed = (int(x) for x in golden[name + "_meta"])
    counts = golden[name + "_counts"]
    ids = golden[name + "_ids"]
    pos = 0
    for rank in range(nr):
        member, gid = rank % gs, rank // gs
        n_rec = [len(range(q, nrec, gs)) for q in range(gs)]
        for plan in (oracle.shuffle_plan_np, oracle.shuffle_plan_c):
            mem, rec = plan(seed, gid, gs, member, rank, m, n_rec)
            assert len(mem) == counts[rank]
            assert np.array_equal(mem + gs * rec, ids[pos : pos + counts[rank]])
        pos += counts[rank]


def test_sgd_replay_through_oracle_matches_reference(golden, oracle):
    """12 distributed steps of the reference's train_step (N=4, m=2, k=4):
    worker fold + multicolor fold + sub_scaled update reproduce its weights."""
    n, m, k, _, p = (int(x) for x in golden["sgd_cfg"])
    workers = golden["sgd_workers"]  # [rank, step, worker, p+2]
    tables = oracle.tables_from_trees(n, oracle.trees(n, 4, 4))
    w = golden["sgd_w0"].copy()
    B = n * m * k
    for step in range(workers.shape[1]):
        bufs = []
        for r in range(n):
            acc = workers[r, step, 0].copy()
            for j in range(1, m):
                acc += workers[r, step, j]
            bufs.append(acc)
        g = oracle.fold_c(tables, bufs)
        w = oracle.sub_scaled_np(w, g[:p], golden["sgd_lr"][step] / B)
        assert np.array_equal(w, golden["sgd_weights"][step]), step
