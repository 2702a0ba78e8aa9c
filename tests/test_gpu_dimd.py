"""DIMD on the GPU: random_batch and shuffle indices bit-exact with the
reference (golden), index parity at the full C4 corpus size, and the P2P
record exchange checked byte for byte on a synthetic corpus."""

import numpy as np
import pytest
import torch

from paper_1711_00705_b200 import dimd, errors, run_ranks
from paper_1711_00705_b200.dimd import (
    BatchRequest,
    parse_index,
    random_batch,
    random_batch_device,
    shard_from_bytes,
    shuffle_all,
    shuffle_group,
)

pytestmark = pytest.mark.gpu


def ids_of(records):
    return np.array([int.from_bytes(r.bytes[:4], "little") for r in records], np.int64)


def test_random_batch_matches_reference(golden):
    blob = golden["rb_blob"].tobytes()
    entries = parse_index(golden["rb_index"].tobytes())
    store = shard_from_bytes(blob, entries, 0, 1, 1, device=torch.device("cuda", 0))
    pos = 0
    for seed, size in zip(golden["rb_seeds"], golden["rb_sizes"]):
        want = golden["rb_picks"][pos : pos + size]
        pos += size
        got = random_batch(store, BatchRequest(int(size), int(seed)))
        assert np.array_equal(ids_of(got), want)
        picks = dimd.random_batch_picks(store, BatchRequest(int(size), int(seed)))
        assert np.array_equal(picks.cpu().numpy(), want)


def test_random_batch_edge_cases():
    dev = torch.device("cuda", 0)
    one = shard_from_bytes(b"zz", [dimd.IndexEntry(0, 2, 9)], 0, 1, 1, device=dev)
    assert random_batch(one, BatchRequest(4, 1)) == [dimd.Record(b"zz", 9)] * 4
    empty = shard_from_bytes(b"", [], 0, 1, 1, device=dev)
    with pytest.raises(errors.EmptyShard):
        random_batch(empty, BatchRequest(1, 0))


def test_random_batch_large_n_and_fixed_size_gather(oracle):
    dev = torch.device("cuda", 0)
    n, L = 160_000, 512
    st = dimd.synth_store(n, L, 3, 8, 1234, 0, 8, 3, device=dev)
    for key in (7, 2**63 + 5, oracle.mix64(0, oracle.SAMP_ROLE, 5, 17)):
        recs, labels, picks = random_batch_device(st, BatchRequest(32, key), L)
        want = oracle.random_batch_picks(key, n, 32)
        assert np.array_equal(picks.cpu().numpy(), want)
        gids = recs[:, :8].contiguous().view(torch.int64).flatten().cpu().numpy()
        assert np.array_equal(gids, 3 + 8 * want)
    # uniformity (pkg/tests/test_dimd.py:198-205): 3 sigma on 100000 draws over 10
    st10 = dimd.synth_store(10, 16, 0, 1, 5, 0, 1, 0, device=dev)
    p = dimd.random_batch_picks(st10, BatchRequest(100_000, 5)).cpu().numpy()
    freq = np.bincount(p, minlength=10)
    assert np.all(np.abs(freq - 10_000) < 3 * (100_000 * 0.09) ** 0.5)


@pytest.fixture(params=["push", "pull"])
def exchange(request, monkeypatch):
    """Both data movements of the shuffle (md_shuffle_push / md_shuffle_pull)
    place every byte identically."""
    monkeypatch.setattr(dimd, "EXCHANGE", request.param)
    return request.param


@pytest.mark.parametrize("name", ["sh_a", "sh_b", "sh_c", "sh_d", "sh_e", "sh_f", "sh_g"])
def test_shuffle_matches_reference(golden, name, exchange):
    nrec, nr, gs, m, seed = (int(x) for x in golden[name + "_meta"])
    blob = golden[name + "_blob"].tobytes()
    entries = parse_index(golden[name + "_index"].tobytes())
    fn = shuffle_group if name in ("sh_b", "sh_g") else shuffle_all

    def body(ep):
        st = shard_from_bytes(blob, entries, ep.rank, ep.n_ranks, gs, device=ep.torch_device)
        out = fn(ep, st, m_segments=m, seed=seed)
        recs = out.records()
        return ids_of(recs), np.array([r.label for r in recs], np.int64)

    res = run_ranks(nr, "cuda", body, emulate=True).results
    assert np.array_equal(np.array([len(r[0]) for r in res]), golden[name + "_counts"])
    assert np.array_equal(np.concatenate([r[0] for r in res]), golden[name + "_ids"])
    assert np.array_equal(np.concatenate([r[1] for r in res]), golden[name + "_labels"])


def test_shuffle_all_equals_shuffle_group(golden, exchange):
    blob = golden["sh_b_blob"].tobytes()
    entries = parse_index(golden["sh_b_index"].tobytes())

    def body(fn):
        def prog(ep):
            st = shard_from_bytes(blob, entries, ep.rank, ep.n_ranks, 2, device=ep.torch_device)
            return ids_of(fn(ep, st, m_segments=2, seed=5).records())
        return prog

    a = run_ranks(4, "cuda", body(shuffle_all), emulate=True).results
    g = run_ranks(4, "cuda", body(shuffle_group), emulate=True).results
    assert all(np.array_equal(x, y) for x, y in zip(a, g))


def test_shuffle_rejects_mismatched_group_shape():
    def prog(ep):
        st = dimd.synth_store(4, 16, ep.rank, 6, 1, ep.rank // 3, 3, ep.rank % 3,
                              device=ep.torch_device)
        with pytest.raises(errors.GroupMismatch):
            shuffle_all(ep, st, seed=1)

    run_ranks(4, "cuda", prog, emulate=True)


@pytest.mark.parametrize("member", [0, 3, 7])
def test_full_size_index_parity_c4(oracle, member):
    """C4: 1.28M records over 8 ranks (160,000 each), m = 23 segments --
    every output slot's source is bit-exact with the reference algorithm."""
    n_rec = [160_000] * 8
    seed = oracle.mix64(0, oracle.SHUF_ROLE, 0)
    fm, fr = dimd.shuffle_plan_device(seed, 0, 8, member, member, 23, n_rec)
    wm, wr = oracle.shuffle_plan_c(seed, 0, 8, member, member, 23, n_rec)
    assert np.array_equal(fm.cpu().numpy(), wm)
    assert np.array_equal(fr.cpu().numpy(), wr)


def test_index_parity_non_power_of_two_group(oracle):
    """S = 3 and 7 exercise Lemire rejection (and its serial fallback)."""
    for S, n in [(3, 50_001), (7, 30_011), (5, 1)]:
        n_rec = [n + q for q in range(S)]
        for member in (0, S - 1):
            fm, fr = dimd.shuffle_plan_device(99, 2, S, member, 2 * S + member, 4, n_rec)
            wm, wr = oracle.shuffle_plan_c(99, 2, S, member, 2 * S + member, 4, n_rec)
            assert np.array_equal(fm.cpu().numpy(), wm) and np.array_equal(fr.cpu().numpy(), wr)


def test_exchange_moves_every_byte(oracle, exchange):
    """8 emulated ranks x 20,000 synthetic 4 KiB records: after the P2P
    shuffle every record is intact, in the reference's order, none lost."""
    n_local, L, seed, S = 20_000, 4096, 4242, 8

    def prog(ep):
        st = dimd.synth_store(n_local, L, ep.rank, S, seed, 0, S, ep.rank, device=ep.torch_device)
        out = shuffle_all(ep, st, m_segments=3, seed=77)
        bad, gids = dimd.synth_verify(out, seed)
        return bad, gids.cpu().numpy()

    res = run_ranks(S, "cuda", prog, emulate=True).results
    assert all(b == 0 for b, _ in res)
    allg = np.sort(np.concatenate([g for _, g in res]))
    assert np.array_equal(allg, np.arange(S * n_local))
    for r, (_, g) in enumerate(res):
        wm, wr = oracle.shuffle_plan_c(77, 0, S, r, r, 3, [n_local] * S)
        assert np.array_equal(g, wm + S * wr)


def test_batch_stream_matches_keyed_batches_eager_and_graph():
    """BatchStream (device step counter) draws exactly sample_node_batch's
    per-step batches, eagerly and from replays of one captured CUDA graph."""
    from paper_1711_00705_b200.dimd import BatchRequest, BatchStream, _mix64, random_batch_device
    from paper_1711_00705_b200.sgd import SAMPLE_ROLE

    dev = torch.device("cuda", 0)
    store = dimd.synth_store(5000, 96, 0, 1, 7, 0, 1, 0, device=dev)
    bs = BatchStream(store, 32, 96, 7, SAMPLE_ROLE, 3, start_step=5)

    def want(step):
        recs, labels, picks = random_batch_device(store, BatchRequest(32, _mix64(7, SAMPLE_ROLE, 3, step)), 96)
        return recs.clone(), labels.clone(), picks.clone()

    for step in (5, 6):
        got = [t.clone() for t in bs.next()]
        for g, w in zip(got, want(step)):
            assert torch.equal(g, w)
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        bs.next()
    assert int(bs.step.item()) == 7  # capture does not execute
    for step in (7, 8, 9):
        graph.replay()
        torch.cuda.synchronize(dev)
        for g, w in zip((bs.slots.records, bs.slots.labels, bs.slots.picks), want(step)):
            assert torch.equal(g, w)
    bs.slots.check()
    with pytest.raises(errors.InvalidConfig):
        BatchStream(store, 2000, 96, 7, SAMPLE_ROLE, 0)


@pytest.mark.parametrize("lead", [0, 7])
def test_fixed_size_gather_multichunk_records(lead):
    """The gather kernel on multi-chunk records (ragged last chunk, unaligned
    sources after a 7-byte record) is byte-equal with the host copy of the
    picked records, and a picked record of the wrong size raises on check()."""
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(11 + lead)
    L = 2 * 32768 + 1040  # three chunks, the last one ragged (multiple of 16)
    recs = ([dimd.Record(b"x" * lead, 999)] if lead else []) + [
        dimd.Record(rng.bytes(L), int(i)) for i in range(300)]
    blob, idx = dimd.build_blob(recs)
    st = shard_from_bytes(blob, parse_index(idx), 0, 1, 1, device=dev)
    picks = torch.tensor([i + (1 if lead else 0) for i in rng.integers(0, 300, 700)],
                         dtype=torch.int64, device=dev)
    slots = dimd.BatchSlots(700, L, dev)
    slots.picks.copy_(picks)
    dimd._gather_fixed(st, slots, 700, L)
    torch.cuda.synchronize(dev)
    slots.check()
    host = np.stack([np.frombuffer(recs[int(p)].bytes, np.uint8) for p in picks.cpu()])
    assert np.array_equal(slots.records.cpu().numpy(), host)
    assert slots.labels.cpu().tolist() == [recs[int(p)].label for p in picks.cpu()]
    if lead:
        bad = dimd.BatchSlots(700, L, dev)
        bad.picks.copy_(picks)
        bad.picks[3] = 0
        dimd._gather_fixed(st, bad, 700, L)
        with pytest.raises(errors.LengthMismatch):
            bad.check()


@pytest.mark.parametrize("n", [2**31 + 1, 3 * 2**30, 160_000])
def test_picks_rejection_heavy_streams(oracle, n):
    """Ranges where numpy's Lemire rejects ~50 % / 25 % of words: every picks
    kernel (one-CTA batch, graph step counter, multi-CTA + block fix-up)
    reproduces Generator(Philox(key)).integers(0, n, batch) exactly."""
    from paper_1711_00705_b200 import _lib
    from paper_1711_00705_b200.dimd import _mix64

    lib = _lib.load()
    dev = torch.device("cuda", 0)
    sp = _lib.stream_ptr(torch.cuda.current_stream(dev))
    for key, batch in ((11, 700), (2**64 - 3, 1024), (5, 5000), (9, 70_000)):
        picks = torch.empty(batch, dtype=torch.int64, device=dev)
        _lib.check(lib.md_random_batch(key, n, batch, picks.data_ptr(), sp))
        assert np.array_equal(picks.cpu().numpy(), oracle.random_batch_picks(key, n, batch))
    step = torch.full((1,), 41, dtype=torch.int64, device=dev)
    picks = torch.empty(1000, dtype=torch.int64, device=dev)
    for st in (41, 42):
        _lib.check(lib.md_random_batch_step(3, 4, 5, step.data_ptr(), n, 1000, picks.data_ptr(), sp))
        want = oracle.random_batch_picks(_mix64(3, 4, 5, st), n, 1000)
        assert np.array_equal(picks.cpu().numpy(), want)
    assert int(step.item()) == 43


def test_batch_stream_with_rejections(oracle):
    """BatchStream (device step counter) over 40 steps of 1024 draws from
    1,000,000 records -- ~21 % of the batches contain a Lemire rejection,
    exercising the block-parallel compaction inside the step kernel."""
    from paper_1711_00705_b200.dimd import BatchStream, _mix64
    from paper_1711_00705_b200.sgd import SAMPLE_ROLE

    dev = torch.device("cuda", 0)
    n, L = 1_000_000, 16
    st = dimd.synth_store(n, L, 0, 1, 3, 0, 1, 0, device=dev)
    bs = BatchStream(st, 1024, L, 3, SAMPLE_ROLE, 7, start_step=100)
    hit = 0
    for step in range(100, 140):
        recs, labels, picks = (t.clone() for t in bs.next())
        want = oracle.random_batch_picks(_mix64(3, SAMPLE_ROLE, 7, step), n, 1024)
        assert np.array_equal(picks.cpu().numpy(), want), step
        gids = recs[:, :8].contiguous().view(torch.int64).flatten().cpu().numpy()
        assert np.array_equal(gids, want)
        assert torch.equal(labels, st.label[picks].to(torch.int32))
        raw = oracle.gen(_mix64(3, SAMPLE_ROLE, 7, step)).bit_generator.random_raw(512)
        w32 = np.stack([raw & 0xFFFFFFFF, raw >> np.uint64(32)], 1).ravel().astype(np.uint64)
        hit += bool(np.any((w32 * np.uint64(n)) & np.uint64(0xFFFFFFFF) < (2**32 - n) % n))
    assert hit >= 3  # the rejection path really ran
    assert int(bs.step.item()) == 140
    bs.slots.check()


@pytest.mark.parametrize("prefetch", [False, True])
@pytest.mark.parametrize("corrupt_prediction", [False, True])
def test_successive_shuffles_plan_from_predicted_counts(oracle, exchange, corrupt_prediction,
                                                       prefetch):
    """From the second epoch on, a shuffle plans with the record counts the
    previous plan predicted (md_shuffle_plan next_counts) while the counts'
    host collective runs; a wrong prediction is caught and re-planned. With
    ``next_seed`` the next epoch's whole plan is computed during this epoch's
    exchange (and recomputed when the counts changed). Every epoch's slots are
    checked against the oracle's plan with the true counts."""
    S, n_local, L, seed = 4, 3_000, 64, 31

    def prog(ep):
        st = dimd.synth_store(n_local, L, ep.rank, S, seed, 0, S, ep.rank, device=ep.torch_device)
        ok = []
        # global record id held by (member, local index) before each epoch
        held = ep.all_gather(np.arange(n_local, dtype=np.int64) * S + ep.rank)
        for epoch in range(3):
            counts = ep.all_gather(st.n_records)
            if epoch and corrupt_prediction:
                st._next_counts = [c + 1 for c in counts]
                if st._prefetched is not None:
                    pk, pc, pp = st._prefetched
                    st._prefetched = (pk, [c + 1 for c in pc], pp)
            elif epoch:
                ok.append(st._next_counts == counts)
                ok.append((st._prefetched is not None) == prefetch)
            key = oracle.mix64(seed, oracle.SHUF_ROLE, epoch)
            nxt = oracle.mix64(seed, oracle.SHUF_ROLE, epoch + 1) if prefetch else None
            st = shuffle_all(ep, st, m_segments=3, seed=key, next_seed=nxt)
            bad, gids = dimd.synth_verify(st, seed)
            mem, rec = oracle.shuffle_plan_c(key, 0, S, ep.rank, ep.rank, 3, counts)
            want = np.array([held[m][r] for m, r in zip(mem, rec)], dtype=np.int64)
            got = gids.cpu().numpy().astype(np.int64)
            ok.append(bad == 0 and np.array_equal(got, want))
            held = ep.all_gather(got)
        return ok

    for r in run_ranks(S, "cuda", prog, emulate=True).results:
        assert all(r), r
