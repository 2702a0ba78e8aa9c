"""The reference's gradient producer (ToyModel, /root/reference/pkg/src/
minidist/sgd.py:148-248) and the whole training loop on top of it.

CPU: the oracle's C restatement (oracle/mdoracle.c mo_toy_grad) and the host
helpers (make_synthetic_corpus, ToyModel.init_weights) against the golden
vectors the REAL reference produced (tests/golden/make_golden_toy.py ->
toy.npz; make_golden.py -> golden.npz's 12-step distributed SGD run).
GPU: md_toy_grad through the C ABI, train_step with the device producer and
run_training end to end -- all bit for bit against the reference.
"""

from pathlib import Path

import numpy as np
import pytest

from paper_1711_00705_b200 import TrainConfig, make_synthetic_corpus
from paper_1711_00705_b200.model import ToyModel
from paper_1711_00705_b200.sgd import SAMPLE_ROLE
from tests.conftest import need_gpus

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def toy():
    with np.load(ROOT / "tests" / "golden" / "toy.npz") as z:
        return {k: z[k] for k in z.files}


def _cases(toy):
    for i in range(int(toy["n_cases"][0])):
        k, n_in, h, c = (int(v) for v in toy[f"case{i}_shape"])
        yield i, k, n_in, h, c


def _golden_worker_inputs(golden, oracle):
    """(rank, step, worker, weights, x float32 [k, 16], y) of the golden
    12-step run (make_golden.py: N=4, m=2, k=4, seed 9, 512-record corpus,
    group_size 1 so every rank holds the whole corpus)."""
    n, m, k, seed, _ = (int(x) for x in golden["sgd_cfg"])
    corpus = make_synthetic_corpus(512, seed=9)
    xs = np.stack([np.frombuffer(r.bytes, "<f4") for r in corpus])
    ys = np.array([r.label for r in corpus])
    for step in range(golden["sgd_workers"].shape[1]):
        w = golden["sgd_w0"] if step == 0 else golden["sgd_weights"][step - 1]
        for r in range(n):
            for j in range(m):
                picks = oracle.random_batch_picks(oracle.mix64(seed, SAMPLE_ROLE, r * m + j, step),
                                                  512, k)
                yield r, step, j, w, xs[picks], ys[picks]


# -- CPU: oracle + host helpers vs the reference ------------------------------------------------


def test_oracle_toy_grad_matches_reference(toy, oracle):
    for i, k, n_in, h, c in _cases(toy):
        out = oracle.toy_grad_c(toy[f"case{i}_w"], n_in, h, c, toy[f"case{i}_x"], toy[f"case{i}_y"])
        p = toy[f"case{i}_w"].size
        assert np.array_equal(out[:p].view(np.uint32), toy[f"case{i}_g"].view(np.uint32)), i
        assert out[p] == np.float32(toy[f"case{i}_loss"][0]), i
        assert out[p + 1] == toy[f"case{i}_correct"][0], i


def test_oracle_reproduces_golden_worker_buffers(golden, oracle):
    """Every per-worker buffer of the reference's 12 distributed steps
    (node_gradient inputs, sgd.py:335-353) from the oracle producer."""
    for r, step, j, w, x, y in _golden_worker_inputs(golden, oracle):
        out = oracle.toy_grad_c(w, 16, 8, 4, x, y)
        assert np.array_equal(out.view(np.uint32), golden["sgd_workers"][r, step, j].view(np.uint32)), \
            (r, step, j)


def test_host_helpers_match_reference(toy):
    for t in range(int(toy["n_train"][0])):
        seed, nrec = int(toy[f"train{t}_cfg"][4]), int(toy[f"train{t}_cfg"][5])
        corpus = make_synthetic_corpus(nrec, seed=seed)
        xs = np.stack([np.frombuffer(r.bytes, "<f4") for r in corpus])
        assert np.array_equal(xs.view(np.uint32), toy[f"train{t}_corpus_x"].view(np.uint32))
        assert [r.label for r in corpus] == toy[f"train{t}_corpus_y"].tolist()
    for i, k, n_in, h, c in _cases(toy):
        seed = i + 1  # make_golden_toy.py SHAPES
        assert np.array_equal(ToyModel.init_weights(n_in, h, c, seed), toy[f"case{i}_w"]), i


def test_run_training_rejects_out_of_range_labels():
    from paper_1711_00705_b200 import run_training
    from paper_1711_00705_b200.dimd import Record

    recs = [Record(np.zeros(16, "<f4").tobytes(), 9)] * 8
    cfg = TrainConfig(n_nodes=1, workers_per_node=1, per_worker_batch=2, epochs=1)
    with pytest.raises(IndexError):
        run_training(cfg, recs)


# -- GPU: the device producer ------------------------------------------------------------------


@pytest.mark.gpu
def test_device_toy_grad_matches_reference(toy):
    import torch

    for i, k, n_in, h, c in _cases(toy):
        model = ToyModel(torch.from_numpy(toy[f"case{i}_w"]).cuda(), n_in=n_in, hidden=h,
                         n_classes=c)
        recs = torch.from_numpy(toy[f"case{i}_x"].view(np.uint8).reshape(k, -1).copy()).cuda()
        g, loss, correct = model.loss_and_grad_sum(recs, toy[f"case{i}_y"])
        assert np.array_equal(g.cpu().numpy().view(np.uint32), toy[f"case{i}_g"].view(np.uint32)), i
        assert np.float32(loss) == np.float32(toy[f"case{i}_loss"][0]), i
        assert correct == toy[f"case{i}_correct"][0], i


@pytest.mark.gpu
def test_device_grad_float64_features(toy):
    """grad(model, batch) (sgd.py:250-257): float64 features, mean gradient."""
    from paper_1711_00705_b200 import grad

    model = ToyModel(toy["grad_w"].copy())
    out = grad(model, list(zip(toy["grad_x"], toy["grad_y"].tolist())))
    assert np.array_equal(out.data.cpu().numpy().view(np.uint32), toy["grad_out"].view(np.uint32))


@pytest.mark.gpu
def test_device_toy_grad_rejects_bad_labels():
    import torch

    from paper_1711_00705_b200 import errors

    model = ToyModel.create(seed=3)
    recs = torch.zeros((4, 64), dtype=torch.uint8, device="cuda")
    with pytest.raises(IndexError):
        model.loss_and_grad_sum(recs, [0, 1, 4, 2])
    g, _, _ = model.loss_and_grad_sum(recs, [0, -1, -4, 2])  # numpy index wrap
    assert torch.isfinite(g).all()
    with pytest.raises(errors.InvalidConfig):
        model.loss_and_grad_sum(np.zeros((4, 15)), [0, 1, 2, 3])


@pytest.mark.gpu
def test_train_step_with_device_producer_matches_reference(golden, oracle):
    """The reference's 12 distributed steps (N=4 emulated, m=2, k=4) with NO
    replayed buffers: DIMD store from the corpus, device ToyModel gradients,
    fused fold + multicolor allreduce + update -> the reference's weights."""
    from paper_1711_00705_b200 import build_blob, build_multicolor_trees, parse_index, run_ranks
    from paper_1711_00705_b200.dimd import shard_from_bytes
    from paper_1711_00705_b200.sgd import StepBuffers, train_step

    n, m, k, seed, p = (int(x) for x in golden["sgd_cfg"])
    cfg = TrainConfig(n_nodes=n, workers_per_node=m, per_worker_batch=k, epochs=1,
                      shuffle_every=0, seed=seed)
    corpus = make_synthetic_corpus(512, seed=9)
    blob, idx = build_blob(corpus)
    entries = parse_index(idx)
    ts = build_multicolor_trees(n, k=4)

    def prog(ep):
        import torch

        dev = ep.torch_device
        store = shard_from_bytes(blob, entries, ep.rank, n, 1, device=dev)
        model = ToyModel(torch.from_numpy(golden["sgd_w0"].copy()).to(dev))
        bufs = StepBuffers(ep, p, m)
        out = []
        for step in range(golden["sgd_weights"].shape[0]):
            model, stats = train_step(ep, model, cfg, store, "multicolor", step=step,
                                      epoch=step / 16.0, tree_set=ts, buffers=bufs)
            out.append((model.weights.cpu().numpy(), [b.cpu().numpy() for b in bufs.workers]))
        return out

    for r, rank_out in enumerate(run_ranks(n, "cuda", prog, emulate=True).results):
        for step, (w, wb) in enumerate(rank_out):
            for j in range(m):
                assert np.array_equal(wb[j].view(np.uint32),
                                      golden["sgd_workers"][r, step, j].view(np.uint32)), (r, step, j)
            assert np.array_equal(w, golden["sgd_weights"][step]), (r, step)


def _run_training_case(toy, t, emulate):
    from paper_1711_00705_b200 import run_training

    nn, m, kb, epochs, seed, nrec, hidden, every, gs = (int(v) for v in toy[f"train{t}_cfg"])
    cfg = TrainConfig(n_nodes=nn, workers_per_node=m, per_worker_batch=kb, epochs=epochs,
                      seed=seed, hidden=hidden, shuffle_every=every, group_size=gs)
    corpus = make_synthetic_corpus(nrec, seed=seed)
    res = run_training(cfg, corpus, str(toy[f"train{t}_algo"]), emulate=emulate)
    assert np.array_equal(res.weights, toy[f"train{t}_weights"])
    got = np.array([[s.step, s.loss, s.correct, s.lr] for s in res.steps])
    assert np.array_equal(got, toy[f"train{t}_steps"])
    hist = np.array([[h.epoch, h.loss, h.acc] for h in res.history])
    assert np.array_equal(hist, toy[f"train{t}_history"])


TRAIN_CASES = [0, 1, 2, 3, 4]  # multicolor x2, ring (3 nodes, one shuffle group of 3),
#   reduce_bcast (4 nodes, shuffle groups of 2), bench_train's 16 -> 2048 -> 4 model


@pytest.mark.gpu
@pytest.mark.parametrize("t", TRAIN_CASES)
def test_run_training_matches_reference(toy, t):
    """run_training(cfg, corpus) (sgd.py:470-542) -- shuffles, device
    ToyModel producer, fused allreduce + update, replica checks -- against
    the reference's own run: final weights, every step's loss / correct / lr,
    every epoch's metrics. Ranks emulated on one GPU."""
    _run_training_case(toy, t, emulate=True)


@pytest.mark.gpu
@pytest.mark.multigpu
@need_gpus(4)
@pytest.mark.parametrize("t", TRAIN_CASES)
def test_run_training_matches_reference_one_gpu_per_rank(toy, t):
    """The same runs with one GPU per rank (NVLink peers)."""
    _run_training_case(toy, t, emulate=False)


@pytest.mark.gpu
def test_device_toy_grad_many_workers_one_call(oracle):
    """grad_into with more workers than one launch holds (MD_MAX_WORKERS = 8):
    every worker's buffer equals the oracle's."""
    import torch

    rng = np.random.default_rng(44)
    model = ToyModel.create(n_in=12, hidden=6, n_classes=5, seed=8)
    w = model.weights.cpu().numpy()
    xs = [rng.standard_normal((7, 12)).astype("<f4") for _ in range(11)]
    ys = [rng.integers(0, 5, size=7) for _ in range(11)]
    batches = [(torch.from_numpy(x.view(np.uint8).copy()).cuda(),
                torch.from_numpy(y.astype(np.int32)).cuda()) for x, y in zip(xs, ys)]
    outs = [torch.empty(model.n_params + 2, dtype=torch.float32, device="cuda") for _ in xs]
    model.grad_into(batches, outs)
    for x, y, o in zip(xs, ys, outs):
        want = oracle.toy_grad_c(w, 12, 6, 5, x, y)
        assert np.array_equal(o.cpu().numpy().view(np.uint32), want.view(np.uint32))
