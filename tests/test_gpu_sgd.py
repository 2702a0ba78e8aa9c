"""Data-parallel-table step on the GPU: 12 steps of the reference's own
distributed run (N=4, m=2, k=4) replayed through train_step -- fused worker
fold + multicolor allreduce + update in one launch -- give the reference's
weights bit for bit; momentum/weight decay against the float32 oracle."""

import numpy as np
import pytest
import torch

from paper_1711_00705_b200 import DeviceModel, TrainConfig, build_multicolor_trees, run_ranks
from paper_1711_00705_b200 import dimd, errors
from paper_1711_00705_b200.sgd import StepBuffers, check_replicas, train_step

pytestmark = pytest.mark.gpu


def replay_grad_fn(table, rank):
    """grad_fn that writes the reference's per-worker buffers of this step."""
    state = {"step": 0}

    def fn(model, batches, worker_bufs):
        for j, buf in enumerate(worker_bufs):
            buf.copy_(torch.from_numpy(table[rank, state["step"], j]))
        state["step"] += 1

    return fn


def test_replay_matches_reference_weights_bitwise(golden):
    n, m, k, seed, p = (int(x) for x in golden["sgd_cfg"])
    cfg = TrainConfig(n_nodes=n, workers_per_node=m, per_worker_batch=k, epochs=1,
                      shuffle_every=0, seed=seed)
    ts = build_multicolor_trees(n, k=4)
    table = golden["sgd_workers"]

    def prog(ep):
        dev = ep.torch_device
        store = dimd.synth_store(64, 64, ep.rank, n, 1, 0, 1, 0, device=dev)
        model = DeviceModel.from_numpy(golden["sgd_w0"], dev)
        bufs = StepBuffers(ep, p, m)
        fn = replay_grad_fn(table, ep.rank)
        out = []
        for step in range(table.shape[1]):
            model, stats = train_step(ep, model, cfg, store, "multicolor", step=step,
                                      epoch=step / 16.0, tree_set=ts, grad_fn=fn, buffers=bufs,
                                      record_bytes=64)
            out.append((model.weights.cpu().numpy(), stats))
        return out

    for rank_out in run_ranks(n, "cuda", prog, emulate=True).results:
        for step, (w, stats) in enumerate(rank_out):
            assert np.array_equal(w, golden["sgd_weights"][step]), step
            assert stats.lr == golden["sgd_lr"][step]
            assert stats.samples == n * m * k


@pytest.mark.parametrize("mu,wd", [(0.9, 0.0), (0.9, 5e-4), (0.0, 5e-4)])
def test_momentum_weight_decay_steps_match_oracle(golden, oracle, mu, wd):
    n, m, k, seed, p = (int(x) for x in golden["sgd_cfg"])
    cfg = TrainConfig(n_nodes=n, workers_per_node=m, per_worker_batch=k, epochs=1,
                      shuffle_every=0, seed=seed, momentum=mu, weight_decay=wd)
    table = golden["sgd_workers"]
    tables = oracle.tables_from_trees(n, oracle.trees(n, 4, 4))
    B = n * m * k
    w = golden["sgd_w0"].copy()
    v = np.zeros_like(w)
    want = []
    for step in range(4):
        folded = []
        for r in range(n):
            acc = table[r, step, 0].copy()
            for j in range(1, m):
                acc += table[r, step, j]
            folded.append(acc)
        g = oracle.fold_c(tables, folded)
        w, v2 = oracle.sgd_np(w, g[:p], v if mu else None, golden["sgd_lr"][step] / B, mu,
                              float(np.float32(wd * B)))
        v = v2 if mu else v
        want.append(w.copy())

    def prog(ep):
        dev = ep.torch_device
        store = dimd.synth_store(64, 64, ep.rank, n, 1, 0, 1, 0, device=dev)
        model = DeviceModel.from_numpy(golden["sgd_w0"], dev, momentum=mu != 0)
        bufs = StepBuffers(ep, p, m)
        fn = replay_grad_fn(table, ep.rank)
        got = []
        for step in range(4):
            model, _ = train_step(ep, model, cfg, store, "multicolor", step=step,
                                  epoch=step / 16.0, grad_fn=fn, buffers=bufs, record_bytes=64)
            got.append(model.weights.cpu().numpy())
        return got

    for got in run_ranks(n, "cuda", prog, emulate=True).results:
        for step in range(4):
            assert np.array_equal(got[step], want[step]), step


def test_replica_check_detects_divergence():
    def prog(ep):
        w = torch.zeros(1000, device=ep.torch_device)
        check_replicas(ep, w, 0)
        if ep.rank == 2:
            w[7] = 1.0
        with pytest.raises(errors.DivergenceDetected):
            check_replicas(ep, w, 1)

    run_ranks(4, "cuda", prog, emulate=True)


def test_train_step_validates_world_size():
    cfg = TrainConfig(n_nodes=4, workers_per_node=1, per_worker_batch=2, epochs=1)

    def prog(ep):
        with pytest.raises(errors.InvalidConfig):
            train_step(ep, DeviceModel(torch.zeros(4, device=ep.torch_device)), cfg, None,
                       grad_fn=lambda *a: None)

    run_ranks(2, "cuda", prog, emulate=True)
