"""Data-parallel-table step on the GPU: 12 steps of the reference's own
distributed run (N=4, m=2, k=4) replayed through train_step -- fused worker
fold + multicolor allreduce + update in one launch -- give the reference's
weights bit for bit; momentum/weight decay against the float32 oracle."""

import numpy as np
import pytest
import torch

from paper_1711_00705_b200 import DeviceModel, TrainConfig, build_multicolor_trees, run_ranks
from paper_1711_00705_b200 import dimd, errors
from paper_1711_00705_b200.sgd import StepBuffers, check_replicas, lr_at, train_step

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


def test_run_training_replays_on_host(oracle):
    """run_training (sgd.py:470-556): 3 epochs x 4 steps on 2 ranks x 2 workers,
    reshuffle every epoch. The gradient is each batch's label sum (integers:
    exact under any fold order), so the final weights, every step's loss/acc
    and the metrics CSV are replayed on the host from the oracle's shuffle
    plan and random_batch picks."""
    from paper_1711_00705_b200 import EpochMetrics, metrics_csv, run_training
    from paper_1711_00705_b200.dimd import Record, default_segments
    from paper_1711_00705_b200.sgd import SAMPLE_ROLE, SHUFFLE_ROLE, lr_schedule

    recs = [Record(bytes([i]) * 16, i % 7) for i in range(64)]
    cfg = TrainConfig(n_nodes=2, workers_per_node=2, per_worker_batch=4, epochs=3, base_lr=0.1,
                      seed=5, group_size=1, shuffle_every=1)
    p = 33
    w0 = np.linspace(-1, 1, p).astype(np.float32)

    def grad_fn(model, batches, bufs):
        for (rec, lab, _), buf in zip(batches, bufs):
            s = lab.to(torch.float32).sum()
            buf[:p] = s
            buf[p] = s
            buf[p + 1] = (lab == 0).sum().to(torch.float32)

    res = run_training(cfg, recs, grad_fn=grad_fn, init_weights=w0, record_bytes=16)

    # host replay
    sched = lr_schedule(cfg)
    labels = np.array([r.label for r in recs])
    order = [np.arange(64), np.arange(64)]  # each rank's shard (group_size 1: the whole corpus)
    w = w0.copy()
    t = 0
    for epoch in range(3):
        key = oracle.mix64(5, SHUFFLE_ROLE, epoch)
        for r in range(2):
            _, rec = oracle.shuffle_plan_c(key, r, 1, 0, r, default_segments(64 * 16), [64])
            order[r] = order[r][rec]
        for _ in range(4):
            tot, zeros = 0, 0
            for r in range(2):
                for j in range(2):
                    pk = oracle.random_batch_picks(oracle.mix64(5, SAMPLE_ROLE, 2 * r + j, t), 64, 4)
                    lab = labels[order[r][pk]]
                    tot += int(lab.sum())
                    zeros += int((lab == 0).sum())
            lr = lr_at(sched, t / 4)
            st = res.steps[t]
            assert st.step == t and st.lr == lr
            assert st.loss == tot / 16 and st.correct == zeros
            w = oracle.sub_scaled_np(w, np.full(p, tot, np.float32), lr / 16)
            t += 1
    assert np.array_equal(res.weights, w)
    assert len(res.history) == 3 and isinstance(res.history[0], EpochMetrics)
    assert res.history[1].loss == sum(s.loss for s in res.steps[4:8]) / 4
    csv = metrics_csv(res).splitlines()
    assert csv[0] == "epoch,step,loss,acc,lr,elapsed_s" and len(csv) == 13
    assert csv[5].startswith(f"1,4,{res.steps[4].loss:.6g},{res.steps[4].acc:.6g},")
