"""Synchronous data-parallel SGD step ("data-parallel table") on B200.

API of /root/reference/pkg/src/minidist/sgd.py around its hot path:
``train_step`` (:382-426) samples each worker's sub-batch from the DIMD
shard (:290-314), obtains per-worker gradient sums with the loss and the
correct count in two tail slots (:335-353), sums them across ranks, applies
``W -= fl32(lr/B) * g`` (:416) and certifies the replicas (:356-379).

On B200 the fold of the worker buffers (gradient accumulation), the
multicolor allreduce and the weight update are ONE kernel launch
(collectives.run_fold with ``workers`` + ``update``); the replica check is a
device digest compared through the host channel.

The gradient producer is pluggable: ``train_step`` takes a ``grad_fn``
writing per-worker gradient buffers; for the reference's own model
(``model.ToyModel``, the 172-parameter MLP of :147-247) it defaults to the
device producer ``md_toy_grad``, so ``run_training(cfg, corpus)`` runs the
reference's whole training loop on the GPU with its bits. The momentum and
weight-decay terms are an extension (the reference has plain SGD); with
``momentum == weight_decay == 0`` the update is bit-identical to
``sub_scaled_f32(W, g[:p], lr / B)``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from paper_1711_00705_b200 import _lib
from paper_1711_00705_b200.collectives import (
    DEFAULT_SEGMENT_ELEMS,
    GradientBuffer,
    SgdUpdate,
    allreduce,
)
from paper_1711_00705_b200.dimd import BatchRequest, ShardStore, _mix64, random_batch_device
from paper_1711_00705_b200.errors import DisjointnessViolation, DivergenceDetected, InvalidConfig
from paper_1711_00705_b200.topology import build_multicolor_trees, build_ring

SAMPLE_ROLE = int.from_bytes(b"samp", "little")
SHUFFLE_ROLE = int.from_bytes(b"shuf", "little")


@dataclass(frozen=True)
class TrainConfig:
    """Job shape and schedule (sgd.py:58-104); ``momentum`` and
    ``weight_decay`` extend the reference's plain SGD."""

    n_nodes: int
    workers_per_node: int
    per_worker_batch: int
    epochs: int
    base_lr: float = 0.1
    warmup_epochs: int = 5
    drop_every: int = 30
    drop_factor: float = 10.0
    seed: int = 0
    group_size: int = 1
    shuffle_every: int = 1
    sim_compute_per_sample: float = 0.0
    hidden: int = 8
    momentum: float = 0.0
    weight_decay: float = 0.0

    def __post_init__(self):
        for name in ("n_nodes", "workers_per_node", "per_worker_batch", "epochs"):
            if getattr(self, name) < 1:
                raise InvalidConfig(f"{name} must be >= 1, got {getattr(self, name)}")
        checks = [
            (self.base_lr > 0, f"base_lr must be > 0, got {self.base_lr}"),
            (self.warmup_epochs >= 0, f"warmup_epochs must be >= 0, got {self.warmup_epochs}"),
            (self.drop_every >= 1, f"drop_every must be >= 1, got {self.drop_every}"),
            (self.drop_factor > 1, f"drop_factor must be > 1, got {self.drop_factor}"),
            (self.group_size >= 1, f"group_size must be >= 1, got {self.group_size}"),
            (self.shuffle_every >= 0, f"shuffle_every must be >= 0, got {self.shuffle_every}"),
            (self.sim_compute_per_sample >= 0, "sim_compute_per_sample must be >= 0"),
            (self.hidden >= 1, f"hidden must be >= 1, got {self.hidden}"),
            (0.0 <= self.momentum < 1.0, f"momentum must be in [0, 1), got {self.momentum}"),
            (self.weight_decay >= 0.0, f"weight_decay must be >= 0, got {self.weight_decay}"),
        ]
        for ok, msg in checks:
            if not ok:
                raise InvalidConfig(msg)

    @property
    def effective_batch(self) -> int:
        return self.n_nodes * self.workers_per_node * self.per_worker_batch


@dataclass(frozen=True)
class LrSchedule:
    base_lr: float
    k: int  # per-worker batch
    n: int  # total workers
    warmup_epochs: int
    drop_every: int
    drop_factor: float


def lr_schedule(cfg: TrainConfig) -> LrSchedule:
    return LrSchedule(cfg.base_lr, cfg.per_worker_batch, cfg.n_nodes * cfg.workers_per_node,
                      cfg.warmup_epochs, cfg.drop_every, cfg.drop_factor)


def lr_at(sched: LrSchedule, epoch: float) -> float:
    """Warm start (sgd.py:128-141): linear ramp base -> base*k*n/256 over
    warmup_epochs, then divide by drop_factor every drop_every epochs. The
    float64 expression order is the reference's, so values are identical."""
    if epoch < 0:
        raise InvalidConfig(f"epoch must be >= 0, got {epoch}")
    target = sched.base_lr * sched.k * sched.n / 256.0
    if epoch < sched.warmup_epochs:
        return sched.base_lr + (target - sched.base_lr) * (epoch / sched.warmup_epochs)
    return target * sched.drop_factor ** (-int((epoch - sched.warmup_epochs) // sched.drop_every))


@dataclass
class DeviceModel:
    """Replicated flat float32 weights (and momentum) resident on the GPU."""

    weights: torch.Tensor
    momentum: torch.Tensor | None = None

    @property
    def n_params(self) -> int:
        return int(self.weights.numel())

    @classmethod
    def from_numpy(cls, w: np.ndarray, device, momentum: bool = False) -> DeviceModel:
        t = torch.from_numpy(np.ascontiguousarray(w, dtype=np.float32)).to(device)
        return cls(t, torch.zeros_like(t) if momentum else None)


@dataclass(frozen=True)
class StepStats:
    step: int
    epoch: float
    lr: float
    loss: float  # mean loss over the effective batch
    correct: int
    samples: int
    elapsed_s: float = 0.0

    @property
    def acc(self) -> float:
        return self.correct / self.samples


def sample_node_batch(store: ShardStore, cfg: TrainConfig, rank: int, step: int,
                      record_bytes: int | None = None, slots=None):
    """Per-worker sub-batches carved at the source (sgd.py:290-314): worker j
    of rank r is global worker r*m+j, keyed _mix64(seed, "samp", worker, step).
    Returns [(records uint8 [k, L], labels int32 [k], picks int64 [k])].
    With ``slots`` (one dimd.BatchSlots per worker) nothing is allocated and
    nothing waits; the caller checks ``slots[j].err``."""
    out = []
    for j in range(cfg.workers_per_node):
        worker = rank * cfg.workers_per_node + j
        key = _mix64(cfg.seed, SAMPLE_ROLE, worker, step)
        out.append(random_batch_device(store, BatchRequest(cfg.per_worker_batch, key),
                                       record_bytes, None if slots is None else slots[j]))
    return out


def node_gradient(worker_bufs: list[torch.Tensor]) -> torch.Tensor:
    """Fold worker gradient buffers in worker order (sgd.py:335-353) -- the
    unfused form; train_step fuses this fold into the allreduce prologue."""
    from paper_1711_00705_b200 import _kernels

    acc = worker_bufs[0].clone()
    for b in worker_bufs[1:]:
        _kernels.add_f32(acc, b)
    return acc


def weights_digest(weights: torch.Tensor) -> int:
    """64-bit device digest of the weight bits (md_digest_f32)."""
    out = ctypes.c_uint64()
    _lib.check(
        _lib.load().md_digest_f32(
            weights.data_ptr(), weights.numel(), ctypes.byref(out),
            _lib.stream_ptr(torch.cuda.current_stream(weights.device)),
        )
    )
    return int(out.value)


def check_replicas(ep, weights: torch.Tensor, step: int) -> None:
    """Every rank raises DivergenceDetected unless all replicas' 64-bit device
    digests agree (sgd.py:356-379; blake2b over host bytes becomes a device
    reduction, only 8 bytes per rank cross to the host)."""
    if ep.n_ranks == 1:
        return
    digests = ep.all_gather(weights_digest(weights))
    if any(d != digests[0] for d in digests):
        raise DivergenceDetected(
            f"step {step}: replica weight digests differ: " + ", ".join(f"{d:016x}" for d in digests)
        )


def comm_plan(n_ranks: int, algo: str):
    """Widest color count the rank count supports (sgd.py:453-467)."""
    tree_set = ring = None
    if n_ranks > 1:
        if algo == "multicolor":
            for k in (4, 2, 1):
                try:
                    tree_set = build_multicolor_trees(n_ranks, k=k)
                    break
                except (InvalidConfig, DisjointnessViolation):
                    continue
        elif algo == "ring":
            ring = build_ring(n_ranks)
    return tree_set, ring


class StepBuffers:
    """Per-rank scratch of a training job: the peer-registered gradient
    buffer (p + 2 floats) and the per-worker gradient buffers."""

    def __init__(self, ep, n_params: int, workers: int):
        self.grad = GradientBuffer.alloc(n_params + 2, ep)
        dev = ep.torch_device
        self.workers = [torch.zeros(n_params + 2, dtype=torch.float32, device=dev)
                        for _ in range(workers)]
        self._slots: dict = {}
        # per-step readback: (loss sum, correct count) + every worker's batch error word
        self.host = torch.zeros(2 + workers, dtype=torch.float32).pin_memory()

    def slots(self, batch: int, record_bytes: int, device):
        """One preallocated minibatch slot set per worker (no per-step allocation)."""
        from paper_1711_00705_b200.dimd import BatchSlots

        key = (batch, record_bytes)
        if key not in self._slots:
            self._slots[key] = [BatchSlots(batch, record_bytes, device) for _ in self.workers]
        return self._slots[key]


def train_step(
    ep,
    model: DeviceModel,
    cfg: TrainConfig,
    store: ShardStore,
    algo: str = "multicolor",
    *,
    step: int = 0,
    epoch: float = 0.0,
    tree_set=None,
    ring=None,
    grad_fn=None,
    buffers: StepBuffers | None = None,
    record_bytes: int | None = None,
    verify_replicas: bool = True,
    segment_elems: int = DEFAULT_SEGMENT_ELEMS,
    sync: bool = True,
):
    """One synchronous step: sample, [fold + allreduce + update] fused, check.

    ``grad_fn(model, batches, worker_bufs)`` writes each worker's summed
    gradient and its (loss sum, correct count) tail into ``worker_bufs[j]``
    (p + 2 floats); None = the device ToyModel producer (model.toy_grad_fn). With ``sync=False`` nothing waits on the device and the
    returned stats are None (the bench's device-resident loop)."""
    if ep.n_ranks != cfg.n_nodes:
        raise InvalidConfig(f"config says {cfg.n_nodes} nodes, running {ep.n_ranks}")
    if grad_fn is None:
        from paper_1711_00705_b200.model import ToyModel, toy_grad_fn

        if not isinstance(model, ToyModel):
            raise InvalidConfig("train_step needs a grad_fn for a model other than ToyModel")
        grad_fn = toy_grad_fn
    lr = lr_at(lr_schedule(cfg), epoch)
    p = model.n_params
    if buffers is None:
        buffers = StepBuffers(ep, p, cfg.workers_per_node)
    slots = (buffers.slots(cfg.per_worker_batch, record_bytes, store.device)
             if record_bytes is not None else None)
    batches = sample_node_batch(store, cfg, ep.rank, step, record_bytes, slots)
    grad_fn(model, batches, buffers.workers)
    b = cfg.effective_batch
    upd = SgdUpdate(
        weights=model.weights,
        c=lr / b,
        momentum=model.momentum,
        mu=cfg.momentum,
        wd_b=cfg.weight_decay * b,
        update_len=p,
    )
    allreduce(
        ep, buffers.grad, algo, tree_set=tree_set, ring=ring, segment_elems=segment_elems,
        workers=buffers.workers, update=upd, check=False,
    )
    if not sync:
        return model, None
    # one wait per step: the metric slots and the batches' error words come
    # back together, then the collective's error word (host-mapped)
    host = buffers.host
    host[0:2].copy_(buffers.grad.data[p : p + 2], non_blocking=True)
    if slots is not None:
        for j, sl in enumerate(slots):
            host[2 + j : 3 + j].copy_(sl.err, non_blocking=True)  # int32 -> float32 value
    torch.cuda.current_stream(ep.torch_device).synchronize()
    ep.take_error()
    if slots is not None and bool((host[2:] != 0).any()):
        for sl in slots:
            sl.check()  # raises LengthMismatch
    if verify_replicas:
        check_replicas(ep, model.weights, step)
    stats = StepStats(step=step, epoch=epoch, lr=lr, loss=float(host[0]) / b,
                      correct=int(host[1]), samples=b)
    return model, stats


# -- the training loop around the step (sgd.py:430-570) ---------------------------------------


@dataclass(frozen=True)
class EpochMetrics:
    epoch: int
    loss: float
    acc: float
    time_s: float  # wall time (there is no simulated clock on real hardware)


@dataclass(frozen=True)
class TrainResult:
    history: list[EpochMetrics]
    steps: list[StepStats]
    weights: np.ndarray
    virtual_time: float | None
    wall_time: float

    @property
    def final_acc(self) -> float:
        return self.history[-1].acc


def run_training(
    cfg: TrainConfig,
    corpus,
    algo: str = "multicolor",
    *,
    grad_fn=None,
    init_weights: np.ndarray | None = None,
    backend: str = "cuda",
    emulate: bool | None = None,
    record_bytes: int | None = None,
) -> TrainResult:
    """Train for cfg.epochs over the corpus, one rank per node (sgd.py:470-542).

    Each epoch optionally reshuffles the DIMD store (``shuffle_all`` keyed
    ``_mix64(seed, "shuf", epoch)``), then runs max(1, len(corpus) //
    effective_batch) steps of ``train_step``; metrics are identical on every
    rank and rank 0's copy is returned. The store, the shuffle, the gradient
    producer, the fused fold + allreduce + update and the replica check run on
    the GPU. By default the model is the reference's ``ToyModel`` (n_in = the
    record size / 4, ``cfg.hidden`` units, 4 classes, ``ToyModel.create(seed=
    cfg.seed)``) with the device producer; ``grad_fn`` + ``init_weights``
    plug in another model.
    """
    from paper_1711_00705_b200.dimd import build_blob, parse_index, shard_from_bytes, shuffle_all
    from paper_1711_00705_b200.transport import run_ranks

    if not corpus:
        raise InvalidConfig("corpus must be non-empty")
    blob, index = build_blob(corpus)
    entries = parse_index(index)
    steps_per_epoch = max(1, len(corpus) // cfg.effective_batch)
    toy = grad_fn is None
    if toy:
        from paper_1711_00705_b200.model import ToyModel

        if init_weights is not None:
            raise InvalidConfig("init_weights needs a grad_fn (the ToyModel initialises itself)")
        n_in = len(corpus[0].bytes) // 4
        record_bytes = len(corpus[0].bytes) if record_bytes is None else record_bytes
        bad = [r.label for r in corpus if not -4 <= r.label < 4]
        if bad:  # the reference fails on p[rows, y] (sgd.py:235)
            raise IndexError(f"label {bad[0]} is out of range for the model's 4 classes")
        w0 = ToyModel.init_weights(n_in, cfg.hidden, 4, cfg.seed)
    elif init_weights is None:
        raise InvalidConfig("a custom grad_fn needs init_weights")
    else:
        w0 = np.ascontiguousarray(init_weights, dtype=np.float32)

    def program(ep):
        import time

        dev = ep.torch_device
        with torch.cuda.device(dev), torch.cuda.stream(ep.stream):
            store = shard_from_bytes(blob, entries, ep.rank, ep.n_ranks, cfg.group_size, device=dev)
            model = DeviceModel.from_numpy(w0, dev, momentum=cfg.momentum != 0)
            if toy:
                model = ToyModel(model.weights, n_in=n_in, hidden=cfg.hidden, n_classes=4,
                                 momentum=model.momentum)
            tree_set, ring = comm_plan(ep.n_ranks, algo)
            buffers = StepBuffers(ep, model.n_params, cfg.workers_per_node)
            t_start = time.perf_counter()
            history: list[EpochMetrics] = []
            rows: list[StepStats] = []
            gstep = 0
            for epoch in range(cfg.epochs):
                if cfg.shuffle_every > 0 and epoch % cfg.shuffle_every == 0:
                    nxt = epoch + cfg.shuffle_every  # the next reshuffle's key: plan it early
                    store = shuffle_all(ep, store, seed=_mix64(cfg.seed, SHUFFLE_ROLE, epoch),
                                        next_seed=(_mix64(cfg.seed, SHUFFLE_ROLE, nxt)
                                                   if nxt < cfg.epochs else None))
                t0 = time.perf_counter()
                loss_sum, correct = 0.0, 0
                for _ in range(steps_per_epoch):
                    model, st = train_step(
                        ep, model, cfg, store, algo, step=gstep, epoch=gstep / steps_per_epoch,
                        tree_set=tree_set, ring=ring, grad_fn=grad_fn, buffers=buffers,
                        record_bytes=record_bytes,
                    )
                    st = StepStats(st.step, st.epoch, st.lr, st.loss, st.correct, st.samples,
                                   elapsed_s=time.perf_counter() - t_start)
                    rows.append(st)
                    loss_sum += st.loss
                    correct += st.correct
                    gstep += 1
                history.append(EpochMetrics(
                    epoch=epoch, loss=loss_sum / steps_per_epoch,
                    acc=correct / (steps_per_epoch * cfg.effective_batch),
                    time_s=time.perf_counter() - t0,
                ))
            return model.weights.cpu().numpy(), history, rows

    rr = run_ranks(cfg.n_nodes, backend, program, emulate=emulate)
    weights, history, rows = rr.results[0]
    return TrainResult(history=history, steps=rows, weights=weights,
                       virtual_time=rr.virtual_time, wall_time=rr.wall_time)


def metrics_csv(result: TrainResult) -> str:
    """Per-step metrics stream: epoch,step,loss,acc,lr,elapsed_s (sgd.py:545-556)."""
    lines = ["epoch,step,loss,acc,lr,elapsed_s"]
    for st in result.steps:
        lines.append(f"{int(st.epoch)},{st.step},{st.loss:.6g},{st.acc:.6g},"
                     f"{st.lr:.6g},{st.elapsed_s:.6g}")
    return "\n".join(lines) + "\n"
