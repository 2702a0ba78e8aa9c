"""The reference's model on the device: ``ToyModel``
(/root/reference/pkg/src/minidist/sgd.py:148-248), the gradient producer of
its training loop.

The weights are the same flat float32 vector ``[W1 | b1 | W2 | b2]``, resident
on the GPU (``DeviceModel``); ``loss_and_grad_sum`` and the per-step producer
``toy_grad_fn`` run ``md_toy_grad`` (csrc/md_toy.cu): float64 math in numpy's
evaluation order, gradient rounded to float32 once -- the reference's bits.
Only ``create`` (the seeded initialisation, numpy's ``default_rng``) runs on
the host, once.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from paper_1711_00705_b200 import _lib
from paper_1711_00705_b200.errors import InvalidConfig


def _ptrs(tensors) -> ctypes.Array:
    arr = (ctypes.c_void_p * len(tensors))()
    for i, t in enumerate(tensors):
        arr[i] = t.data_ptr()
    return arr


@dataclass
class ToyModel:
    """One-hidden-layer tanh MLP with softmax cross-entropy loss (sgd.py:148-160),
    weights on the GPU. ``momentum`` is the optional SGD state of the
    momentum extension (``DeviceModel``'s field)."""

    weights: torch.Tensor
    n_in: int = 16
    hidden: int = 8
    n_classes: int = 4
    momentum: torch.Tensor | None = None
    _work: torch.Tensor | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        w = self.weights
        if isinstance(w, np.ndarray):  # the reference's form: move it to the current GPU
            if w.dtype != np.float32 or w.ndim != 1:
                raise InvalidConfig("weights must be a flat float32 vector")
            w = self.weights = torch.from_numpy(np.ascontiguousarray(w)).to(
                torch.device("cuda", torch.cuda.current_device()))
        if not isinstance(w, torch.Tensor) or w.dtype != torch.float32 or w.dim() != 1:
            raise InvalidConfig("weights must be a flat float32 vector")
        if w.numel() != self.n_params:
            raise InvalidConfig(
                f"expected {self.n_params} weights for "
                f"{self.n_in}->{self.hidden}->{self.n_classes}, got {w.numel()}"
            )
        if not w.is_cuda or not w.is_contiguous():
            raise InvalidConfig("weights must be a contiguous CUDA tensor")

    @property
    def n_params(self) -> int:
        return (self.n_in * self.hidden + self.hidden + self.hidden * self.n_classes
                + self.n_classes)

    @staticmethod
    def init_weights(n_in: int = 16, hidden: int = 8, n_classes: int = 4,
                     seed: int = 0) -> np.ndarray:
        """ToyModel.create's seeded initialisation (sgd.py:183-190)."""
        n = n_in * hidden + hidden + hidden * n_classes + n_classes
        rng = np.random.default_rng(seed)
        return (rng.standard_normal(n) * 0.1).astype(np.float32)

    @classmethod
    def create(cls, n_in: int = 16, hidden: int = 8, n_classes: int = 4, seed: int = 0,
               device=None, momentum: bool = False) -> ToyModel:
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        w = torch.from_numpy(cls.init_weights(n_in, hidden, n_classes, seed)).to(dev)
        return cls(w, n_in=n_in, hidden=hidden, n_classes=n_classes,
                   momentum=torch.zeros_like(w) if momentum else None)

    def grad_into(self, batches, outs, status: torch.Tensor | None = None,
                  feature_bytes: int = 4) -> None:
        """Per-worker gradient buffers (node_gradient's layout, sgd.py:335-353):
        ``batches[j] = (records uint8 [k, L], labels int32 [k], ...)`` from the
        DIMD batch slots, ``outs[j]`` float32 [p + 2] on the same device. Six
        small launches for all workers together (up to 8 per group),
        asynchronous on the current stream."""
        if len(batches) != len(outs) or not batches:
            raise InvalidConfig("need one output buffer per worker batch")
        recs = [b[0] for b in batches]
        labs = [b[1] for b in batches]
        k, stride = int(recs[0].shape[0]), int(recs[0].stride(0))
        for r, lab, o in zip(recs, labs, outs):
            if r.dtype != torch.uint8 or r.dim() != 2 or r.shape[0] != k or r.stride(0) != stride \
                    or r.stride(1) != 1 or r.device != self.weights.device:
                raise InvalidConfig("worker records must be uint8 [k, L] rows on the model's device")
            if lab.dtype != torch.int32 or lab.numel() != k or not lab.is_contiguous() \
                    or lab.device != self.weights.device:
                raise InvalidConfig("worker labels must be k contiguous int32 on the model's device")
            if o.dtype != torch.float32 or o.numel() != self.n_params + 2 or not o.is_contiguous() \
                    or o.device != self.weights.device:
                raise InvalidConfig(f"gradient buffers must be {self.n_params + 2} contiguous "
                                    "float32 on the model's device")
        if int(recs[0].shape[1]) < feature_bytes * self.n_in:
            raise InvalidConfig(f"expected {self.n_in} features, records hold "
                                f"{int(recs[0].shape[1]) // feature_bytes}")
        lib = _lib.load()
        nbytes = int(lib.md_toy_work_bytes(self.n_in, self.hidden, self.n_classes, k))
        if self._work is None or self._work.numel() * 8 < nbytes \
                or self._work.device != self.weights.device:
            self._work = torch.empty((nbytes + 7) // 8, dtype=torch.float64,
                                     device=self.weights.device)
        stream = torch.cuda.current_stream(self.weights.device)
        self._work.record_stream(stream)  # a workspace reallocated later waits for this use
        _lib.check(
            lib.md_toy_grad(
                self.weights.data_ptr(), self.n_in, self.hidden, self.n_classes,
                _ptrs(recs), feature_bytes, _ptrs(labs), stride, k, _ptrs(outs), len(outs),
                self._work.data_ptr(), self._work.numel() * 8,
                None if status is None else status.data_ptr(),
                _lib.stream_ptr(stream),
            )
        )

    def loss_and_grad_sum(self, x, y):
        """sgd.py:220-248 on one batch: (float32 gradient sum [p] on the device,
        loss sum, correct count). ``x``: uint8 [k, L] device records (float32
        features, the DIMD batch) or a float array [k, n_in] (float64 math like
        the reference); ``y``: class indices. Synchronizes (host scalars; the
        loss sum is the float32 value node_gradient's buffer holds)."""
        dev = self.weights.device
        recs, fb = _as_records(x, self.n_in, dev)
        labels = torch.as_tensor(np.asarray(y) if not isinstance(y, torch.Tensor) else y)
        labels = labels.to(device=dev, dtype=torch.int32).reshape(-1).contiguous()
        if labels.numel() != recs.shape[0]:
            raise InvalidConfig(f"{recs.shape[0]} rows but {labels.numel()} labels")
        out = torch.empty(self.n_params + 2, dtype=torch.float32, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.grad_into([(recs, labels)], [out], status, feature_bytes=fb)
        bad = int(status.item())
        if bad:
            raise IndexError(f"label of row {bad - 1} is out of range for {self.n_classes} classes")
        tail = out[self.n_params:].cpu().numpy()
        return out[: self.n_params], float(tail[0]), int(tail[1])


def toy_grad_fn(model: ToyModel, batches, worker_bufs) -> None:
    """``train_step``'s gradient producer for a ``ToyModel``: every worker's
    buffer from its DIMD sub-batch (the reference's node_gradient inputs)."""
    model.grad_into(batches, worker_bufs)


def _as_records(x, n_in: int, dev):
    """(uint8 [k, L] device rows, feature bytes) from device records or a
    host/device float array of features (float64 rows, the reference's x)."""
    if isinstance(x, torch.Tensor) and x.dtype == torch.uint8:
        if x.dim() != 2:
            raise InvalidConfig("records must be uint8 [k, L]")
        return x.to(dev), 4
    a = x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
    a = np.atleast_2d(np.ascontiguousarray(a, dtype="<f8"))
    if a.shape[1] != n_in:
        raise InvalidConfig(f"expected {n_in} features, got {a.shape[1]}")
    return torch.from_numpy(a.view(np.uint8).reshape(a.shape[0], -1)).to(dev), 8


def grad(model: ToyModel, batch):
    """Mean gradient of the loss over a list of (features, label) pairs
    (sgd.py:250-257): ``GradientBuffer`` of ``gsum / float32(len(batch))`` on
    the model's device."""
    from paper_1711_00705_b200.collectives import GradientBuffer

    if not batch:
        raise InvalidConfig("batch must be non-empty")
    x = np.stack([np.asarray(f, dtype=np.float64) for f, _ in batch])
    y = np.array([lbl for _, lbl in batch], dtype=np.int64)
    gsum, _, _ = model.loss_and_grad_sum(x, y)
    return GradientBuffer(torch.div(gsum, torch.tensor(float(len(batch)), dtype=torch.float32,
                                                       device=gsum.device)))


def make_synthetic_corpus(n_records: int, n_in: int = 16, n_classes: int = 4, seed: int = 0,
                          margin: float = 4.0, noise: float = 1.0):
    """The reference's corpus generator (sgd.py:263-283): linearly separable
    gaussian blobs, little-endian float32 features, label = class (host data
    generation, numpy's default_rng)."""
    from paper_1711_00705_b200.dimd import Record

    rng = np.random.default_rng(seed)
    means = rng.standard_normal((n_classes, n_in))
    means *= margin / np.linalg.norm(means, axis=1, keepdims=True)
    ys = rng.integers(0, n_classes, size=n_records)
    xs = means[ys] + noise * rng.standard_normal((n_records, n_in))
    return [Record(xs[i].astype("<f4").tobytes(), int(ys[i])) for i in range(n_records)]


def decode_record(rec) -> tuple[np.ndarray, int]:
    """sgd.py:286-287: a record's float32 features as float64, and its label."""
    return np.frombuffer(rec.bytes, dtype="<f4").astype(np.float64), rec.label
