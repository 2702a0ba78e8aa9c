"""Operator seam: the float32 kernels of minidist._kernels, on sm_100a.

Same names and contract as the reference module
(/root/reference/pkg/src/minidist/_kernels/__init__.py:33-43): in-place,
the caller owns the buffers, ``ValueError`` on a length mismatch, results
bit-identical to the reference's -ffp-contract=off C loops (_accel.pyx:12-29)
and numpy twins (fallback.py:6-23). Inputs are float32 CUDA tensors; the
work is enqueued on the current torch stream of the tensor's device.

``BACKEND`` is "cuda" and there is no other implementation to fall back to:
a missing libmdb200.so raises at import.
"""

from __future__ import annotations

import torch

from paper_1711_00705_b200 import _lib

_LIB = _lib.load()
BACKEND = "cuda"


def _flat(t, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (the B200 path has no CPU fallback)")
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32, got {t.dtype}")
    if t.dim() != 1 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous 1-D tensor")
    return t


def _stream(t: torch.Tensor):
    return _lib.stream_ptr(torch.cuda.current_stream(t.device))


def _mismatch(rc: int) -> None:
    if rc == -1:
        raise ValueError(_LIB.md_last_error().decode())
    _lib.check(rc)


def add_f32(dst, src) -> None:
    """dst += src, elementwise. Lengths must match."""
    d, s = _flat(dst, "dst"), _flat(src, "src")
    _mismatch(_LIB.md_add_f32(d.data_ptr(), d.numel(), s.data_ptr(), s.numel(), _stream(d)))


def sub_scaled_f32(dst, src, c) -> None:
    """dst -= float32(c) * src, elementwise, two roundings. Lengths must match."""
    d, s = _flat(dst, "dst"), _flat(src, "src")
    _mismatch(
        _LIB.md_sub_scaled_f32(d.data_ptr(), d.numel(), s.data_ptr(), s.numel(), float(c), _stream(d))
    )


def sgd_update(w, g, mom=None, c: float = 0.0, mu: float = 0.0, wd_b: float = 0.0) -> None:
    """Momentum / weight-decay SGD step (extension; see include/mdb200.h)."""
    w_, g_ = _flat(w, "w"), _flat(g, "g")
    if w_.numel() != g_.numel() or (mom is not None and _flat(mom, "mom").numel() != w_.numel()):
        raise ValueError("length mismatch between weights, gradient and momentum")
    m_ptr = mom.data_ptr() if (mom is not None and mu != 0.0) else None
    _lib.check(
        _LIB.md_sgd_update(
            w_.data_ptr(), g_.data_ptr(), m_ptr, w_.numel(), float(c), float(mu), float(wd_b),
            _stream(w_),
        )
    )


def available_impls():
    """Implementation name -> module (there is exactly one)."""
    import sys

    return {"cuda": sys.modules[__name__]}
