"""Allreduce (multi-color tree, ring, reduce+broadcast) and AllToAllV on B200.

API of /root/reference/pkg/src/minidist/collectives.py, executed by
libmdb200's persistent P2P kernels (csrc/md_ar_*.cu, routed by csrc/md_allreduce.cu):

* ``allreduce_multicolor`` (:225-268), ``allreduce_ring`` (:302-359) and
  ``reduce_then_broadcast`` (:365-409) differ only in their fold tree
  (topology.fold_tables / ring_fold_tables / star_fold_tables); the device
  reproduces each element's reference accumulation order, so results are
  bitwise equal to the reference (and to pkg/tests/oracles.py).
* The data-parallel-table extensions ride the same launch: ``workers``
  (fused gradient accumulation, sgd.py:335-353) and ``update`` (fused SGD
  epilogue, sgd.py:416, plus momentum / weight decay).
* ``alltoallv`` (:475-525): lengths travel host-side, bytes are pulled from
  the peers' registered send buffers by one copy kernel.

A ``GradientBuffer`` may hold a CUDA tensor (the fast path) or a numpy array
(drop-in for reference callers: staged through a registered device buffer,
host<->device copies included).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from paper_1711_00705_b200 import _lib
from paper_1711_00705_b200.errors import InvalidConfig, LengthMismatch, OffsetOverflow
from paper_1711_00705_b200.topology import (
    ColorTreeSet,
    FoldTables,
    RingOrder,
    build_multicolor_trees,
    build_ring,
    fold_tables,
    make_chunk_plan,
    ring_fold_tables,
    star_fold_tables,
)

# Pipeline granularity (elements per flag), the reference's own default
# (collectives.py:40). Bits do not depend on it; on B200 it is also the
# measured optimum of the channelized kernel (64 KiB per source per segment;
# sweep in profiles/README.md).
DEFAULT_SEGMENT_ELEMS = 16384
ALGORITHMS = ("multicolor", "ring", "reduce_bcast")
# route of calls that leave ``route="auto"`` (tests pin every kernel through it)
_DEFAULT_ROUTE = "auto"

_MAX_SLICE = 1 << 31
_SEG_BITS = 21      # the reference's tag layout bound, kept for make_segment_schedule
_MAX_COLORS = _lib.MD_MAX_COLORS


# -- buffers -------------------------------------------------------------------------


class GradientBuffer:
    """Flat float32 payload; owned by a collective for the call's duration.

    ``data`` is a 1-D float32 CUDA tensor or numpy array. ``peers`` is set on
    buffers allocated with ``alloc(n, ep)``: they are registered with every
    rank once, so collectives on them need no host round trip at all.
    """

    def __init__(self, data, peers=None):
        if isinstance(data, torch.Tensor):
            if data.dtype != torch.float32:
                raise InvalidConfig(f"buffer must be float32, got {data.dtype}")
            if data.dim() != 1:
                raise InvalidConfig(f"buffer must be 1-D, got {data.dim()}-D")
            if not data.is_contiguous():
                data = data.contiguous()
        else:
            arr = np.asarray(data)
            if arr.dtype != np.float32:
                raise InvalidConfig(f"buffer must be float32, got {arr.dtype}")
            if arr.ndim != 1:
                raise InvalidConfig(f"buffer must be 1-D, got {arr.ndim}-D")
            data = np.ascontiguousarray(arr)
        self.data = data
        self.peers = peers

    @property
    def len(self) -> int:
        return int(self.data.shape[0])

    @property
    def on_device(self) -> bool:
        return isinstance(self.data, torch.Tensor) and self.data.is_cuda

    @classmethod
    def zeros(cls, n: int, device=None) -> GradientBuffer:
        if device is None:
            return cls(np.zeros(n, dtype=np.float32))
        return cls(torch.zeros(n, dtype=torch.float32, device=device))

    @classmethod
    def of(cls, values, device=None) -> GradientBuffer:
        arr = np.asarray(values, dtype=np.float32)
        if device is None:
            return cls(arr)
        return cls(torch.from_numpy(arr.copy()).to(device))

    @classmethod
    def alloc(cls, n: int, ep=None) -> GradientBuffer:
        """Zeroed buffer. With an endpoint: device memory registered with
        every rank (collective call) -- the reference's prefaulted mmap
        (collectives.py:89-108) becomes a peer-mapped HBM allocation."""
        if ep is None:
            return cls(np.zeros(n, dtype=np.float32))
        t, view = ep.alloc(n, torch.float32)
        return cls(t, peers=(ep, view))

    def numpy(self) -> np.ndarray:
        if isinstance(self.data, torch.Tensor):
            return self.data.detach().cpu().numpy()
        return self.data

    def __repr__(self) -> str:
        where = "cuda" if self.on_device else "host"
        return f"GradientBuffer(len={self.len}, {where})"


@dataclass(frozen=True)
class SegmentSchedule:
    """Per-color segment ranges covering each color's chunk in order."""

    segment_elems: int
    per_color: tuple[tuple[tuple[int, int], ...], ...]


def make_segment_schedule(payload_len: int, k: int, segment_elems: int) -> SegmentSchedule:
    """Host-side segment plan of the reference pipeline (collectives.py:119-142).
    The device pipeline segments differently (4-element aligned) -- results
    are independent of segmentation (pkg/tests/test_collectives.py:131-147)."""
    if segment_elems < 1:
        raise InvalidConfig(f"segment_elems must be >= 1, got {segment_elems}")
    per_color = []
    for ch in make_chunk_plan(payload_len, k).chunks:
        bounds = list(range(ch.start, ch.start + ch.length, segment_elems))
        ranges = tuple((lo, min(lo + segment_elems, ch.start + ch.length)) for lo in bounds)
        if len(ranges) >= 1 << _SEG_BITS:
            raise InvalidConfig(
                f"{len(ranges)} segments for one color exceeds the tag space; raise segment_elems"
            )
        per_color.append(ranges)
    return SegmentSchedule(segment_elems, tuple(per_color))


def elementwise_add(dst: GradientBuffer, src: GradientBuffer) -> None:
    """dst[i] += src[i] (the reduction kernel, collectives.py:145-149)."""
    if dst.len != src.len:
        raise LengthMismatch(f"add of length {src.len} into length {dst.len}")
    from paper_1711_00705_b200 import _kernels

    _kernels.add_f32(dst.data, src.data)


# -- the fold engine -------------------------------------------------------------------


@dataclass
class SgdUpdate:
    """Fused SGD epilogue: W[:update_len] -= c * (g (+ wd_b*W)) with optional
    momentum (include/mdb200.h, md_sgd_update).

    ``sharded=True`` (md_allreduce_ex, MD_UPDATE_SHARDED): the owner of each
    buffer slice updates it and pushes the new weights to every rank -- the
    same weights bit for bit (replicas are identical, ref sgd.py:5-10) with
    1/N of the update's HBM traffic per rank. Momentum becomes sharded state
    (only this rank's slice is kept current) and the gradient buffer holds
    the sum only on this rank's slice and past ``update_len``. The weights
    are registered with every rank on first use (``ep.view_of``)."""

    weights: torch.Tensor
    c: float
    momentum: torch.Tensor | None = None
    mu: float = 0.0
    wd_b: float = 0.0
    update_len: int | None = None
    sharded: bool = False


def _check_operand(ep, t, what: str) -> None:
    """Device operands are passed by address: they must be float32, contiguous
    and on the rank's device (a temporary contiguous copy would be freed
    before the asynchronous kernel reads it)."""
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise InvalidConfig(f"{what} must be a CUDA tensor")
    if t.dtype != torch.float32:
        raise InvalidConfig(f"{what} must be float32, got {t.dtype}")
    if not t.is_contiguous():
        raise InvalidConfig(f"{what} must be contiguous")
    if t.device != ep.torch_device:
        raise InvalidConfig(f"{what} on {t.device}, rank on {ep.torch_device}")


def _device_tensor(ep, buf: GradientBuffer):
    """(device tensor, peer view, host array or None) for one call."""
    if buf.on_device:
        if buf.data.device != ep.torch_device:
            raise InvalidConfig(f"buffer on {buf.data.device}, rank on {ep.torch_device}")
        if buf.peers is not None and buf.peers[0] is ep:
            return buf.data, buf.peers[1], None
        # not pre-registered: one host exchange per call (also the length check)
        torch.cuda.current_stream(ep.torch_device).synchronize()
        return buf.data, ep.register(buf.data), None
    # host numpy buffer: stage through a registered device buffer
    n = buf.len
    if ep.n_ranks > 1:
        lens = ep.all_gather(n)
        if any(x != n for x in lens):
            raise LengthMismatch(f"ranks disagree on buffer length: {lens}")
    stage = ep._staging.get(n)
    if stage is None:
        stage = ep.alloc(n, torch.float32)
        ep._staging[n] = stage
    t, view = stage
    t.copy_(torch.from_numpy(buf.data), non_blocking=False)
    return t, view, buf.data


def run_fold(
    ep,
    buf: GradientBuffer,
    tables: FoldTables,
    *,
    segment_elems: int = DEFAULT_SEGMENT_ELEMS,
    workers: list | None = None,
    update: SgdUpdate | None = None,
    check: bool = True,
    ctas: int = 0,
    schedule: str = "tree",
    route: str = "auto",
    tile: int = 0,
) -> GradientBuffer:
    """One fused device collective: [worker fold] -> fold tree -> [SGD epilogue].

    ``schedule``: "tree" moves the data along each color's tree (the
    reference's schedule, collectives.py:225-296); "owner" cuts the buffer
    into n slices that one rank each folds with the same per-color fold order,
    then broadcasts -- the same bits, balanced traffic for any k.
    ``route``/``tile``: pin the kernel (md_plan_set_route; "auto" picks by
    size) -- every route gives the same bits."""
    if segment_elems < 1:
        raise InvalidConfig(f"segment_elems must be >= 1, got {segment_elems}")
    if schedule not in ("tree", "owner"):
        raise InvalidConfig(f"schedule must be 'tree' or 'owner', got {schedule!r}")
    if tables.n_ranks != ep.n_ranks:
        raise InvalidConfig(f"plan built for {tables.n_ranks} ranks, run has {ep.n_ranks}")
    dev, view, host = _device_tensor(ep, buf)
    n = dev.numel()
    wk = []
    for w in workers or []:
        _check_operand(ep, w, "worker buffer")
        if w.numel() != n:
            raise LengthMismatch(f"worker buffer of length {w.numel()} for payload {n}")
        wk.append(w.data_ptr())
    if len(wk) > _lib.MD_MAX_WORKERS:
        raise InvalidConfig(f"at most {_lib.MD_MAX_WORKERS} worker buffers")
    upd = None
    if update is not None:
        ulen = n if update.update_len is None else int(update.update_len)
        _check_operand(ep, update.weights, "weights")
        if update.weights.numel() < ulen:
            raise LengthMismatch("weights shorter than the update range")
        mom = update.momentum if (update.momentum is not None and update.mu != 0.0) else None
        if mom is not None:
            _check_operand(ep, mom, "momentum")
            if mom.numel() < ulen:
                raise LengthMismatch("momentum shorter than the update range")
        sharded = bool(update.sharded) and ep.n_ranks > 1
        # sharded: every rank's weights, as addressable from here
        wptrs = ep.view_of(update.weights).ptrs if sharded else [update.weights.data_ptr()]
        upd = (wptrs, mom.data_ptr() if mom is not None else None, ulen,
               float(update.c), float(update.mu), float(update.wd_b),
               _lib.MD_UPDATE_SHARDED if sharded else _lib.MD_UPDATE_REPLICATED)
    plan = ep.plan(tables, schedule, _DEFAULT_ROUTE if route == "auto" else route, tile)
    arg = (ep.comm, view.ptrs, wk, upd)
    lib = _lib.load()

    def launch(args_list):
        comms = [a[0] for a in args_list]
        ptrs = [p for a in args_list for p in a[1]]
        nw = len(args_list[0][2])
        wptrs = [p for a in args_list for p in a[2]]
        u0 = args_list[0][3]
        u = None
        if u0:
            u = _lib.MdUpdate()
            u.w = _lib.ptr_array([p for a in args_list for p in a[3][0]])
            u.mom = _lib.ptr_array([a[3][1] for a in args_list]) if u0[1] else None
            u.len, u.c, u.mu, u.wd_b, u.mode = u0[2], u0[3], u0[4], u0[5], u0[6]
        rc = lib.md_allreduce_ex(
            _lib.ptr_array(comms),
            len(args_list),
            plan,
            _lib.ptr_array(ptrs),
            n,
            _lib.ptr_array(wptrs) if nw else None,
            nw,
            C.byref(u) if u is not None else None,
            int(segment_elems),
            int(ctas),
            _lib.stream_ptr(ep.stream),
        )
        _lib.check(rc)

    # the kernel runs on the endpoint stream, after the caller's pending work
    cur = torch.cuda.current_stream(ep.torch_device)
    if cur.cuda_stream != ep.stream.cuda_stream:
        ep.stream.wait_stream(cur)
    if ep.mode == "emulated" and ep.n_ranks > 1:
        ep.rendezvous.run(ep.rank, arg, launch)
    else:
        launch([arg])
    if cur.cuda_stream != ep.stream.cuda_stream:
        cur.wait_stream(ep.stream)
    if host is not None:
        host[:] = dev.cpu().numpy()
        ep.take_error()
    elif check:
        ep.synchronize()
    return buf


# -- the three algorithms ------------------------------------------------------------------

_TABLES: dict = {}


def _tables_for(key_obj, make) -> FoldTables:
    """Fold tables per planning object (tree sets and rings are immutable);
    keeps the per-call host cost of a collective to a dict lookup."""
    hit = _TABLES.get(id(key_obj))
    if hit is None or hit[0] is not key_obj:
        hit = (key_obj, make(key_obj))
        _TABLES[id(key_obj)] = hit
    return hit[1]


def _debug_check_finite(buf: GradientBuffer) -> None:
    # collectives.py:152-154; on device only when asked (it costs a sync)
    if __debug__ and buf.len and not buf.on_device:
        assert bool(np.isfinite(buf.data).all()), "non-finite values in gradient buffer"


def allreduce_multicolor(
    ep, buf: GradientBuffer, ts: ColorTreeSet | None = None,
    segment_elems: int = DEFAULT_SEGMENT_ELEMS, **fused
) -> GradientBuffer:
    """Sum buffers across ranks along k color trees (collectives.py:225-268)."""
    _debug_check_finite(buf)
    if ep.n_ranks == 1 and not fused:  # one rank always agrees with itself
        return buf
    if ep.n_ranks == 1:
        from paper_1711_00705_b200.topology import single_rank_tables

        return run_fold(ep, buf, single_rank_tables(), segment_elems=segment_elems, **fused)
    if ts is None:
        ts = build_multicolor_trees(ep.n_ranks)
    if ts.n_ranks != ep.n_ranks:
        raise InvalidConfig(f"tree set built for {ts.n_ranks} ranks, run has {ep.n_ranks}")
    if ts.k > _MAX_COLORS:
        raise InvalidConfig(f"{ts.k} colors exceeds the device limit {_MAX_COLORS}")
    return run_fold(ep, buf, _tables_for(ts, fold_tables), segment_elems=segment_elems, **fused)


def allreduce_ring(
    ep, buf: GradientBuffer, ring: RingOrder | None = None,
    segment_elems: int = DEFAULT_SEGMENT_ELEMS, **fused
) -> GradientBuffer:
    """Reduce hop by hop to the ring root, broadcast back (collectives.py:302-359)."""
    _debug_check_finite(buf)
    if ep.n_ranks == 1 and not fused:  # one rank always agrees with itself
        return buf
    if ring is None:
        ring = build_ring(ep.n_ranks)
    if sorted(ring.order) != list(range(ep.n_ranks)):
        raise InvalidConfig(f"ring order {ring.order} is not a permutation of all ranks")
    return run_fold(ep, buf, _tables_for(ring, ring_fold_tables), segment_elems=segment_elems,
                    **fused)


def reduce_then_broadcast(ep, buf: GradientBuffer, root: int = 0, **fused) -> GradientBuffer:
    """Root folds every rank in ascending rank order, then broadcasts
    (collectives.py:365-409)."""
    _debug_check_finite(buf)
    if not 0 <= root < ep.n_ranks:
        raise InvalidConfig(f"root {root} out of range")
    if ep.n_ranks == 1 and not fused:  # one rank always agrees with itself
        return buf
    return run_fold(ep, buf, star_fold_tables(ep.n_ranks, root), **fused)


def allreduce(
    ep,
    buf: GradientBuffer,
    algo: str,
    *,
    tree_set: ColorTreeSet | None = None,
    ring: RingOrder | None = None,
    root: int = 0,
    segment_elems: int = DEFAULT_SEGMENT_ELEMS,
    **fused,
) -> GradientBuffer:
    """Dispatch by algorithm name (collectives.py:412-429). ``fused`` may carry
    ``workers=[...]``, ``update=SgdUpdate(...)``, ``check=False``."""
    if algo == "multicolor":
        return allreduce_multicolor(ep, buf, tree_set, segment_elems, **fused)
    if algo == "ring":
        return allreduce_ring(ep, buf, ring, segment_elems, **fused)
    if algo == "reduce_bcast":
        return reduce_then_broadcast(ep, buf, root, **fused)
    raise InvalidConfig(f"unknown allreduce algorithm {algo!r}, expected one of {ALGORITHMS}")


# -- alltoallv ----------------------------------------------------------------------------


@dataclass(frozen=True)
class VarPayload:
    """Per-destination byte slices of one contiguous send buffer. ``data`` is
    bytes (host) or a uint8 CUDA tensor."""

    data: object
    offsets: tuple[int, ...]
    lengths: tuple[int, ...]

    @classmethod
    def from_slices(cls, slices) -> VarPayload:
        slices = [bytes(s) for s in slices]
        offs = tuple(int(x) for x in np.concatenate([[0], np.cumsum([len(s) for s in slices])])[:-1])
        return cls(b"".join(slices), offs, tuple(len(s) for s in slices))

    def _nbytes(self) -> int:
        if isinstance(self.data, torch.Tensor):
            return self.data.numel()
        return len(self.data)

    def slice_for(self, rank: int):
        off, ln = self.offsets[rank], self.lengths[rank]
        if isinstance(self.data, torch.Tensor):
            return self.data[off : off + ln]
        return memoryview(self.data)[off : off + ln]

    def validate(self, n_ranks: int) -> None:
        if len(self.offsets) != n_ranks or len(self.lengths) != n_ranks:
            raise LengthMismatch(
                f"need {n_ranks} offset/length entries, got "
                f"{len(self.offsets)}/{len(self.lengths)}"
            )
        for ln in self.lengths:
            if ln < 0:
                raise LengthMismatch(f"negative slice length {ln}")
            if ln >= _MAX_SLICE:
                raise OffsetOverflow(f"slice of {ln} bytes exceeds the 32-bit limit")
        end = 0
        for off, ln in zip(self.offsets, self.lengths):
            if off < end or off + ln > self._nbytes():
                raise LengthMismatch("offsets/lengths are not disjoint in-order slices")
            end = off + ln


def alltoallv(ep, send: VarPayload) -> VarPayload:
    """Personalized exchange; received slices ordered by source rank.

    Lengths/offsets are gathered host-side together with the send buffers'
    IPC handles (one collective; the reference's length round,
    collectives.py:485-494); the bytes are pulled by one kernel from every
    source's registered send buffer (NVLink reads); a final barrier keeps
    every send buffer alive until its readers are done."""
    send.validate(ep.n_ranks)
    host = not isinstance(send.data, torch.Tensor)
    if host:
        raw = bytearray(send.data)
        src = (torch.frombuffer(raw, dtype=torch.uint8).to(ep.torch_device) if raw
               else torch.zeros(1, dtype=torch.uint8, device=ep.torch_device))
    else:
        src = send.data
    if src.numel() == 0:
        src = torch.zeros(1, dtype=torch.uint8, device=ep.torch_device)
    torch.cuda.current_stream(ep.torch_device).synchronize()
    # one host collective: every rank's slice table (the reference's length
    # round, collectives.py:485-494) rides with its send buffer's IPC handle
    (view,), tables = ep.register_varlen_many(
        [src], (tuple(send.offsets), tuple(send.lengths)))
    me = ep.rank
    lens = [tables[s][1][me] for s in range(ep.n_ranks)]
    offs_out = np.concatenate([[0], np.cumsum(lens)])[:-1].astype(np.int64).tolist()
    total = int(sum(lens))
    out = torch.empty(max(total, 1), dtype=torch.uint8, device=ep.torch_device)
    dst_ptrs, src_ptrs, nbytes = [], [], []
    for s in range(ep.n_ranks):
        if lens[s] == 0:
            continue
        dst_ptrs.append(out.data_ptr() + offs_out[s])
        src_ptrs.append(view.ptrs[s] + tables[s][0][me])
        nbytes.append(lens[s])
    if nbytes:
        lib = _lib.load()
        arr = (C.c_uint64 * len(nbytes))(*nbytes)
        _lib.check(
            lib.md_copy_segments(
                len(nbytes), _lib.ptr_array(dst_ptrs), _lib.ptr_array(src_ptrs), arr,
                _lib.stream_ptr(torch.cuda.current_stream(ep.torch_device)),
            )
        )
    torch.cuda.current_stream(ep.torch_device).synchronize()
    ep.barrier()  # nobody may reuse its send buffer while a peer still reads it
    data = out[:total]
    if host:
        data = bytes(data.cpu().numpy().tobytes())
    return VarPayload(data, tuple(offs_out), tuple(lens))
