"""DIMD: the distributed in-memory dataset, resident in HBM.

API of /root/reference/pkg/src/minidist/dimd.py. A ``ShardStore`` here keeps
its blob and index on the GPU: ``blob`` (uint8), ``off`` (int64 bit-cast of
the u64 offsets), ``length`` / ``label`` (int32 bit-casts of u32). The three
hot operations run on device, bit-exact with the reference's numpy Philox:

* ``random_batch`` (dimd.py:213-220): picks drawn by md_random_batch, records
  gathered by md_gather (``random_batch_device`` returns tensors; the
  reference-shaped ``random_batch`` copies Records to the host for parity);
* ``shuffle_all`` / ``shuffle_group`` (dimd.py:261-350): destination draws of
  every member recomputed locally, receive order + final permutation
  resolved before any byte moves (md_shuffle_plan), then each record crosses
  NVLink once, straight into its final slot: pushed by its source member
  (md_shuffle_sendlist + md_shuffle_push, the default) or pulled by its
  receiver (md_shuffle_pull, ``EXCHANGE = "pull"``);
* ``shard_from_bytes`` / ``load_partition`` (dimd.py:166-207): striping rule
  ``i mod group_size == rank_in_group`` applied on the host index, records
  staged into HBM once.

The blob + index codec (``build_blob``/``parse_index``) is the reference's
on-disk format (magic "DIMD", version 1, ``<u8 offset, <u4 length, <u4 label``).
"""

from __future__ import annotations

import ctypes as C
import struct
import threading
from dataclasses import dataclass

import numpy as np
import torch

from paper_1711_00705_b200 import _lib
from paper_1711_00705_b200.errors import (
    EmptyShard,
    FormatError,
    GroupMismatch,
    InvalidConfig,
    IoError,
    LengthMismatch,
    RecordTooLarge,
    SegmentOverflow,
)

INDEX_MAGIC = b"DIMD"
INDEX_VERSION = 1

_HEADER = struct.Struct("<4sIQ")  # magic, version, record count
_ENTRY_DTYPE = np.dtype([("offset", "<u8"), ("length", "<u4"), ("label", "<u4")])

_MAX_RECORD = 1 << 31
_MAX_LABEL = 1 << 32
_MASK64 = (1 << 64) - 1
_SEGMENT_TARGET = 1 << 30  # dimd.py:44

# role constants, little-endian ASCII (dimd.py:237-238, sgd.py:47-48)
PERM_ROLE = int.from_bytes(b"perm", "little")
DEST_ROLE = int.from_bytes(b"dest", "little")


@dataclass(frozen=True)
class IndexEntry:
    offset: int
    length: int
    label: int


@dataclass(frozen=True)
class Record:
    bytes: bytes
    label: int


@dataclass(frozen=True)
class BatchRequest:
    """batch_size records from the Philox stream keyed by rng_seed."""

    batch_size: int
    rng_seed: int

    def __post_init__(self):
        if self.batch_size < 1:
            raise InvalidConfig(f"batch_size must be >= 1, got {self.batch_size}")


class ShardStore:
    """One rank's resident slice of the dataset, in device memory."""

    def __init__(self, blob, off, length, label, group_id, group_size, rank_in_group):
        self.blob = blob            # uint8 CUDA tensor (>= 1 byte)
        self.off = off              # int64 CUDA tensor [n]
        self.length = length        # int32 CUDA tensor [n]
        self.label = label          # int32 CUDA tensor [n]
        self.group_id = group_id
        self.group_size = group_size
        self.rank_in_group = rank_in_group
        self._nbytes = None

    @property
    def device(self) -> torch.device:
        return self.blob.device

    @property
    def n_records(self) -> int:
        return int(self.off.numel())

    @property
    def nbytes(self) -> int:
        """Resident payload bytes (sum of record lengths)."""
        if self._nbytes is None:
            self._nbytes = int((self.length.to(torch.int64) & 0xFFFFFFFF).sum().item())
        return self._nbytes

    @property
    def index(self) -> list[IndexEntry]:
        off = self.off.cpu().numpy().view(np.uint64)
        ln = self.length.cpu().numpy().view(np.uint32)
        lb = self.label.cpu().numpy().view(np.uint32)
        return [IndexEntry(int(o), int(n), int(b)) for o, n, b in zip(off, ln, lb)]

    def record(self, i: int) -> Record:
        e = self.index[i]
        return Record(bytes(self.blob[e.offset : e.offset + e.length].cpu().numpy()), e.label)

    def records(self) -> list[Record]:
        idx = self.index
        host = self.blob.cpu().numpy()
        return [Record(bytes(host[e.offset : e.offset + e.length]), e.label) for e in idx]

    def labels(self) -> np.ndarray:
        return self.label.cpu().numpy().view(np.uint32)


def empty_index(device) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    z = torch.zeros(0, device=device)
    return z.to(torch.int64), z.to(torch.int32), z.to(torch.int32)


# -- blob + index codec (host) -------------------------------------------------------------


def build_blob(records) -> tuple[bytes, bytes]:
    """Concatenate records into (blob_bytes, index_bytes) (dimd.py:109-126)."""
    table = np.zeros(len(records), dtype=_ENTRY_DTYPE)
    pos = 0
    for i, rec in enumerate(records):
        size = len(rec.bytes)
        if size == 0:
            raise InvalidConfig(f"record {i} is empty")
        if size >= _MAX_RECORD:
            raise RecordTooLarge(f"record {i} is {size} bytes, limit is {_MAX_RECORD - 1}")
        if not 0 <= rec.label < _MAX_LABEL:
            raise InvalidConfig(f"label {rec.label} does not fit an unsigned 32-bit field")
        table[i] = (pos, size, rec.label)
        pos += size
    header = _HEADER.pack(INDEX_MAGIC, INDEX_VERSION, len(records))
    return b"".join(r.bytes for r in records), header + table.tobytes()


def _parse_table(data: bytes) -> np.ndarray:
    if len(data) < _HEADER.size:
        raise FormatError(f"index truncated: {len(data)} bytes, header needs {_HEADER.size}")
    magic, version, count = _HEADER.unpack_from(data)
    if magic != INDEX_MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {INDEX_MAGIC!r}")
    if version != INDEX_VERSION:
        raise FormatError(f"unsupported index version {version}")
    need = _HEADER.size + count * _ENTRY_DTYPE.itemsize
    if len(data) != need:
        raise FormatError(f"index holds {len(data)} bytes, {count} records need {need}")
    table = np.frombuffer(data, dtype=_ENTRY_DTYPE, count=count, offset=_HEADER.size)
    if count:
        if np.any(table["length"] == 0):
            i = int(np.flatnonzero(table["length"] == 0)[0])
            raise FormatError(f"record {i} has zero length")
        ends = table["offset"].astype(np.uint64) + table["length"].astype(np.uint64)
        overlap = table["offset"][1:] < ends[:-1]
        if np.any(overlap):
            i = int(np.flatnonzero(overlap)[0]) + 1
            raise FormatError(f"record {i} at offset {int(table['offset'][i])} overlaps the previous record")
    return table


def parse_index(data: bytes) -> list[IndexEntry]:
    """Decode an index file; FormatError on anything malformed (dimd.py:129-152)."""
    table = _parse_table(data)
    return [IndexEntry(int(o), int(n), int(b)) for o, n, b in table]


def _read_file(path) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError as e:
        raise IoError(f"cannot read {path}: {e}") from e


def _entries_array(entries) -> np.ndarray:
    if isinstance(entries, np.ndarray):
        return entries
    arr = np.zeros(len(entries), dtype=_ENTRY_DTYPE)
    for i, e in enumerate(entries):
        arr[i] = (e.offset, e.length, e.label)
    return arr


def store_from_host(blob, table: np.ndarray, group_id: int, group_size: int, rank_in_group: int,
                    device=None) -> ShardStore:
    """Stage a compact host shard (blob + entry table) into HBM."""
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    host = np.frombuffer(bytes(blob), dtype=np.uint8) if not isinstance(blob, np.ndarray) else blob
    dblob = torch.empty(max(1, host.size), dtype=torch.uint8, device=device)
    if host.size:
        dblob[: host.size].copy_(torch.from_numpy(host.copy()))
    off = torch.from_numpy(table["offset"].astype(np.uint64).view(np.int64).copy()).to(device)
    ln = torch.from_numpy(table["length"].astype(np.uint32).view(np.int32).copy()).to(device)
    lb = torch.from_numpy(table["label"].astype(np.uint32).view(np.int32).copy()).to(device)
    return ShardStore(dblob, off, ln, lb, group_id, group_size, rank_in_group)


def shard_from_bytes(
    blob, entries, rank: int, n_ranks: int, group_size: int, device=None
) -> ShardStore:
    """This rank's records by the striping rule, resident on the GPU
    (dimd.py:166-200): record i belongs to member ``i mod group_size``."""
    if n_ranks < 1:
        raise InvalidConfig(f"need at least 1 rank, got {n_ranks}")
    if not 0 <= rank < n_ranks:
        raise InvalidConfig(f"rank {rank} out of range for {n_ranks} ranks")
    if group_size < 1:
        raise InvalidConfig(f"group_size must be >= 1, got {group_size}")
    if n_ranks % group_size:
        raise GroupMismatch(f"group size {group_size} does not divide {n_ranks} ranks")
    table = _entries_array(entries)
    size = len(blob)
    if table.size:
        ends = table["offset"].astype(np.uint64) + table["length"].astype(np.uint64)
        over = ends > np.uint64(size)
        if np.any(over):
            i = int(np.flatnonzero(over)[0])
            raise FormatError(
                f"record {i} spans [{int(table['offset'][i])}, {int(ends[i])}) "
                f"outside the {size}-byte blob"
            )
    member = rank % group_size
    mine = table[member::group_size]
    direct = isinstance(blob, (bytes, bytearray, memoryview, np.ndarray))
    view = memoryview(blob) if direct else None
    parts = []
    for e in mine:
        lo, hi = int(e["offset"]), int(e["offset"]) + int(e["length"])
        parts.append(bytes(view[lo:hi]) if direct else bytes(blob[lo:hi]))
    compact = np.zeros(len(mine), dtype=_ENTRY_DTYPE)
    if len(mine):
        compact["length"] = mine["length"]
        compact["label"] = mine["label"]
        compact["offset"][1:] = np.cumsum(mine["length"].astype(np.uint64))[:-1]
    return store_from_host(b"".join(parts), compact, rank // group_size, group_size, member, device)


def load_partition(blob_path, index_path, rank: int, n_ranks: int, group_size: int,
                   device=None) -> ShardStore:
    """This rank's shard of an on-disk blob + index (dimd.py:203-207)."""
    table = _parse_table(_read_file(index_path))
    blob = _read_file(blob_path)
    return shard_from_bytes(blob, table, rank, n_ranks, group_size, device)


# -- random batches -----------------------------------------------------------------------


def _stream(dev) -> int | None:
    return _lib.stream_ptr(torch.cuda.current_stream(dev))


def random_batch_picks(store: ShardStore, req: BatchRequest,
                       out: torch.Tensor | None = None) -> torch.Tensor:
    """Philox(req.rng_seed).integers(0, n_records, batch_size), on device."""
    n = store.n_records
    if n == 0:
        raise EmptyShard("cannot sample from an empty shard")
    picks = out if out is not None else torch.empty(req.batch_size, dtype=torch.int64,
                                                    device=store.device)
    _lib.check(
        _lib.load().md_random_batch(
            req.rng_seed & _MASK64, n, req.batch_size, picks.data_ptr(), _stream(store.device)
        )
    )
    return picks


class BatchSlots:
    """Preallocated outputs of ``random_batch_device`` for a training loop
    (no allocation, no host sync per step; ``err`` is checked by the caller)."""

    def __init__(self, batch: int, record_bytes: int, device):
        self.records = torch.empty((batch, record_bytes), dtype=torch.uint8, device=device)
        self.labels = torch.empty(batch, dtype=torch.int32, device=device)
        self.picks = torch.empty(batch, dtype=torch.int64, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)

    def check(self) -> None:
        if int(self.err.item()):
            raise LengthMismatch("a sampled record does not have the batch's record size")


def random_batch_device(store: ShardStore, req: BatchRequest, record_bytes: int | None = None,
                        slots: BatchSlots | None = None):
    """Hot-path minibatch: (records uint8 [B, record_bytes], labels int32 [B], picks).

    Every picked record must be ``record_bytes`` long (fixed-size corpora such
    as 224x224x3 images); use ``random_batch`` for ragged records. Without
    ``slots`` the outputs are fresh and the length check synchronizes; with
    ``slots`` nothing waits on the device (call ``slots.check()`` later)."""
    B = req.batch_size
    if record_bytes is None:
        record_bytes = int((store.length[:1].to(torch.int64) & 0xFFFFFFFF).item())
    own = slots is None
    if own:
        slots = BatchSlots(B, record_bytes, store.device)
    random_batch_picks(store, req, slots.picks)
    _gather_fixed(store, slots, B, record_bytes)
    if own:
        slots.check()
    return slots.records, slots.labels, slots.picks


def _gather_fixed(store: ShardStore, slots: BatchSlots, batch: int, record_bytes: int) -> None:
    _lib.check(
        _lib.load().md_gather(
            store.blob.data_ptr(), store.off.data_ptr(), store.length.data_ptr(),
            store.label.data_ptr(), slots.picks.data_ptr(), batch, slots.records.data_ptr(),
            record_bytes, None, slots.labels.data_ptr(), slots.err.data_ptr(),
            _stream(store.device),
        )
    )


class BatchStream:
    """One worker's per-step minibatches as a graph-replayable pair of kernels.

    ``next()`` draws the batch of the current step with the key
    ``_mix64(seed, role, worker, step)`` -- the key sgd.sample_node_batch uses
    (reference sgd.py:303-307) -- gathers it into ``slots`` and advances the
    step counter, which lives on the device: a CUDA graph that captured one
    ``next()`` draws a fresh, bit-identical-to-the-reference batch on every
    replay. Fixed-size records only (as ``random_batch_device``), batch <= 1024."""

    def __init__(self, store: ShardStore, batch: int, record_bytes: int, seed: int, role: int,
                 worker: int, start_step: int = 0):
        if store.n_records == 0:
            raise EmptyShard("cannot sample from an empty shard")
        if not 1 <= batch <= 1024:
            raise InvalidConfig(f"BatchStream batch must be in [1, 1024], got {batch}")
        self.store, self.batch, self.record_bytes = store, batch, record_bytes
        self.seed, self.role, self.worker = seed & _MASK64, role & _MASK64, worker & _MASK64
        self.step = torch.full((1,), start_step, dtype=torch.int64, device=store.device)
        self.slots = BatchSlots(batch, record_bytes, store.device)

    def next(self, slots: BatchSlots | None = None):
        """Draw and gather the next step's batch into ``slots`` (default
        ``self.slots``) on the current stream. A training loop that prefetches
        (batch i+1 gathered on a side stream while step i computes) passes
        alternating slot sets; the step counter still advances in stream order."""
        # Two launches (picks, gather). A fused one-kernel variant, where every
        # (record, chunk) CTA derives its own pick, measured slower on B200
        # (8.9 vs 6.0 us per 32-record batch): the per-CTA Philox + vote chain
        # is longer than the separate picks launch it saves.
        st = self.store
        slots = self.slots if slots is None else slots
        _lib.check(
            _lib.load().md_random_batch_step(
                self.seed, self.role, self.worker, self.step.data_ptr(), st.n_records, self.batch,
                slots.picks.data_ptr(), _stream(st.device),
            )
        )
        _gather_fixed(st, slots, self.batch, self.record_bytes)
        return slots.records, slots.labels, slots.picks


def random_batch(store: ShardStore, req: BatchRequest) -> list[Record]:
    """Sample batch_size records uniformly with replacement (dimd.py:213-220)."""
    picks = random_batch_picks(store, req)
    dev = store.device
    lens = (store.length.index_select(0, picks).to(torch.int64) & 0xFFFFFFFF)
    out_off = torch.zeros(req.batch_size, dtype=torch.int64, device=dev)
    if req.batch_size > 1:
        out_off[1:] = torch.cumsum(lens, 0)[:-1]
    total = int(lens.sum().item())
    out = torch.empty(max(1, total), dtype=torch.uint8, device=dev)
    labels = torch.empty(req.batch_size, dtype=torch.int32, device=dev)
    _lib.check(
        _lib.load().md_gather(
            store.blob.data_ptr(), store.off.data_ptr(), store.length.data_ptr(),
            store.label.data_ptr(), picks.data_ptr(), req.batch_size, out.data_ptr(), 0,
            out_off.data_ptr(), labels.data_ptr(), None, _stream(dev),
        )
    )
    host = out.cpu().numpy()
    offs = out_off.cpu().numpy()
    ls = lens.cpu().numpy()
    lb = labels.cpu().numpy().view(np.uint32)
    return [Record(bytes(host[o : o + n]), int(b)) for o, n, b in zip(offs, ls, lb)]


# -- shuffle --------------------------------------------------------------------------------


def _mix64(*parts: int) -> int:
    """splitmix64-style fold of role integers into one key (dimd.py:226-234);
    the same function the device uses (md_mix64)."""
    arr = (C.c_uint64 * max(1, len(parts)))(*[int(p) & _MASK64 for p in parts])
    return int(_lib.load().md_mix64(arr, len(parts))) if _lib.LIB_PATH.exists() else _mix64_py(*parts)


def _mix64_py(*parts: int) -> int:
    acc = 0
    for p in parts:
        acc = (acc + (int(p) & _MASK64) + 0x9E3779B97F4A7C15) & _MASK64
        acc = ((acc ^ (acc >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
        acc = ((acc ^ (acc >> 27)) * 0x94D049BB133111EB) & _MASK64
        acc ^= acc >> 31
    return acc


def default_segments(shard_bytes: int) -> int:
    """Segment count keeping per-exchange slices far below 2^31 bytes."""
    return max(1, -(-shard_bytes // _SEGMENT_TARGET))


def _check_group(ep, store: ShardStore) -> None:
    if ep.n_ranks % store.group_size:
        raise GroupMismatch(f"group size {store.group_size} does not divide {ep.n_ranks} ranks")
    if store.group_id != ep.rank // store.group_size or store.rank_in_group != ep.rank % store.group_size:
        raise GroupMismatch(
            f"rank {ep.rank} holds a shard labeled group {store.group_id} "
            f"member {store.rank_in_group}, which is not its position"
        )


def shuffle_all(ep, store: ShardStore, m_segments: int | None = None, seed: int = 0, *,
                next_seed: int | None = None) -> ShardStore:
    """Exchange records within each group, all ranks participating (dimd.py:261-269).

    ``next_seed`` (extension, optional): the next epoch's shuffle key. The
    next epoch's plan is then computed on a side stream while this epoch's
    records cross the links, and the returned store carries it; the next
    ``shuffle_all`` with that key (and the same record counts) skips its plan.
    The bits never depend on it."""
    _check_group(ep, store)
    return _shuffle(ep, store, m_segments, seed, next_seed)


def shuffle_group(ep, store: ShardStore, m_segments: int | None = None, seed: int = 0, *,
                  next_seed: int | None = None) -> ShardStore:
    """Exchange inside this rank's group (dimd.py:272-278). Keys do not depend
    on the communicator layout, so the result equals ``shuffle_all``'s."""
    _check_group(ep, store)
    return _shuffle(ep, store, m_segments, seed, next_seed)


def group_record_counts(channel, members, n_records: int, m_segments: int) -> list[int]:
    """Host step of the shuffle (collective over every world rank): gather the
    members' record counts -- all a receiver needs to recompute every source's
    destination draws -- and insist the group agrees on m_segments (dest keys
    depend on the segment index, dimd.py:308; the reference would deadlock
    on a disagreement, here it is an InvalidConfig on every member)."""
    return _group_counts(channel.all_gather((int(n_records), int(m_segments))), members, m_segments)


def _group_counts(rows, members, m_segments: int) -> list[int]:
    seen = [rows[m][1] for m in members]
    if any(x != m_segments for x in seen):
        raise InvalidConfig(f"group members disagree on m_segments: {seen}")
    return [rows[m][0] for m in members]


LAST_SHUFFLE_PHASES: dict[str, float] = {}
# how the shuffle's bytes cross the links: "push" (sources store records into
# the receivers' new blobs, md_shuffle_push) or "pull" (receivers load them,
# md_shuffle_pull). Same placement, same bytes.
EXCHANGE = "push"


class _ShardArena:
    """Reusable output allocations for successive shuffles of one endpoint.

    Peers map a shard's arrays through CUDA IPC (md_mem_import): mapping a
    24 GB blob costs tens of ms, and even a fresh 1 MB index allocation costs
    ~1-3 ms across the group (tools/register_probe.py). So each slot keeps a
    blob allocation AND one index allocation (off | len | label) that are
    reused epoch after epoch; the imports then hit the per-process cache. A
    slot is reused only when the ShardStore that owned it has been garbage
    collected, so no live store is ever overwritten."""

    HEADROOM = 1.03

    def __init__(self):
        self.slots: list[list] = []  # [blob tensor, weakref to owner or None, index tensor]

    def take(self, n_records: int, device) -> tuple[tuple[torch.Tensor, ...], list]:
        """A free slot and its (off int64, len int32, label int32) views."""
        free = [s for s in self.slots if s[1] is None or s[1]() is None]
        need = 16 * max(1, n_records)
        fits = [s for s in free if s[2] is not None and s[2].numel() >= need]
        if fits:
            slot = min(fits, key=lambda s: s[2].numel())
        elif free:
            slot = max(free, key=lambda s: 0 if s[0] is None else s[0].numel())
        else:
            slot = [None, None, None, None]
            self.slots.append(slot)
        if slot[2] is None or slot[2].numel() < need:
            slot[2] = None
            slot[2] = torch.empty(int(need * self.HEADROOM) + 64, dtype=torch.uint8, device=device)
        n = max(1, n_records)
        raw = slot[2]
        off = raw[: 8 * n].view(torch.int64)
        ln = raw[8 * n: 12 * n].view(torch.int32)
        lb = raw[12 * n: 16 * n].view(torch.int32)
        slot[1] = None
        return (off, ln, lb), slot

    def blob(self, slot: list, nbytes: int, device) -> torch.Tensor:
        if slot[0] is None or slot[0].numel() < nbytes:
            slot[0] = None
            slot[0] = torch.empty(max(1, int(nbytes * self.HEADROOM)), dtype=torch.uint8,
                                  device=device)
        return slot[0][: max(1, nbytes)]

    SENDLIST_HEAD = 1024  # begin[S + 1] first, at the same offset on every rank

    def sendlist(self, slot: list, n_final: int, S: int, device):
        """The receiver's begin[S + 1] array and send list (24-byte entries,
        md_shuffle_sendlist) in one peer-registrable allocation per slot:
        begin at offset 0 and the list at SENDLIST_HEAD, so a peer finds both
        from the base address whatever this rank's record count."""
        need = self.SENDLIST_HEAD + 24 * max(1, n_final)
        if slot[3] is None or slot[3].numel() < need:
            slot[3] = None
            slot[3] = torch.empty(int(need * self.HEADROOM) + 64, dtype=torch.uint8,
                                  device=device)
        raw = slot[3]
        return raw, raw[self.SENDLIST_HEAD: need], raw[: 8 * (S + 1)].view(torch.int64)

    @staticmethod
    def bind(slot: list, store) -> None:
        import weakref

        slot[1] = weakref.ref(store)


def _arena(ep) -> _ShardArena:
    ar = getattr(ep, "_shard_arena", None)
    if ar is None:
        ar = _ShardArena()
        ep._shard_arena = ar
    return ar


class _PhaseClock:
    """Host wall time per shuffle phase (MD_DIMD_TIMING=1: synchronizes
    between phases and records into LAST_SHUFFLE_PHASES)."""

    def __init__(self, dev):
        import os
        import time

        self.on = os.environ.get("MD_DIMD_TIMING") == "1"
        self.dev, self.time = dev, time
        self.t = time.perf_counter()
        if self.on:
            LAST_SHUFFLE_PHASES.clear()

    def __call__(self, name: str) -> None:
        if not self.on:
            return
        torch.cuda.synchronize(self.dev)
        now = self.time.perf_counter()
        LAST_SHUFFLE_PHASES[name] = now - self.t
        self.t = now


def _side_stream(ep) -> torch.cuda.Stream:
    st = getattr(ep, "_dimd_side_stream", None)
    if st is None:
        st = torch.cuda.Stream(device=ep.torch_device)
        ep._dimd_side_stream = st
    return st


def _shuffle(ep, store: ShardStore, m_segments, seed: int, next_seed: int | None = None
             ) -> ShardStore:
    S = store.group_size
    if S > _lib.MD_MAX_GROUP:
        raise InvalidConfig(f"group size {S} exceeds {_lib.MD_MAX_GROUP}")
    if m_segments is None:
        m_segments = default_segments(store.nbytes)
    if m_segments < 1:
        raise InvalidConfig(f"m_segments must be >= 1, got {m_segments}")
    if store.n_records and int((store.length.to(torch.int64) & 0xFFFFFFFF).max().item()) >= _MAX_RECORD:
        raise SegmentOverflow(f"a record reaches {_MAX_RECORD} bytes; no exchange slice may")
    dev = store.device
    first = store.group_id * S
    members = list(range(first, first + S))
    # make every source's shard visible (sync: the blob must be complete)
    torch.cuda.current_stream(dev).synchronize()
    mark = _PhaseClock(dev)
    # one host collective: the members' record counts (group_record_counts)
    # and every source's shard arrays, mapped into this process
    empty = store.n_records == 0
    arrays = [store.blob,
              torch.zeros(1, dtype=torch.int64, device=dev) if empty else store.off,
              torch.zeros(1, dtype=torch.int32, device=dev) if empty else store.length,
              torch.zeros(1, dtype=torch.int32, device=dev) if empty else store.label]
    lib = _lib.load()
    s = _stream(dev)

    def plan(n_rec, key=seed, stream=s):
        cap = max(1, sum(n_rec))
        fm = torch.empty(cap, dtype=torch.int32, device=dev)
        fr = torch.empty(cap, dtype=torch.int64, device=dev)
        nf = C.c_int64()
        nxt = (C.c_int64 * S)()
        _lib.check(lib.md_shuffle_plan(
            key & _MASK64, store.group_id, S, store.rank_in_group, ep.rank, int(m_segments),
            (C.c_int64 * S)(*n_rec), fm.data_ptr(), fr.data_ptr(), cap, C.byref(nf), nxt, stream))
        return fm, fr, int(nf.value), [int(x) for x in nxt]

    def plan_key(key):
        return (key & _MASK64, store.group_id, S, store.rank_in_group, ep.rank, int(m_segments))

    meta = (int(store.n_records), int(m_segments))
    pre = getattr(store, "_prefetched", None)  # (key, counts, plan) from the previous epoch
    pred = getattr(store, "_next_counts", None)
    if pred is not None and (len(pred) != S or pred[store.rank_in_group] != store.n_records):
        pred = None
    if pre is not None and pre[0] == plan_key(seed):
        # planned during the previous exchange (next_seed): only the counts'
        # collective remains, and a changed count re-plans
        (v_blob, v_off, v_len, v_lab), rows = ep.register_varlen_many(arrays, meta)
        n_rec = _group_counts(rows, members, int(m_segments))
        fm, fr, n_final, next_counts = pre[2] if n_rec == pre[1] else plan(n_rec)
        for t in (fm, fr):  # allocated on the side stream, used on this one
            t.record_stream(torch.cuda.current_stream(dev))
        mark("register (plan prefetched)")
    elif pred is None:
        (v_blob, v_off, v_len, v_lab), rows = ep.register_varlen_many(arrays, meta)
        n_rec = _group_counts(rows, members, int(m_segments))
        mark("register")
        fm, fr, n_final, next_counts = plan(n_rec)
        mark("plan")
    else:
        # the previous shuffle's plan already counted every member's records
        # (md_shuffle_plan next_counts): plan on this thread (the C call drops
        # the GIL) while the host collective runs on a helper thread, then check
        # the prediction against the gathered counts
        box: dict = {}

        def register():
            try:
                torch.cuda.set_device(dev)  # IPC imports map into the current device
                box["r"] = ep.register_varlen_many(arrays, meta)
            except BaseException as e:  # noqa: BLE001  (re-raised on the caller's thread)
                box["e"] = e

        th = threading.Thread(target=register, daemon=True)
        th.start()
        try:
            planned = plan(pred)
        finally:
            th.join()
        if "e" in box:
            raise box["e"]
        (v_blob, v_off, v_len, v_lab), rows = box["r"]
        n_rec = _group_counts(rows, members, int(m_segments))
        if n_rec != pred:
            planned = plan(n_rec)
        fm, fr, n_final, next_counts = planned
        mark("register+plan")
    arena = _arena(ep)
    (off, ln, lb), slot = arena.take(n_final, dev)
    total = C.c_uint64()
    _lib.check(
        lib.md_shuffle_index(
            S, _lib.ptr_array([v_len.ptrs[m] for m in members]),
            _lib.ptr_array([v_lab.ptrs[m] for m in members]), fm.data_ptr(), fr.data_ptr(),
            n_final, off.data_ptr(), ln.data_ptr(), lb.data_ptr(), C.byref(total), s,
        )
    )
    mark("index")
    blob = arena.blob(slot, int(total.value), dev)
    if EXCHANGE == "push":
        # receiver side: our output slots grouped by source member; then one
        # host collective publishes (new blob, send list) to every source
        raw, lst, begin = arena.sendlist(slot, n_final, S, dev)
        _lib.check(lib.md_shuffle_sendlist(S, fm.data_ptr(), fr.data_ptr(), n_final,
                                           off.data_ptr(), ln.data_ptr(), lst.data_ptr(),
                                           begin.data_ptr(), s))
        torch.cuda.current_stream(dev).synchronize()  # lists complete before peers read them
        (v_out, v_list), _ = ep.register_varlen_many([blob, raw])
        mark("sendlist")
        beg_ptrs = [v_list.ptrs[m] for m in members]
        lst_ptrs = [p + _ShardArena.SENDLIST_HEAD for p in beg_ptrs]
        _lib.check(lib.md_shuffle_push(
            S, store.rank_in_group, store.blob.data_ptr(),
            (store.off if not empty else arrays[1]).data_ptr(),
            _lib.ptr_array(lst_ptrs), _lib.ptr_array(beg_ptrs),
            _lib.ptr_array([v_out.ptrs[m] for m in members]), s))
    else:
        _lib.check(
            lib.md_shuffle_pull(
                S, _lib.ptr_array([v_blob.ptrs[m] for m in members]),
                _lib.ptr_array([v_off.ptrs[m] for m in members]), fm.data_ptr(), fr.data_ptr(),
                n_final, off.data_ptr(), ln.data_ptr(), blob.data_ptr(), s,
            )
        )
    prefetched = None
    if next_seed is not None:
        # the next epoch's plan, on a side stream while the bytes move (the
        # exchange kernel leaves room on every SM for the plan's kernels)
        side = _side_stream(ep)
        box: dict = {}

        def prefetch():
            try:
                torch.cuda.set_device(dev)
                with torch.cuda.stream(side):
                    box["p"] = plan(next_counts, next_seed, _lib.stream_ptr(side))
                side.synchronize()
            except BaseException as e:  # noqa: BLE001  (no prefetch: the next epoch plans)
                box["e"] = e

        th = threading.Thread(target=prefetch, daemon=True)
        th.start()
    torch.cuda.current_stream(dev).synchronize()
    mark(EXCHANGE)
    if next_seed is not None:
        th.join()
        if "p" in box:
            prefetched = (plan_key(next_seed), next_counts, box["p"])
    # pull: every read of our old shard is done before anyone frees it;
    # push: every record pushed into our new blob has landed
    ep.barrier()
    mark("barrier")
    out = ShardStore(blob, off[:n_final], ln[:n_final], lb[:n_final], store.group_id, S,
                     store.rank_in_group)
    out._nbytes = int(total.value)
    out._next_counts = next_counts  # lets the next shuffle plan while its counts travel
    out._prefetched = prefetched
    _ShardArena.bind(slot, out)
    return out


def shuffle_plan_device(seed: int, group_id: int, S: int, member: int, global_rank: int,
                        m_segments: int, n_rec, device=None) -> tuple[torch.Tensor, torch.Tensor]:
    """The index half of the shuffle alone (md_shuffle_plan): (source member,
    source record) of every output slot, on device. Needs only record counts,
    so index parity can be checked at full corpus size without the bytes."""
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    cap = max(1, int(sum(n_rec)))
    fm = torch.empty(cap, dtype=torch.int32, device=device)
    fr = torch.empty(cap, dtype=torch.int64, device=device)
    nf = C.c_int64()
    arr = (C.c_int64 * S)(*[int(x) for x in n_rec])
    _lib.check(
        _lib.load().md_shuffle_plan(
            seed & _MASK64, group_id, S, member, global_rank, int(m_segments), arr,
            fm.data_ptr(), fr.data_ptr(), cap, C.byref(nf), None, _stream(device),
        )
    )
    return fm[: nf.value], fr[: nf.value]


# -- synthetic corpus on device (bench / tests) ------------------------------------------------


def synth_store(n_local: int, rec_bytes: int, first_gid: int, gid_stride: int, seed: int,
                group_id: int, group_size: int, rank_in_group: int, device=None,
                n_labels: int = 1000) -> ShardStore:
    """Shard of a synthetic corpus generated in HBM: local record j is global
    record ``first_gid + j * gid_stride`` (striping, dimd.py:192)."""
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    blob = torch.empty(max(1, n_local * rec_bytes), dtype=torch.uint8, device=device)
    off = torch.empty(n_local, dtype=torch.int64, device=device)
    ln = torch.empty(n_local, dtype=torch.int32, device=device)
    lb = torch.empty(n_local, dtype=torch.int32, device=device)
    _lib.check(
        _lib.load().md_synth_records(
            blob.data_ptr(), off.data_ptr(), ln.data_ptr(), lb.data_ptr(), n_local, rec_bytes,
            first_gid, gid_stride, seed & _MASK64, n_labels, _stream(device),
        )
    )
    st = ShardStore(blob, off, ln, lb, group_id, group_size, rank_in_group)
    st._nbytes = n_local * rec_bytes
    return st


def synth_verify(store: ShardStore, seed: int, n_labels: int = 1000) -> tuple[int, torch.Tensor]:
    """(number of corrupt records, gid of every slot) of a synthetic shard."""
    n = store.n_records
    gids = torch.empty(max(1, n), dtype=torch.int64, device=store.device)
    bad = C.c_int64()
    _lib.check(
        _lib.load().md_synth_verify(
            store.blob.data_ptr(), store.off.data_ptr(), store.length.data_ptr(),
            store.label.data_ptr(), n, seed & _MASK64, n_labels, gids.data_ptr(), C.byref(bad),
            _stream(store.device),
        )
    )
    return int(bad.value), gids[:n]
