"""The CUDA endpoint: one rank's handle on its GPU, its peers and its comm.

Mirrors the role of the reference endpoints (``rank``, ``n_ranks``,
``max_segment`` -- /root/reference/pkg/src/minidist/transport/base.py:265-313)
but the data path is device memory:

* mode ``"p2p"``: one GPU per rank. Peers' buffers are mapped into this
  process -- directly (cudaDeviceEnablePeerAccess) when the ranks are threads
  of one process, through CUDA IPC handles when they are processes
  (torchrun). NVLink/NVSwitch carries every load.
* mode ``"emulated"``: all ranks of the world share ONE GPU (a 1-GPU box or
  tests). Collectives whose CTAs wait on each other are launched once for
  all ranks through a ``Rendezvous`` so every CTA is co-resident.

Registration (``register``) is the B200 replacement for ``expose``: it makes
a tensor addressable by every peer. It is collective and cached.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import torch

from paper_1711_00705_b200 import _lib
from paper_1711_00705_b200.errors import InvalidConfig, LengthMismatch, PeerUnreachable

DEFAULT_MAX_SEGMENT = 4 * 1024 * 1024  # transport/base.py:26, kept for API parity
DEFAULT_PULL_TIMEOUT = 30.0            # transport/base.py:28 -> device watchdog


@dataclass
class PeerView:
    """Every rank's address of one registered tensor, as seen from here."""

    ptrs: list[int]
    nbytes: int
    keep: object = field(default=None, repr=False)  # the local tensor


class _ImportCache:
    """IPC imports are per process; one mapping per exported allocation."""

    def __init__(self):
        self.lock = threading.Lock()
        self.bases: dict[bytes, int] = {}

    def get(self, handle: bytes) -> int:
        with self.lock:
            base = self.bases.get(handle)
            if base is None:
                out = C.c_void_p()
                rc = _lib.load().md_mem_import(handle, C.byref(out))
                if rc != 0:
                    raise PeerUnreachable(_lib.load().md_last_error().decode())
                base = int(out.value)
                self.bases[handle] = base
            return base


_IMPORTS = _ImportCache()


class CudaEndpoint:
    """One rank. Construction is collective over ``channel``."""

    def __init__(
        self,
        rank: int,
        n_ranks: int,
        device: int,
        channel,
        *,
        mode: str = "p2p",
        multiprocess: bool = False,
        rendezvous=None,
        stream: torch.cuda.Stream | None = None,
        max_segment: int = DEFAULT_MAX_SEGMENT,
        pull_timeout: float = DEFAULT_PULL_TIMEOUT,
    ):
        if mode not in ("p2p", "emulated"):
            raise InvalidConfig(f"unknown endpoint mode {mode!r}")
        self.rank = rank
        self.n_ranks = n_ranks
        self.device = device
        self.channel = channel
        self.mode = mode
        self.multiprocess = multiprocess
        self.rendezvous = rendezvous
        self.max_segment = max_segment
        self.lib = _lib.load()
        self.torch_device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.torch_device)
        self._plans: dict = {}
        self._views: dict = {}
        self._staging: dict = {}
        self.closed = False

        comm = C.c_void_p()
        with torch.cuda.device(device):
            _lib.check(self.lib.md_comm_create(rank, n_ranks, device, C.byref(comm)))
        self.comm = comm
        _lib.check(self.lib.md_comm_set_timeout(self.comm, float(pull_timeout)))
        ctrl = C.c_void_p()
        _lib.check(self.lib.md_comm_ctrl_ptr(self.comm, C.byref(ctrl)))
        self._ctrl_ptr = int(ctrl.value)
        # control blocks of every rank, mapped here
        peers = self._exchange_pointer(self._ctrl_ptr, 0)
        _lib.check(self.lib.md_comm_set_peer_ctrl(self.comm, _lib.ptr_array(peers), n_ranks))

    # -- host collectives ---------------------------------------------------------------
    def all_gather(self, obj) -> list:
        return self.channel.all_gather(obj)

    def barrier(self) -> None:
        self.channel.barrier()

    # -- peer memory -------------------------------------------------------------------
    def _exchange_pointer(self, ptr: int, nbytes: int) -> list[int]:
        """Every rank's address of a tensor at ``ptr``, mapped into this process."""
        if self.n_ranks == 1:
            return [ptr]
        if self.multiprocess:
            handle = C.create_string_buffer(_lib.IPC_BYTES)
            off = C.c_uint64()
            _lib.check(self.lib.md_mem_export(C.c_void_p(ptr), handle, C.byref(off)))
            rows = self.all_gather((nbytes, bytes(handle.raw), int(off.value), ptr))
            out = []
            for r, (nb, h, o, p) in enumerate(rows):
                out.append(p if r == self.rank else _IMPORTS.get(h) + o)
            return out
        if self.mode == "p2p":
            self._enable_peers()
        rows = self.all_gather((nbytes, None, 0, ptr))
        return [p for (_, _, _, p) in rows]

    def _exchange_pointers(self, items, extra=None):
        """``_exchange_pointer`` for several (ptr, nbytes) at once -- ONE host
        collective -- plus an optional per-rank payload gathered alongside.
        Returns (per item: every rank's address, per rank: its payload)."""
        if self.n_ranks == 1:
            return [[p] for p, _ in items], [extra]
        if self.multiprocess:
            mine = []
            for ptr, nbytes in items:
                handle = C.create_string_buffer(_lib.IPC_BYTES)
                off = C.c_uint64()
                _lib.check(self.lib.md_mem_export(C.c_void_p(ptr), handle, C.byref(off)))
                mine.append((nbytes, bytes(handle.raw), int(off.value), ptr))
            rows = self.all_gather((mine, extra))
            out = []
            for i in range(len(items)):
                out.append([row[i][3] if r == self.rank else _IMPORTS.get(row[i][1]) + row[i][2]
                            for r, (row, _) in enumerate(rows)])
            return out, [e for _, e in rows]
        if self.mode == "p2p":
            self._enable_peers()
        rows = self.all_gather(([p for p, _ in items], extra))
        return [[row[0][i] for row in rows] for i in range(len(items))], [row[1] for row in rows]

    _peers_enabled = False

    def _enable_peers(self) -> None:
        if CudaEndpoint._peers_enabled:
            return
        n = C.c_int()
        _lib.check(self.lib.md_device_count(C.byref(n)))
        for a in range(n.value):
            for b in range(n.value):
                if a != b:
                    _lib.check(self.lib.md_enable_peer_access(a, b))
        CudaEndpoint._peers_enabled = True

    def register(self, tensor: torch.Tensor) -> PeerView:
        """Collective: make ``tensor`` addressable by every rank.

        All ranks must call it with their counterpart tensors in the same
        order. Lengths are compared host-side (LengthMismatch), which is the
        reference's length-header exchange (collectives.py:157-174).
        """
        if tensor.device != self.torch_device:
            raise InvalidConfig(f"tensor on {tensor.device}, endpoint on {self.torch_device}")
        nbytes = tensor.numel() * tensor.element_size()
        ptr = tensor.data_ptr()
        if self.n_ranks > 1:
            sizes = self.all_gather(nbytes)
            if any(s != nbytes for s in sizes):
                raise LengthMismatch(f"ranks disagree on buffer length (bytes): {sizes}")
        if self.multiprocess and self.n_ranks > 1:
            # IPC export/import needs the allocation to be quiescent-safe only
            # in the sense that it stays alive; keep a reference to it
            torch.cuda.current_stream(self.torch_device).synchronize()
        ptrs = self._exchange_pointer(ptr, nbytes)
        return PeerView(ptrs, nbytes, tensor)

    def register_varlen(self, tensor: torch.Tensor) -> PeerView:
        """Like ``register`` but every rank may pass a different size (DIMD shards)."""
        nbytes = tensor.numel() * tensor.element_size()
        ptrs = self._exchange_pointer(tensor.data_ptr() if nbytes else 0, nbytes)
        return PeerView(ptrs, nbytes, tensor)

    def register_varlen_many(self, tensors, extra=None):
        """``register_varlen`` of several tensors in one host collective;
        ``extra`` (any picklable) is all-gathered with the handles."""
        items = []
        for t in tensors:
            if t.device != self.torch_device:
                raise InvalidConfig(f"tensor on {t.device}, endpoint on {self.torch_device}")
            nbytes = t.numel() * t.element_size()
            items.append((t.data_ptr() if nbytes else 0, nbytes))
        ptrs, extras = self._exchange_pointers(items, extra)
        return [PeerView(p, nb, t) for p, (_, nb), t in zip(ptrs, items, tensors)], extras

    def alloc(self, n: int, dtype=torch.float32) -> tuple[torch.Tensor, PeerView]:
        """Collective allocation of a peer-registered tensor (zeroed)."""
        t = torch.zeros(n, dtype=dtype, device=self.torch_device)
        torch.cuda.synchronize(self.torch_device)
        view = self.register(t)
        self._views[(t.data_ptr(), t.numel() * t.element_size())] = view
        return t, view

    # -- plans --------------------------------------------------------------------------
    def plan(self, tables, schedule: str = "tree", route: str = "auto",
             tile: int = 0) -> C.c_void_p:
        """Device plan for fold tables (cached per tables object, schedule and
        route: "tree" = the reference's per-color trees, "owner" =
        owner-computes slices with the same fold order, md_plan_set_schedule;
        ``route``/``tile`` pin md_allreduce's kernel, md_plan_set_route)."""
        opts = (schedule, route, int(tile))
        fast = self._plans.get((id(tables), opts))
        if fast is not None and fast[0] is tables:
            return fast[1]
        if route not in _lib.ROUTES or route == "local":
            raise InvalidConfig(f"unknown allreduce route {route!r}")
        key = (tables.key(), opts)
        p = self._plans.get(key)
        if p is None:
            p = C.c_void_p()
            with torch.cuda.device(self.device):
                _lib.check(
                    self.lib.md_plan_create(
                        tables.n_ranks,
                        tables.k,
                        tables.parent.ctypes.data_as(C.POINTER(C.c_int32)),
                        tables.child_ptr.ctypes.data_as(C.POINTER(C.c_int32)),
                        tables.child_idx.ctypes.data_as(C.POINTER(C.c_int32))
                        if tables.child_idx.size
                        else None,
                        tables.self_pos.ctypes.data_as(C.POINTER(C.c_int32)),
                        self.device,
                        C.byref(p),
                    )
                )
                sched = _lib.MD_SCHED_OWNER if schedule == "owner" else _lib.MD_SCHED_TREE
                _lib.check(self.lib.md_plan_set_schedule(p, sched))
                _lib.check(self.lib.md_plan_set_route(p, _lib.ROUTES[route], int(tile)))
            self._plans[key] = p
        self._plans[(id(tables), opts)] = (tables, p)
        return p

    def view_of(self, tensor: torch.Tensor) -> PeerView:
        """Peer view of a tensor registered once (collective on first use, then
        cached by address and size; the view keeps the tensor alive, so the
        address cannot be recycled): the sharded update's weights."""
        key = (tensor.data_ptr(), tensor.numel() * tensor.element_size())
        v = self._views.get(key)
        if v is None:
            v = self.register(tensor)
            self._views[key] = v
        return v

    # -- errors / sync -------------------------------------------------------------------
    def take_error(self) -> None:
        code, detail = C.c_int32(), C.c_int32()
        self.lib.md_comm_take_error(self.comm, C.byref(code), C.byref(detail))
        if code.value != 0:
            from paper_1711_00705_b200 import errors

            cls = errors.FROM_CODE.get(code.value, RuntimeError)
            raise cls(f"rank {self.rank}: device collective failed (code {code.value}, "
                      f"detail {detail.value})")

    def synchronize(self) -> None:
        self.stream.synchronize()
        self.take_error()

    def close(self) -> None:
        if self.closed:
            return
        self.closed = True
        try:
            torch.cuda.synchronize(self.torch_device)
        finally:
            for p in self._plans.values():
                if not isinstance(p, tuple):
                    self.lib.md_plan_destroy(p)
            self._plans.clear()
            self.lib.md_comm_destroy(self.comm)
