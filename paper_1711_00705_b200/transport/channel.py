"""Host-side control channels between ranks.

The reference moves every control message (length headers, hash verdicts,
alltoallv length tables) over its endpoint's send/recv
(/root/reference/pkg/src/minidist/transport/base.py). On the B200 path the
data never touches the host; what remains host-side is rare, small metadata
(IPC handles at registration, the per-call length table for unregistered
buffers, shuffle record counts). A channel offers exactly two collective
operations: ``all_gather(obj)`` and ``barrier()``.

* ``ThreadChannel``: ranks are threads of one process (run_ranks "cuda").
* ``TorchChannel``: one process per rank (torchrun), over a torch.distributed
  group (gloo on CPU, so it works in this container's multi-process tests).
"""

from __future__ import annotations

import threading
import time

from paper_1711_00705_b200.errors import Closed


class Board:
    """Shared rendezvous state for the threads of one run."""

    def __init__(self, n: int, timeout: float = 120.0):
        self.n = n
        self.timeout = timeout
        self.slots: list = [None] * n
        self.barrier = threading.Barrier(n)
        self.error: BaseException | None = None
        self.lock = threading.Lock()

    def abort(self, err: BaseException) -> None:
        with self.lock:
            if self.error is None:
                self.error = err
        self.barrier.abort()


class ThreadChannel:
    def __init__(self, board: Board, rank: int):
        self.board = board
        self.rank = rank
        self.n_ranks = board.n

    def _wait(self) -> None:
        try:
            self.board.barrier.wait(timeout=self.board.timeout)
        except threading.BrokenBarrierError:
            raise Closed(f"rank {self.rank}: peer failed: {self.board.error!r}") from None

    def all_gather(self, obj) -> list:
        self.board.slots[self.rank] = obj
        self._wait()
        out = list(self.board.slots)
        self._wait()
        return out

    def barrier(self) -> None:
        self._wait()


class TorchChannel:
    def __init__(self, group=None):
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.n_ranks = dist.get_world_size(group)

    def all_gather(self, obj) -> list:
        out = [None] * self.n_ranks
        self._dist.all_gather_object(out, obj, group=self.group)
        return out

    def barrier(self) -> None:
        self._dist.barrier(group=self.group)


class SubChannel:
    """A channel restricted to ``members``; every world rank must call the
    collective at the same time (each with its own member list)."""

    def __init__(self, parent, members):
        self.parent = parent
        self.members = tuple(members)
        self.rank = self.members.index(parent.rank)
        self.n_ranks = len(self.members)

    def all_gather(self, obj) -> list:
        everyone = self.parent.all_gather(obj)
        return [everyone[m] for m in self.members]

    def barrier(self) -> None:
        self.parent.barrier()


class Rendezvous:
    """Collective kernel launch for ranks emulated on ONE GPU.

    Kernels that wait on each other must run as one launch on one device
    (co-resident CTAs); each rank thread deposits its arguments, the last one
    to arrive runs ``fn(list_of_args)`` and everybody gets its result.
    """

    def __init__(self, n: int, timeout: float = 120.0):
        self.n = n
        self.timeout = timeout
        self.cv = threading.Condition()
        self.args: list = [None] * n
        self.count = 0
        self.gen = 0
        self.result = None
        self.error: BaseException | None = None
        self.aborted: BaseException | None = None

    def abort(self, err: BaseException) -> None:
        with self.cv:
            self.aborted = err
            self.cv.notify_all()

    def run(self, rank: int, arg, fn):
        with self.cv:
            if self.aborted is not None:
                raise Closed(f"rank {rank}: peer failed: {self.aborted!r}")
            gen = self.gen
            self.args[rank] = arg
            self.count += 1
            if self.count == self.n:
                try:
                    self.result, self.error = fn(list(self.args)), None
                except BaseException as e:  # noqa: BLE001 - handed to every rank
                    self.result, self.error = None, e
                self.count = 0
                self.args = [None] * self.n
                self.gen += 1
                self.cv.notify_all()
            else:
                deadline = time.monotonic() + self.timeout
                while self.gen == gen and self.aborted is None:
                    left = deadline - time.monotonic()
                    if left <= 0:
                        raise Closed(f"rank {rank}: collective rendezvous timed out")
                    self.cv.wait(timeout=min(left, 1.0))
                if self.gen == gen:
                    raise Closed(f"rank {rank}: peer failed: {self.aborted!r}")
            if self.error is not None:
                raise self.error
            return self.result
