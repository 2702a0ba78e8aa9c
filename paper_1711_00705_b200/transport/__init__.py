"""Rank runtime of the B200 path: endpoints, host channels, run_ranks."""

from paper_1711_00705_b200.transport.channel import SubChannel, ThreadChannel, TorchChannel
from paper_1711_00705_b200.transport.endpoint import (
    DEFAULT_MAX_SEGMENT,
    DEFAULT_PULL_TIMEOUT,
    CudaEndpoint,
    PeerView,
)
from paper_1711_00705_b200.transport.runner import BACKENDS, RunResult, init_from_env, run_ranks


class SubCommunicator:
    """Rank-translated view of an endpoint over ``members``
    (transport/base.py:265-313): host collectives are restricted to the
    members; device work keeps using the parent endpoint's GPU and comm."""

    def __init__(self, ep, members):
        members = tuple(members)
        from paper_1711_00705_b200.errors import InvalidConfig

        if len(set(members)) != len(members):
            raise InvalidConfig("duplicate ranks in subcommunicator")
        if ep.rank not in members:
            raise InvalidConfig(f"rank {ep.rank} is not a member of {members}")
        if any(not 0 <= m < ep.n_ranks for m in members):
            raise InvalidConfig(f"member out of range in {members}")
        self._ep = ep
        self.members = members
        self.rank = members.index(ep.rank)
        self.n_ranks = len(members)
        self.max_segment = ep.max_segment
        self.channel = SubChannel(ep.channel, members)

    def all_gather(self, obj) -> list:
        return self.channel.all_gather(obj)

    def barrier(self) -> None:
        self.channel.barrier()

    def __getattr__(self, name):
        return getattr(self._ep, name)


__all__ = [
    "BACKENDS",
    "DEFAULT_MAX_SEGMENT",
    "DEFAULT_PULL_TIMEOUT",
    "CudaEndpoint",
    "PeerView",
    "RunResult",
    "SubCommunicator",
    "SubChannel",
    "ThreadChannel",
    "TorchChannel",
    "init_from_env",
    "run_ranks",
]
