"""N > 1 host logic with one process per rank over gloo (CPU, world_size 2
and 4): the control channel, sub-group restriction, the shuffle's count
agreement, and -- with the oracle -- that the per-receiver shuffle plans of
all ranks partition the corpus exactly (every record lands once)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_1711_00705_b200.dimd import group_record_counts
        from paper_1711_00705_b200.errors import InvalidConfig
        from paper_1711_00705_b200.transport import SubChannel, TorchChannel

        ch = TorchChannel()
        out = {"gather": ch.all_gather(rank * 10)}
        half = [r for r in range(world) if r % 2 == rank % 2]
        out["sub"] = SubChannel(ch, half).all_gather(rank)
        # shuffle host step: counts gathered, m_segments agreement enforced
        n_local = 1000 + 37 * rank
        counts = group_record_counts(ch, list(range(world)), n_local, 3)
        out["counts"] = counts
        try:
            group_record_counts(ch, list(range(world)), n_local, 3 + (rank == 1))
            out["disagree"] = "no error"
        except InvalidConfig:
            out["disagree"] = "InvalidConfig"
        # every receiver plans its own shard; the plans partition the corpus
        mem, rec = O.shuffle_plan_c(77, 0, world, rank, rank, 3, counts)
        out["plan"] = (mem.tolist(), rec.tolist())
        ch.barrier()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_host_path(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r]["gather"] == [10 * x for x in range(world)]
        assert res[r]["sub"] == [x for x in range(world) if x % 2 == r % 2]
        assert res[r]["counts"] == [1000 + 37 * x for x in range(world)]
        assert res[r]["disagree"] == "InvalidConfig"
    seen = set()
    for r in range(world):
        mem, rec = res[r]["plan"]
        for q_, i in zip(mem, rec):
            assert (q_, i) not in seen
            seen.add((q_, i))
    assert len(seen) == sum(1000 + 37 * x for x in range(world))
    assert np.all(np.array([len(res[r]["plan"][0]) for r in range(world)]) > 0)
