"""Remaining API surface on the GPU: alltoallv (collectives.py:475-525 cases of
pkg/tests/test_collectives.py:279-339), elementwise_add, load_partition from
disk (dimd.py:203-207)."""

import numpy as np
import pytest
import torch

from paper_1711_00705_b200 import GradientBuffer, VarPayload, alltoallv, errors, run_ranks
from paper_1711_00705_b200.collectives import elementwise_add
from paper_1711_00705_b200.dimd import IndexEntry, Record, build_blob, load_partition

pytestmark = pytest.mark.gpu


def test_alltoallv_two_rank_swap_and_empty():
    def prog(ep):
        send = VarPayload.from_slices([b"", b"ab"] if ep.rank == 0 else [b"xyz", b""])
        return bytes(alltoallv(ep, send).slice_for(1 - ep.rank))

    assert run_ranks(2, "cuda", prog, emulate=True).results == [b"xyz", b"ab"]
    res = run_ranks(4, "cuda", lambda ep: alltoallv(ep, VarPayload.from_slices([b""] * 4)).data,
                    emulate=True).results
    assert res == [b""] * 4


def test_alltoallv_matches_transpose_host_and_device():
    rng = np.random.default_rng(15)
    mats = [[rng.bytes(int(rng.integers(0, 2000))) for _ in range(4)] for _ in range(4)]
    want = [b"".join(mats[src][dst] for src in range(4)) for dst in range(4)]
    res = run_ranks(4, "cuda", lambda ep: alltoallv(ep, VarPayload.from_slices(mats[ep.rank])).data,
                    emulate=True).results
    assert res == want

    def dev_prog(ep):
        p = VarPayload.from_slices(mats[ep.rank])
        t = torch.frombuffer(bytearray(p.data), dtype=torch.uint8).to(ep.torch_device)
        out = alltoallv(ep, VarPayload(t, p.offsets, p.lengths))
        return bytes(out.data.cpu().numpy().tobytes())

    assert run_ranks(4, "cuda", dev_prog, emulate=True).results == want


def test_alltoallv_self_slice_and_validation():
    def prog(ep):
        slices = [b""] * 4
        slices[ep.rank] = f"keep {ep.rank}".encode()
        return bytes(alltoallv(ep, VarPayload.from_slices(slices)).slice_for(ep.rank))

    assert run_ranks(4, "cuda", prog, emulate=True).results == [f"keep {r}".encode() for r in range(4)]

    def bad(ep):
        with pytest.raises(errors.LengthMismatch):
            alltoallv(ep, VarPayload.from_slices([b"x"]))

    run_ranks(2, "cuda", bad, emulate=True)


def test_elementwise_add_on_device():
    a = GradientBuffer.of([1, 2], device="cuda")
    elementwise_add(a, GradientBuffer.of([10, 20], device="cuda"))
    assert a.data.cpu().tolist() == [11.0, 22.0]
    with pytest.raises(errors.LengthMismatch):
        elementwise_add(a, GradientBuffer.zeros(3, device="cuda"))


def test_load_partition_from_files(tmp_path):
    rng = np.random.default_rng(5)
    recs = [Record(bytes(rng.integers(0, 256, size=int(rng.integers(1, 40)), dtype=np.uint8)),
                   int(rng.integers(0, 1000))) for _ in range(100)]
    blob, idx = build_blob(recs)
    (tmp_path / "d.blob").write_bytes(blob)
    (tmp_path / "d.idx").write_bytes(idx)
    dev = torch.device("cuda", 0)
    store = load_partition(tmp_path / "d.blob", tmp_path / "d.idx", 0, 1, 1, device=dev)
    assert store.records() == recs
    s1 = load_partition(tmp_path / "d.blob", tmp_path / "d.idx", 1, 2, 2, device=dev)
    assert s1.records() == recs[1::2]
    assert s1.index[0] == IndexEntry(0, len(recs[1].bytes), recs[1].label)
    with pytest.raises(errors.IoError):
        load_partition(tmp_path / "missing.blob", tmp_path / "d.idx", 0, 1, 1, device=dev)
