"""Host-side API parity with the reference (CPU only): LR schedule values,
DIMD codec bytes and validation, config validation, VarPayload, segment
schedule, GradientBuffer constructors. Mirrors pkg/tests/test_{sgd,dimd,
collectives}.py cases that do not need a device."""

import math

import numpy as np
import pytest
from hypothesis import given
from hypothesis import strategies as st

from paper_1711_00705_b200 import errors
from paper_1711_00705_b200.collectives import GradientBuffer, VarPayload, make_segment_schedule
from paper_1711_00705_b200.dimd import (
    IndexEntry,
    Record,
    _mix64,
    _mix64_py,
    build_blob,
    default_segments,
    parse_index,
)
from paper_1711_00705_b200.sgd import LrSchedule, TrainConfig, comm_plan, lr_at, lr_schedule


def test_lr_schedule_matches_reference_values(golden):
    for base, k, n, epoch, want in golden["lr_rows"]:
        cfg = TrainConfig(n_nodes=1, workers_per_node=int(n), per_worker_batch=int(k), epochs=1,
                          base_lr=float(base))
        assert lr_at(lr_schedule(cfg), float(epoch)) == want


def test_lr_targets_and_drops():
    s = LrSchedule(0.1, k=32, n=256, warmup_epochs=5, drop_every=30, drop_factor=10.0)
    assert lr_at(s, 5.0) == 3.2 and lr_at(s, 0.0) == 0.1
    assert abs(lr_at(s, 35.0) - 0.32) < 1e-12 and abs(lr_at(s, 65.0) - 0.032) < 1e-13
    with pytest.raises(errors.InvalidConfig):
        lr_at(s, -0.1)


@given(st.floats(0, 200), st.floats(0.001, 2), st.integers(1, 512), st.integers(1, 512))
def test_lr_positive_and_bounded(epoch, base, k, n):
    s = LrSchedule(base, k=k, n=n, warmup_epochs=5, drop_every=30, drop_factor=10.0)
    assert 0 < lr_at(s, epoch) <= max(base, base * k * n / 256) + 1e-12


def test_train_config_validation():
    for bad in (dict(n_nodes=0), dict(workers_per_node=0), dict(per_worker_batch=0), dict(epochs=0),
                dict(base_lr=0.0), dict(drop_factor=1.0), dict(momentum=1.0), dict(weight_decay=-1)):
        kw = dict(n_nodes=1, workers_per_node=1, per_worker_batch=1, epochs=1) | bad
        with pytest.raises(errors.InvalidConfig):
            TrainConfig(**kw)
    assert TrainConfig(n_nodes=4, workers_per_node=2, per_worker_batch=8, epochs=1).effective_batch == 64


def test_comm_plan_adapts_color_count():
    ts, ring = comm_plan(4, "multicolor")
    assert ts.k == 4 and ring is None
    ts6, _ = comm_plan(6, "multicolor")
    assert ts6.k in (1, 2)
    tsr, ring4 = comm_plan(4, "ring")
    assert tsr is None and ring4.order == (0, 1, 2, 3)
    assert comm_plan(1, "multicolor") == (None, None)


def test_codec_matches_reference_bytes(golden):
    blob, index = golden["codec_blob"].tobytes(), golden["codec_index"].tobytes()
    entries = parse_index(index)
    recs = [Record(blob[e.offset : e.offset + e.length], e.label) for e in entries]
    assert build_blob(recs) == (blob, index)


def test_codec_small_exact_and_errors():
    blob, index = build_blob([Record(b"hello", 3)])
    assert blob == b"hello" and index[:4] == b"DIMD"
    assert parse_index(index) == [IndexEntry(0, 5, 3)]
    assert build_blob([]) == (b"", build_blob([])[1]) and parse_index(build_blob([])[1]) == []
    with pytest.raises(errors.InvalidConfig):
        build_blob([Record(b"", 0)])
    with pytest.raises(errors.InvalidConfig):
        build_blob([Record(b"x", 1 << 32)])

    class Huge:
        def __len__(self):
            return 1 << 31

    with pytest.raises(errors.RecordTooLarge):
        build_blob([Record(Huge(), 0)])
    _, idx = build_blob([Record(b"ab", 1)])
    for bad in (b"DIMX" + idx[4:], idx[:-3], idx + b"\0" * 16, b""):
        with pytest.raises(errors.FormatError):
            parse_index(bad)
    v = bytearray(idx)
    v[4] = 99
    with pytest.raises(errors.FormatError):
        parse_index(bytes(v))


def test_default_segments_and_mix64(golden):
    assert [default_segments(x) for x in (0, 1, 1 << 30, (1 << 30) + 1, 10 << 30)] == [1, 1, 1, 2, 10]
    for parts, n, want in zip(golden["mix64_parts"], golden["mix64_n"], golden["mix64_out"]):
        p = [int(x) for x in parts[:n]]
        assert _mix64(*p) == int(want) == _mix64_py(*p)


def test_var_payload_validation():
    p = VarPayload.from_slices([b"ab", b"c"])
    p.validate(2)
    assert bytes(p.slice_for(1)) == b"c"
    with pytest.raises(errors.LengthMismatch):
        p.validate(3)
    with pytest.raises(errors.LengthMismatch):
        VarPayload(b"abc", (0, 2), (2, 2)).validate(2)
    with pytest.raises(errors.LengthMismatch):
        VarPayload(b"abc", (0, 1), (1, -1)).validate(2)
    with pytest.raises(errors.OffsetOverflow):
        VarPayload(b"", (0, 0), (0, 1 << 31)).validate(2)


@given(st.integers(0, 5000), st.integers(1, 8), st.sampled_from([1, 7, 64, 16384]))
def test_segment_schedule_covers_every_chunk(payload_len, k, seg):
    sched = make_segment_schedule(payload_len, k, seg)
    covered = 0
    for segs in sched.per_color:
        for lo, hi in segs:
            assert 0 < hi - lo <= seg
            covered += hi - lo
        for (_, a_hi), (b_lo, _) in zip(segs, segs[1:]):
            assert a_hi == b_lo
    assert covered == payload_len and len(sched.per_color) == k


def test_segment_schedule_rejects_absurd_counts():
    with pytest.raises(errors.InvalidConfig):
        make_segment_schedule(1 << 22, 1, 1)
    with pytest.raises(errors.InvalidConfig):
        make_segment_schedule(100, 1, 0)


def test_gradient_buffer_host_constructors():
    assert GradientBuffer.zeros(5).data.tolist() == [0.0] * 5
    b = GradientBuffer.of([1, 2, 3])
    assert b.data.dtype == np.float32 and b.len == 3 and not b.on_device
    a = GradientBuffer.alloc(1024)
    assert a.len == 1024
    with pytest.raises(errors.InvalidConfig):
        GradientBuffer(np.zeros(4, dtype=np.float64))
    with pytest.raises(errors.InvalidConfig):
        GradientBuffer(np.zeros((2, 2), dtype=np.float32))
    c = GradientBuffer(np.arange(8, dtype=np.float32)[::2])
    assert c.data.flags.c_contiguous and c.data.tolist() == [0.0, 2.0, 4.0, 6.0]
    assert math.isfinite(float(c.data.sum()))


def test_metrics_csv_format():
    """metrics_csv (sgd.py:545-556): header + one row per step, %.6g fields."""
    from paper_1711_00705_b200.sgd import EpochMetrics, StepStats, TrainResult, metrics_csv

    steps = [StepStats(step=i, epoch=i / 3, lr=0.1 * (i + 1), loss=1.0 / (i + 1), correct=i,
                       samples=4, elapsed_s=0.5 * i) for i in range(4)]
    res = TrainResult(history=[EpochMetrics(0, 1.0, 0.5, 0.1)], steps=steps,
                      weights=np.zeros(3, np.float32), virtual_time=None, wall_time=1.0)
    assert metrics_csv(res) == (
        "epoch,step,loss,acc,lr,elapsed_s\n"
        "0,0,1,0,0.1,0\n0,1,0.5,0.25,0.2,0.5\n0,2,0.333333,0.5,0.3,1\n1,3,0.25,0.75,0.4,1.5\n")
    assert res.final_acc == 0.5
