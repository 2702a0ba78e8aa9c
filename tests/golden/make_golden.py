"""Generate golden vectors by running the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory, builds the reference's
Cython kernels there (never into this repo), puts a thread-backed greenlet
stand-in (tests/golden/_shim) on sys.path, imports ``minidist`` and records
its outputs on small seeded inputs into tests/golden/golden.npz and
tests/golden/trees.json. The GPU box has no /root/reference; the committed
fixtures travel instead. Everything recorded is an output of reference code:
allreduce_multicolor / allreduce_ring / reduce_then_broadcast through
run_ranks (sim backend), _kernels.sub_scaled_f32, random_batch, shuffle_all,
shuffle_group, train_step, lr_at, build_blob, _mix64.
"""

from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg")
SCRATCH = Path(os.environ.get("MD_REF_SCRATCH", "/tmp/md_refpkg"))


def import_reference():
    if not (SCRATCH / "src" / "minidist").exists():
        shutil.copytree(REF, SCRATCH, dirs_exist_ok=True)
    if not list((SCRATCH / "src" / "minidist" / "_kernels").glob("_accel*.so")):
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       check=True, capture_output=True)
    sys.path[:0] = [str(HERE / "_shim"), str(SCRATCH / "src")]
    import minidist  # noqa: F401

    return minidist


def unique_records(n, rng, max_len=40, label_range=1000, fixed=None):
    """Records whose first 4 bytes encode their corpus index (so outputs can
    be mapped back to indices), random tail, random label."""
    from minidist.dimd import Record

    out = []
    for i in range(n):
        ln = fixed if fixed is not None else int(rng.integers(4, max_len))
        body = i.to_bytes(4, "little") + bytes(rng.integers(0, 256, size=ln - 4, dtype=np.uint8))
        out.append(Record(body, int(rng.integers(0, label_range))))
    return out


def rec_ids(records):
    return np.array([int.from_bytes(r.bytes[:4], "little") for r in records], np.int64)


def main() -> None:
    md = import_reference()
    from minidist import _kernels
    from minidist.collectives import (
        GradientBuffer,
        allreduce_multicolor,
        allreduce_ring,
        reduce_then_broadcast,
    )
    from minidist.dimd import (
        BatchRequest,
        _mix64,
        build_blob,
        parse_index,
        random_batch,
        shard_from_bytes,
        shuffle_all,
        shuffle_group,
    )
    from minidist.sgd import (
        ToyModel,
        TrainConfig,
        lr_at,
        lr_schedule,
        make_synthetic_corpus,
        sample_node_batch,
        train_step,
    )
    from minidist.topology import build_multicolor_trees, build_ring, tree_set_to_dict
    from minidist.transport import run_ranks

    assert _kernels.BACKEND == "compiled", _kernels.BACKEND
    G: dict[str, np.ndarray] = {}

    # -- tree sets ------------------------------------------------------------------
    trees = {}
    for n in range(2, 17):
        for k in (1, 2, 4, 8):
            for arity in (1, 2, 3, 4, 7):
                try:
                    ts = build_multicolor_trees(n, k, arity)
                except Exception as e:  # noqa: BLE001 - record the failure class
                    trees[f"{n},{k},{arity}"] = {"error": type(e).__name__}
                    continue
                trees[f"{n},{k},{arity}"] = tree_set_to_dict(ts.with_plan(1000))
    (HERE / "trees.json").write_text(json.dumps(trees, sort_keys=True))

    # -- multicolor folds ------------------------------------------------------------
    mc_cases = [(8, 1000, 4, 4), (8, 997, 4, 4), (4, 7, 4, 4), (3, 1, 3, 4), (2, 0, 2, 4),
                (16, 250, 4, 4), (2, 4099, 1, 4), (2, 4099, 2, 4), (4, 4099, 1, 4),
                (4, 4099, 2, 4), (4, 4099, 4, 4), (8, 4099, 1, 4), (8, 4099, 2, 4),
                (8, 4099, 8, 7), (8, 10007, 4, 4), (4, 10007, 4, 4)]
    for n, L, k, arity in mc_cases:
        rng = np.random.default_rng(7000 + n * 17 + L + k)
        arrays = [rng.standard_normal(L).astype(np.float32) for _ in range(n)]
        ts = build_multicolor_trees(n, k, arity)
        res = run_ranks(
            n, "sim",
            lambda ep: allreduce_multicolor(ep, GradientBuffer(arrays[ep.rank].copy()), ts,
                                            segment_elems=64).data,
        ).results
        assert all(np.array_equal(r, res[0]) for r in res)
        tag = f"mc_{n}_{L}_{k}_{arity}"
        G[tag + "_in"] = np.stack(arrays) if L else np.zeros((n, 0), np.float32)
        G[tag + "_out"] = res[0]

    # -- ring and reduce-then-broadcast ----------------------------------------------
    for n, L in [(8, 1000), (5, 333), (2, 4), (4, 4099)]:
        rng = np.random.default_rng(3000 + n + L)
        arrays = [rng.standard_normal(L).astype(np.float32) for _ in range(n)]
        ring = build_ring(n)
        res = run_ranks(
            n, "sim",
            lambda ep: allreduce_ring(ep, GradientBuffer(arrays[ep.rank].copy()), ring,
                                      segment_elems=100).data,
        ).results
        G[f"ring_{n}_{L}_in"] = np.stack(arrays)
        G[f"ring_{n}_{L}_out"] = res[0]
    for n, L, root in [(8, 513, 0), (4, 100, 2), (4, 4099, 3)]:
        rng = np.random.default_rng(12 + n + L + root)
        arrays = [rng.standard_normal(L).astype(np.float32) for _ in range(n)]
        res = run_ranks(
            n, "sim",
            lambda ep: reduce_then_broadcast(ep, GradientBuffer(arrays[ep.rank].copy()),
                                             root=root).data,
        ).results
        G[f"rb_{n}_{L}_{root}_in"] = np.stack(arrays)
        G[f"rb_{n}_{L}_{root}_out"] = res[0]

    # -- float kernels ---------------------------------------------------------------
    rng = np.random.default_rng(1)
    a = rng.standard_normal(20003).astype(np.float32)
    b = rng.standard_normal(20003).astype(np.float32)
    G["kern_a"], G["kern_b"] = a, b
    d = a.copy()
    _kernels.add_f32(d, b)
    G["kern_add"] = d
    cs = np.array([0.0, 1.0, 1 / 3, 0.025, -7.5, 0.0123], np.float64)
    G["kern_c"] = cs
    G["kern_sub"] = np.stack([_sub(_kernels, a, b, c) for c in cs])

    # -- mix64 + lr schedule -----------------------------------------------------------
    parts = [(0,), (1, 2, 3), (7, int.from_bytes(b"dest", "little"), 0, 3, 11),
             ((1 << 64) - 1, 5), (123456789, int.from_bytes(b"samp", "little"), 17, 42)]
    G["mix64_parts"] = np.array([list(p) + [0] * (5 - len(p)) for p in parts], np.uint64)
    G["mix64_n"] = np.array([len(p) for p in parts], np.int64)
    G["mix64_out"] = np.array([_mix64(*p) for p in parts], np.uint64)
    lr_rows = []
    for base, k, nn in [(0.1, 64, 4), (0.1, 32, 256), (0.05, 8, 32)]:
        cfg_s = TrainConfig(n_nodes=1, workers_per_node=nn, per_worker_batch=k, epochs=1,
                            base_lr=base)
        for ep_ in (0.0, 1.25, 2.5, 4.999, 5.0, 34.999, 35.0, 65.0, 94.9):
            lr_rows.append([base, k, nn, ep_, lr_at(lr_schedule(cfg_s), ep_)])
    G["lr_rows"] = np.array(lr_rows, np.float64)

    # -- DIMD: codec, random_batch, shuffle -------------------------------------------
    rng = np.random.default_rng(5)
    recs = unique_records(50, rng)
    blob, index = build_blob(recs)
    G["codec_blob"] = np.frombuffer(blob, np.uint8)
    G["codec_index"] = np.frombuffer(index, np.uint8)

    rng = np.random.default_rng(6)
    recs = unique_records(37, rng)
    blob, index = build_blob(recs)
    store = shard_from_bytes(blob, parse_index(index), 0, 1, 1)
    G["rb_blob"] = np.frombuffer(blob, np.uint8)
    G["rb_index"] = np.frombuffer(index, np.uint8)
    picks = []
    for seed, bs in [(42, 64), (43, 64), (5, 1000), ((1 << 64) - 3, 17), (0, 1)]:
        got = random_batch(store, BatchRequest(bs, seed))
        picks.append((seed, bs, rec_ids(got)))
    G["rb_seeds"] = np.array([p[0] for p in picks], np.uint64)
    G["rb_sizes"] = np.array([p[1] for p in picks], np.int64)
    G["rb_picks"] = np.concatenate([p[2] for p in picks])

    shuffle_cases = [
        # (name, n_records, n_ranks, group_size, m_segments, seed, fixed_len, which)
        ("sh_a", 200, 4, 4, 3, 77, None, "all"),
        ("sh_b", 200, 4, 2, 2, 5, None, "group"),
        ("sh_c", 3, 2, 2, 16, 2, None, "all"),
        ("sh_d", 60, 4, 4, 2, 4, None, "all"),
        ("sh_e", 10, 1, 1, 2, 9, None, "all"),
        ("sh_f", 999, 8, 8, 5, 31337, 48, "all"),
        ("sh_g", 601, 6, 3, 4, 11, None, "group"),
    ]
    for name, nrec, nr, gs, m, seed, fixed, which in shuffle_cases:
        rng = np.random.default_rng(int.from_bytes(name.encode(), "little"))
        recs = unique_records(nrec, rng, fixed=fixed)
        blob, index = build_blob(recs)
        entries = parse_index(index)
        fn = shuffle_all if which == "all" else shuffle_group

        def body(ep, fn=fn, blob=blob, entries=entries, gs=gs, m=m, seed=seed):
            st = shard_from_bytes(blob, entries, ep.rank, ep.n_ranks, gs)
            out = fn(ep, st, m_segments=m, seed=seed)
            return rec_ids(out.records()), np.array([e.label for e in out.index], np.int64)

        res = run_ranks(nr, "sim", body).results
        G[name + "_blob"] = np.frombuffer(blob, np.uint8)
        G[name + "_index"] = np.frombuffer(index, np.uint8)
        G[name + "_meta"] = np.array([nrec, nr, gs, m, seed], np.int64)
        G[name + "_counts"] = np.array([len(r[0]) for r in res], np.int64)
        G[name + "_ids"] = np.concatenate([r[0] for r in res]) if nrec else np.zeros(0, np.int64)
        G[name + "_labels"] = np.concatenate([r[1] for r in res]) if nrec else np.zeros(0, np.int64)

    # -- SGD: 12 distributed steps; per-worker gradient buffers + weights ----------------
    cfg = TrainConfig(n_nodes=4, workers_per_node=2, per_worker_batch=4, epochs=1,
                      shuffle_every=0, seed=9)
    corpus = make_synthetic_corpus(512, seed=9)
    blob, idx = build_blob(corpus)
    entries = parse_index(idx)
    ts = build_multicolor_trees(4, k=4)
    n_steps = 12
    p = ToyModel.create(seed=cfg.seed).n_params
    G["sgd_w0"] = ToyModel.create(seed=cfg.seed).weights.copy()

    def body(ep):
        store = shard_from_bytes(blob, entries, ep.rank, ep.n_ranks, cfg.group_size)
        model = ToyModel.create(seed=cfg.seed)
        wbufs, weights, lrs = [], [], []
        for step in range(n_steps):
            epoch = step / 16.0
            per_worker = []
            for x, y in sample_node_batch(store, cfg, ep.rank, step):
                g, loss, correct = model.loss_and_grad_sum(x, y)
                buf = np.empty(p + 2, dtype=np.float32)
                buf[:p], buf[p], buf[p + 1] = g, loss, correct
                per_worker.append(buf)
            wbufs.append(np.stack(per_worker))
            lrs.append(lr_at(lr_schedule(cfg), epoch))
            model, _ = train_step(ep, model, cfg, store, "multicolor", step=step, epoch=epoch,
                                  tree_set=ts)
            weights.append(model.weights.copy())
        return np.stack(wbufs), np.stack(weights), np.array(lrs)

    res = run_ranks(4, "sim", body).results
    G["sgd_workers"] = np.stack([r[0] for r in res])  # [rank, step, worker, p+2]
    G["sgd_weights"] = res[0][1]                       # [step, p]
    G["sgd_lr"] = res[0][2]
    G["sgd_cfg"] = np.array([4, 2, 4, 9, p], np.int64)

    np.savez_compressed(HERE / "golden.npz", **G)
    print(f"wrote {len(G)} arrays to {HERE / 'golden.npz'} and {len(trees)} tree sets")


def _sub(k, a, b, c):
    d = a.copy()
    k.sub_scaled_f32(d, b, c)
    return d


if __name__ == "__main__":
    main()
