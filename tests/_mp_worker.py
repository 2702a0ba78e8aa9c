"""torchrun worker for tests/test_gpu_multiproc.py: the multi-PROCESS path
(one process per GPU, CUDA IPC handles over the gloo channel, plain kernel
launch per rank) checked against the oracle. Prints one JSON line on rank 0.

    torchrun --nproc-per-node N tests/_mp_worker.py
"""

import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1711_00705_b200 import (  # noqa: E402
    GradientBuffer,
    SgdUpdate,
    VarPayload,
    allreduce,
    alltoallv,
    build_multicolor_trees,
    dimd,
)
from paper_1711_00705_b200.transport import init_from_env  # noqa: E402


def main() -> None:
    ep = init_from_env()
    N, rank, dev = ep.n_ranks, ep.rank, ep.torch_device
    out: dict = {}
    rng = np.random.default_rng(2017)
    L, P = 100_003, 100_001
    inputs = [rng.standard_normal(L).astype(np.float32) for _ in range(N)]
    w0 = rng.standard_normal(P).astype(np.float32)
    m0 = rng.standard_normal(P).astype(np.float32)
    ks = [k for k in (1, 2, 4) if k <= N]
    with torch.cuda.stream(ep.stream):
        # 1. multicolor allreduce, bitwise vs the oracle fold, and the fused
        #    momentum/weight-decay update vs the float32 restatement
        for k in ks:
            ts = build_multicolor_trees(N, k, 4)
            want = O.fold_numpy(O.tables_from_trees(N, O.trees(N, k, 4)), inputs)
            buf = GradientBuffer(torch.from_numpy(inputs[rank].copy()).to(dev))
            w = torch.from_numpy(w0.copy()).to(dev)
            m = torch.from_numpy(m0.copy()).to(dev)
            upd = SgdUpdate(weights=w, c=0.0125, momentum=m, mu=0.9, wd_b=0.0032, update_len=P)
            allreduce(ep, buf, "multicolor", tree_set=ts, segment_elems=1000, update=upd)
            ep.synchronize()
            w_want, m_want = O.sgd_np(w0, want[:P], m0.copy(), 0.0125, 0.9, 0.0032)
            out[f"allreduce_k{k}"] = bool(np.array_equal(buf.data.cpu().numpy(), want))
            out[f"update_k{k}"] = bool(np.array_equal(w.cpu().numpy(), w_want)
                                       and np.array_equal(m.cpu().numpy(), m_want))
        # 2. back-to-back calls on one registered buffer (device epochs)
        g = GradientBuffer.alloc(4099, ep)
        for _ in range(3):
            g.data.fill_(float(rank + 1))
            allreduce(ep, g, "multicolor", tree_set=build_multicolor_trees(N, ks[-1], 4))
        ep.synchronize()
        out["repeat"] = bool(torch.all(g.data == N * (N + 1) / 2).item())
        # 3. DIMD shuffle: every slot's source index vs the oracle's plan, bytes
        #    vs the generator (shard arrays mapped through IPC)
        n = 3000
        store = dimd.synth_store(n, 256, rank, N, 11, 0, N, rank, device=dev)
        held = ep.all_gather(np.arange(n, dtype=np.int64) * N + rank)  # gid per (member, index)
        for epoch in range(2):
            key = O.mix64(11, O.SHUF_ROLE, epoch)
            counts = ep.all_gather(store.n_records)
            dimd.EXCHANGE = "push" if epoch == 0 else "pull"  # both data movements
            new = dimd.shuffle_all(ep, store, m_segments=3, seed=key)
            dimd.EXCHANGE = "push"
            bad, gids = dimd.synth_verify(new, 11)
            mem, rec = O.shuffle_plan_c(key, 0, N, rank, rank, 3, counts)
            out[f"shuffle{epoch}_bytes"] = int(bad) == 0
            out[f"shuffle{epoch}_count"] = new.n_records == len(mem)
            store = new
            # epoch 1 plans from the counts epoch 0 predicted (dimd._shuffle)
            got = gids.cpu().numpy().astype(np.int64)
            want = np.array([held[q][r] for q, r in zip(mem, rec)], dtype=np.int64)
            out[f"shuffle{epoch}_indices"] = bool(np.array_equal(got, want))
            held = ep.all_gather(got)
        # 4. every allreduce kernel under CUDA-graph replay (device epochs,
        #    LL inbox parity, read-done / arrival flags): 3 captured calls, each
        #    on a refilled buffer, replayed twice; bitwise vs the oracle fold
        ts = build_multicolor_trees(N, ks[-1], 4)
        tabs = O.tables_from_trees(N, O.trees(N, ks[-1], 4))
        for name, L2 in (("ll", 4099), ("oneshot", 400_003), ("tree", 6_000_001)):
            src = [np.random.default_rng(r + L2).standard_normal(L2).astype(np.float32)
                   for r in range(N)]
            want2 = O.fold_numpy(tabs, src)
            srcd = torch.from_numpy(src[rank]).to(dev)
            gb = GradientBuffer.alloc(L2, ep)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=ep.stream, capture_error_mode="thread_local"):
                for _ in range(3):
                    gb.data.copy_(srcd)
                    allreduce(ep, gb, "multicolor", tree_set=ts, check=False)
            ok = True
            for _ in range(2):
                ep.barrier()
                gr.replay()
                ep.synchronize()
                ep.take_error()
                ok = ok and bool(np.array_equal(gb.data.cpu().numpy(), want2))
            out[f"graph_{name}"] = ok
        # 5. the C5 call at full size (25.6M + 2 floats, momentum + weight
        #    decay), two calls back to back, on the default route of each update
        #    mode (replicated: stream kernel at N = 2, tree above; sharded:
        #    owner-push) -- md_last_route says which kernel ran
        from paper_1711_00705_b200 import _lib

        P5, L5 = 25_600_000, 25_600_002
        src5 = [np.random.default_rng(77 + r).standard_normal(L5, dtype=np.float32)
                for r in range(N)]
        w5 = np.random.default_rng(78).standard_normal(P5, dtype=np.float32)
        ts5 = build_multicolor_trees(N, ks[-1], 4)
        g5 = O.fold_c(O.tables_from_trees(N, O.trees(N, ks[-1], 4)), src5)
        c5, wd5 = float(np.float32(0.1 / (32 * N))), float(np.float32(1e-4 * 32 * N))
        ww, mm = w5, np.zeros(P5, np.float32)
        for _ in range(2):
            ww, mm = O.sgd_np(ww, g5[:P5], mm.copy(), c5, 0.9, wd5)
        want_route = {False: "stream" if N == 2 else "tree", True: "push"}
        for sharded in (False, True):
            w, _ = ep.alloc(P5)
            w.copy_(torch.from_numpy(w5))
            m = torch.zeros(P5, device=dev)
            gb = GradientBuffer.alloc(L5, ep)
            for _ in range(2):
                gb.data.copy_(torch.from_numpy(src5[rank]))
                allreduce(ep, gb, "multicolor", tree_set=ts5,
                          update=SgdUpdate(weights=w, c=c5, momentum=m, mu=0.9, wd_b=wd5,
                                           update_len=P5, sharded=sharded))
            ep.synchronize()
            route = _lib.last_route(ep.device)
            tag = "sharded" if sharded else "replicated"
            out[f"c5_{tag}_route"] = route[0] == want_route[sharded] and route[2] == sharded
            out[f"c5_{tag}_w"] = bool(np.array_equal(w.cpu().numpy(), ww))
            if not sharded:
                out[f"c5_{tag}_g"] = bool(np.array_equal(gb.data.cpu().numpy(), g5))
                out[f"c5_{tag}_m"] = bool(np.array_equal(m.cpu().numpy(), mm))
            del w, m, gb
        del src5, g5
        # 6. alltoallv (host payloads, device exchange)
        mats = [[bytes([s, d]) * (s + d + 1) for d in range(N)] for s in range(N)]
        got = alltoallv(ep, VarPayload.from_slices(mats[rank])).data
        out["alltoallv"] = bytes(got) == b"".join(mats[s][rank] for s in range(N))
    # 7. run_training (the reference's loop and model) with one process per
    # rank, against the reference's own run (tests/golden/toy.npz)
    with np.load(ROOT / "tests" / "golden" / "toy.npz") as z:
        toy = {k: z[k] for k in z.files}
    from paper_1711_00705_b200 import TrainConfig, make_synthetic_corpus, run_training

    for t in range(int(toy["n_train"][0])):
        nn, m, kb, epochs, seed, nrec, hidden, every, gs = (int(v) for v in toy[f"train{t}_cfg"])
        if nn != N:
            continue
        cfg = TrainConfig(n_nodes=nn, workers_per_node=m, per_worker_batch=kb, epochs=epochs,
                          seed=seed, hidden=hidden, shuffle_every=every, group_size=gs)
        res = run_training(cfg, make_synthetic_corpus(nrec, seed=seed),
                           str(toy[f"train{t}_algo"]), backend="torchrun")
        steps = np.array([[s.step, s.loss, s.correct, s.lr] for s in res.steps])
        out[f"run_training_{t}"] = bool(np.array_equal(res.weights, toy[f"train{t}_weights"])
                                        and np.array_equal(steps, toy[f"train{t}_steps"]))
    rows = ep.all_gather(out)
    if rank == 0:
        print(json.dumps({"n": N, "ok": all(all(r.values()) for r in rows), "rows": rows}))


if __name__ == "__main__":
    main()
