"""Golden vectors for the gradient producer: the reference's own ToyModel
(/root/reference/pkg/src/minidist/sgd.py:147-247) and run_training
(sgd.py:470-542), run in the build container:

    python tests/golden/make_golden_toy.py      (-> tests/golden/toy.npz)

Records
  * ``case{i}_*``: ToyModel.loss_and_grad_sum on seeded inputs of several
    shapes (batch 1..300, n_in/hidden/classes incl. 1) -- weights, x (float32
    record values), labels, the float32 gradient, the loss sum, the count;
  * ``grad_*``: grad(model, batch) (sgd.py:250-257) on float64 features;
  * ``train_*``: run_training (sim backend) of make_synthetic_corpus records
    for four configurations (multicolor / ring / reduce_bcast, shuffle groups),
    with reshuffles -- final weights and every step's (loss, correct, lr).
Everything recorded is an output of reference code (make_golden.py's import
recipe: scratch copy, thread-backed greenlet stand-in).
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from make_golden import import_reference

HERE = Path(__file__).resolve().parent

SHAPES = [  # (batch, n_in, hidden, classes, seed)
    (4, 16, 8, 4, 1), (1, 16, 8, 4, 2), (2, 16, 8, 4, 3), (7, 16, 8, 4, 4), (8, 16, 8, 4, 5),
    (9, 16, 8, 4, 6), (32, 16, 8, 4, 7), (128, 16, 8, 4, 8), (129, 16, 8, 4, 9),
    (300, 16, 8, 4, 10), (5, 3, 5, 2, 11), (6, 1, 1, 1, 12), (16, 24, 12, 10, 13),
    (3, 40, 32, 7, 14), (64, 8, 2, 3, 15),
    (8, 16, 2048, 4, 16),  # the reference's bench_train model (bench.py:71-75)
]

TRAIN = [  # (n_nodes, workers, per_worker_batch, epochs, seed, n_records, hidden, shuffle_every,
    #    group_size, algo)
    (2, 2, 4, 3, 5, 96, 8, 1, 1, "multicolor"),
    (4, 1, 8, 2, 11, 160, 6, 2, 1, "multicolor"),
    (3, 2, 3, 2, 17, 120, 5, 1, 3, "ring"),
    (4, 1, 4, 2, 23, 100, 8, 1, 2, "reduce_bcast"),
    (4, 2, 8, 2, 29, 512, 2048, 1, 1, "multicolor"),  # bench_train's model width
]


def main() -> None:
    import_reference()
    from minidist.sgd import ToyModel, TrainConfig, make_synthetic_corpus, run_training

    G: dict[str, np.ndarray] = {}
    for i, (k, n_in, hidden, ncls, seed) in enumerate(SHAPES):
        rng = np.random.default_rng(1000 + seed)
        model = ToyModel.create(n_in=n_in, hidden=hidden, n_classes=ncls, seed=seed)
        x32 = (rng.standard_normal((k, n_in)) * 1.5).astype("<f4")
        y = rng.integers(0, ncls, size=k)
        g, loss, correct = model.loss_and_grad_sum(x32.astype(np.float64), y)
        G[f"case{i}_shape"] = np.array([k, n_in, hidden, ncls], np.int64)
        G[f"case{i}_w"] = model.weights.copy()
        G[f"case{i}_x"] = x32
        G[f"case{i}_y"] = y.astype(np.int64)
        G[f"case{i}_g"] = g
        G[f"case{i}_loss"] = np.array([loss], np.float64)
        G[f"case{i}_correct"] = np.array([correct], np.int64)
    G["n_cases"] = np.array([len(SHAPES)], np.int64)

    # grad(model, batch) (sgd.py:250-257) on float64 features (not float32-exact)
    from minidist.sgd import grad

    rng = np.random.default_rng(77)
    model = ToyModel.create(seed=21)
    feats = rng.standard_normal((6, 16)) * 2.0
    labels = rng.integers(0, 4, size=6)
    G["grad_w"] = model.weights.copy()
    G["grad_x"] = feats
    G["grad_y"] = labels.astype(np.int64)
    G["grad_out"] = np.asarray(grad(model, list(zip(feats, labels.tolist()))).data, np.float32)

    for j, (nn, m, kb, epochs, seed, nrec, hidden, every, gs, algo) in enumerate(TRAIN):
        cfg = TrainConfig(n_nodes=nn, workers_per_node=m, per_worker_batch=kb, epochs=epochs,
                          seed=seed, hidden=hidden, shuffle_every=every, group_size=gs)
        corpus = make_synthetic_corpus(nrec, seed=seed)
        res = run_training(cfg, corpus, algo, backend="sim")
        G[f"train{j}_cfg"] = np.array([nn, m, kb, epochs, seed, nrec, hidden, every, gs], np.int64)
        G[f"train{j}_algo"] = np.array(algo)
        G[f"train{j}_corpus_x"] = np.stack([np.frombuffer(r.bytes, "<f4") for r in corpus])
        G[f"train{j}_corpus_y"] = np.array([r.label for r in corpus], np.int64)
        G[f"train{j}_weights"] = np.asarray(res.weights, np.float32)
        G[f"train{j}_steps"] = np.array([[s.step, s.loss, s.correct, s.lr] for s in res.steps],
                                        np.float64)
        G[f"train{j}_history"] = np.array([[h.epoch, h.loss, h.acc] for h in res.history],
                                          np.float64)
    G["n_train"] = np.array([len(TRAIN)], np.int64)
    np.savez_compressed(HERE / "toy.npz", **G)
    print(f"wrote {len(G)} arrays to {HERE / 'toy.npz'}")


if __name__ == "__main__":
    main()
