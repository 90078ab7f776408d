"""Golden vectors for the cost-model drop-ins (costmodel.py on the GPU),
written by the UNMODIFIED reference (run in the build container):

    python tests/golden/make_model_golden.py

For the stencil_chain and chain20 golden candidate sets (tests/golden/*.json.gz):
  * reference `featurize` of every candidate (rows, keys, AlgorithmFeatures);
  * `predict_coefficients` of every row, `stage_cost` of every row with those
    coefficients (the six terms + total), `pipeline_cost` per candidate;
  * a `train` run (TrainConfig(epochs=30, seed=0), init_weights(0)) on
    `make_training_sample(featurize(s), simulate_runtime(s).runtime)` of the
    stencil_chain candidates the machine oracle accepts: loss history and
    final weights.
Output: model.json.gz (metadata) + model.npz (arrays)."""

from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src"), os.path.join(REF, "tests")]
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from gpusched.costmodel import (TrainConfig, init_weights, make_training_sample, pipeline_cost,  # noqa: E402
                                predict_coefficients, stage_cost, train)
from gpusched.featurize import featurize  # noqa: E402
from gpusched.loopnest import replay_schedule  # noqa: E402
from gpusched.machine import MachineParams, simulate_runtime  # noqa: E402
from gpusched.pipeline import parse_pipeline  # noqa: E402

NAMES = ("stencil_chain", "chain20")
TENSORS = ("algo_w", "algo_b", "sched_w", "sched_b", "head_w", "head_b", "out_w", "out_b")


def main():
    params = MachineParams()
    w = init_weights(0)
    meta, arr = {"sets": {}}, {}
    dataset, dataset2 = [], []
    rng = np.random.default_rng(7)
    for name in NAMES:
        with gzip.open(os.path.join(HERE, f"{name}.json.gz"), "rt") as fh:
            m = json.load(fh)
        graph = parse_pipeline(m["pipeline"], name)
        keys, coeffs, bds, totals, feats, algo = [], [], [], [], [], []
        for i, text in enumerate(m["candidates"]):
            state = replay_schedule(graph, text)
            fd = featurize(state, graph, params)
            keys.append([[k[0], k[1]] for k in fd])
            for k, f in fd.items():
                c = predict_coefficients(f.algorithm, f, w)
                b = stage_cost(f, c)
                coeffs.append(c)
                bds.append([b.compute, b.load, b.store, b.malloc, b.parallelism, b.working_set, b.total])
                feats.append(f.to_vector())
                algo.append(f.algorithm.to_vector())
            totals.append(pipeline_cost(fd, w)[0])
            if name == "chain20":   # runtimes near the model's own predictions: O(1) log errors
                dataset2.append(make_training_sample(fd, totals[-1] * float(rng.uniform(0.25, 4.0)), name, str(i)))
            if name == "stencil_chain":
                try:
                    rt = simulate_runtime(state, graph, params).runtime
                except ValueError:
                    rt = None
                if rt is not None:
                    dataset.append(make_training_sample(fd, rt, name, str(i)))
        meta["sets"][name] = {"keys": keys}
        arr[f"{name}_coeffs"] = np.array(coeffs)
        arr[f"{name}_breakdown"] = np.array(bds)
        arr[f"{name}_totals"] = np.array(totals)
        arr[f"{name}_feats"] = np.array(feats)
        arr[f"{name}_algo"] = np.array(algo)
    cfg = TrainConfig(epochs=30, seed=0)
    res = train(dataset, cfg, init=init_weights(0))
    meta["train"] = {"epochs": cfg.epochs, "learning_rate": cfg.learning_rate, "momentum": cfg.momentum,
                     "seed": cfg.seed, "n_samples": len(dataset),
                     "sample_ids": [s.schedule_id for s in dataset], "runtimes": [s.runtime for s in dataset]}
    arr["train_loss"] = np.array(res.loss_history)
    arr["train_weights"] = np.concatenate([res.weights.tensors[n].ravel() for n in TENSORS])
    cfg2 = TrainConfig(learning_rate=1e-3, momentum=0.9, epochs=40, seed=3)
    res2 = train(dataset2, cfg2, init=init_weights(0))
    meta["train2"] = {"epochs": cfg2.epochs, "learning_rate": cfg2.learning_rate, "momentum": cfg2.momentum,
                      "seed": cfg2.seed, "n_samples": len(dataset2),
                      "sample_ids": [s.schedule_id for s in dataset2], "runtimes": [s.runtime for s in dataset2]}
    arr["train2_loss"] = np.array(res2.loss_history)
    arr["train2_weights"] = np.concatenate([res2.weights.tensors[n].ravel() for n in TENSORS])
    print("train2 loss", res2.loss_history[0], "->", res2.final_loss)
    with gzip.open(os.path.join(HERE, "model.json.gz"), "wt") as fh:
        json.dump(meta, fh)
    np.savez_compressed(os.path.join(HERE, "model.npz"), **arr)
    print("samples", len(dataset), "final loss", res.final_loss)


if __name__ == "__main__":
    main()
