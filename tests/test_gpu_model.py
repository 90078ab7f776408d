"""GPU: the cost-model drop-ins (paper_2012_07145_b200.costmodel — K1 + K7)
against vectors written by the unmodified reference
(tests/golden/make_model_golden.py):

* featurize(state) returns the reference's rows, keys and AlgorithmFeatures;
* predict_coefficients within 1e-9 relative (fp64, BLAS order differs);
* stage_cost with the reference's coefficients: every CostBreakdown term
  bit-exact (same operations, same rounding steps);
* pipeline_cost totals within 1e-9 relative;
* train (SGD + momentum, every epoch in one launch): loss history and final
  weights within 1e-6 relative — on the machine-oracle dataset the reference
  driver builds (saturated, loss flat) and on a well-conditioned one whose
  loss falls 0.72 -> 0.18."""

import gzip
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import PARAMS, candidate_set  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
REL = 1e-9


@pytest.fixture(scope="module")
def gold():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with gzip.open(os.path.join(GOLD, "model.json.gz"), "rt") as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(GOLD, "model.npz"))


@pytest.mark.parametrize("name", ["stencil_chain", "chain20"])
def test_featurize_predict_stage_cost_pipeline_cost(gold, name):
    from paper_2012_07145_b200 import costmodel
    from paper_2012_07145_b200.params import init_weights
    meta, arr = gold
    cs = candidate_set(name)
    w = init_weights(0)
    keys = meta["sets"][name]["keys"]
    feats, algo = [], []
    totals = []
    for i, state in enumerate(cs.decisions):
        fd = costmodel.featurize(state, cs.graph, PARAMS, thresholds=cs.thresholds)
        assert [list(k) for k in fd] == keys[i], i
        for f in fd.values():
            feats.append(f.to_vector())
            algo.append(f.algorithm.to_vector())
        totals.append(costmodel.pipeline_cost(fd, w)[0])
    feats, algo = np.array(feats), np.array(algo)
    assert np.array_equal(feats, arr[f"{name}_feats"])
    assert np.array_equal(algo, arr[f"{name}_algo"])
    np.testing.assert_allclose(totals, arr[f"{name}_totals"], rtol=REL, atol=0)
    c, _ = costmodel._predict(algo, feats, w, breakdown=False)
    np.testing.assert_allclose(c, arr[f"{name}_coeffs"], rtol=REL, atol=0)
    # stage_cost with the reference's own coefficients: bit-exact terms
    _, bd = costmodel._predict(None, feats, coeffs=arr[f"{name}_coeffs"])
    assert np.array_equal(bd, arr[f"{name}_breakdown"])
    # the single-row drop-ins agree with the batch
    fd = costmodel.featurize(cs.decisions[0], cs.graph, PARAMS, thresholds=cs.thresholds)
    f0 = next(iter(fd.values()))
    c0 = costmodel.predict_coefficients(f0.algorithm, f0, w)
    np.testing.assert_allclose(c0, arr[f"{name}_coeffs"][0], rtol=REL, atol=0)
    b0 = costmodel.stage_cost(f0, arr[f"{name}_coeffs"][0])
    assert [b0.compute, b0.load, b0.store, b0.malloc, b0.parallelism, b0.working_set, b0.total] == \
        arr[f"{name}_breakdown"][0].tolist()


def test_drop_in_errors(gold):
    from paper_2012_07145_b200 import costmodel
    from paper_2012_07145_b200.params import init_weights
    cs = candidate_set("stencil_chain")
    fd = costmodel.featurize(cs.decisions[0], cs.graph, PARAMS, thresholds=cs.thresholds)
    f0 = next(iter(fd.values()))
    with pytest.raises(ValueError):
        costmodel.stage_cost(f0, np.ones(29))
    with pytest.raises(ValueError):
        costmodel.stage_cost(f0, np.zeros(30))
    with pytest.raises(ValueError):
        costmodel.predict_coefficients(np.zeros(9), f0, init_weights(0))


@pytest.mark.parametrize("tag", ["train", "train2"])
def test_train_matches_reference(gold, tag):
    from paper_2012_07145_b200 import costmodel
    from paper_2012_07145_b200.params import init_weights
    meta, arr = gold
    t = meta[tag]
    cs = candidate_set("stencil_chain" if tag == "train" else "chain20")

    class Sample:
        def __init__(self, stages, runtime, sid):
            self.stages, self.runtime, self.pipeline_id, self.schedule_id = stages, runtime, cs.name, sid

    data = []
    for sid, rt in zip(t["sample_ids"], t["runtimes"]):
        c = cs.cand(int(sid))
        stages = [(c["algo"][r], c["feats"][r], c["g"][r], float(c["h"][r])) for r in range(len(c["rows"]))]
        data.append(Sample(stages, rt, sid))
    cfg = costmodel.TrainConfig(learning_rate=t["learning_rate"], momentum=t["momentum"], epochs=t["epochs"],
                                seed=t["seed"])
    res = costmodel.train(data, cfg, init=init_weights(0))
    np.testing.assert_allclose(res.loss_history, arr[f"{tag}_loss"], rtol=1e-6, atol=0)
    flat = costmodel.pack_weights(res.weights)
    np.testing.assert_allclose(flat, arr[f"{tag}_weights"], rtol=1e-6, atol=1e-12)
    assert res.final_loss == res.loss_history[-1]
    with pytest.raises(ValueError):
        costmodel.train(data[:1], cfg)
