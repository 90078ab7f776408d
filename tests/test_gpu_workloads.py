"""The BASELINE.json workloads beyond the C5 bench:

* C2 — unsharp / Harris beam steps (parents x all step-root tilings), 64K
  candidates on one GPU: features with sibling reuse equal the full
  recompute bit for bit, a strided subsample equals the CPU oracle exactly
  (costs to 1e-9), hashes and hierarchical-sampling representatives equal
  the oracle's bit for bit.
* C4 — ResNet-50 bottleneck block, 262,144 random schedules: prune verdicts
  and depth-3 hashes against the oracle on a subsample, buckets +
  representatives against the oracle over the whole batch.  The full-size
  block's 256-channel windows are beyond the brute-force oracle's memory
  (as they are beyond the reference's), so its features are checked by
  reuse-on == reuse-off; `resnet_small` (same structure) is checked against
  the oracle feature by feature.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import PARAMS, decisions_from_records, weights  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _graph(name):
    from paper_2012_07145_b200.pipeline import builtin_pipeline
    return builtin_pipeline(name)


def _oracle_rows(graph, dec):
    from oracle import costing
    total, _, rows = costing.score(graph, dec, PARAMS, weights().tensors)
    return total, np.array([f for _, f, _ in rows])


def _check_sample(sc, graph, info, recs, f, total, idx):
    feats = f["feats"].cpu().numpy()
    nrows = f["n_rows"].cpu().numpy()
    tot = total.cpu().numpy()
    for i in idx:
        want_total, want = _oracle_rows(graph, decisions_from_records(info, recs[i]))
        assert nrows[i] == len(want)
        bad = np.argwhere(feats[i, :len(want)] != want)
        assert bad.size == 0, (graph.name, i, bad[:4])
        assert tot[i] == pytest.approx(want_total, rel=1e-9)


def _check_select(sc, graph, info, recs, hashes, verdict, phase_seed, sample):
    from oracle import structure
    h = hashes.cpu().numpy().view(np.uint64)
    for i in sample:
        assert int(h[i]) == structure.structural_hash(decisions_from_records(info, recs[i]), 3)
    v = verdict.cpu().numpy()
    rep, rej, cnt = sc.select(hashes, verdict, phase_seed)
    nrep, nrej = (int(x) for x in cnt.tolist())
    want_reps, want_rej = structure.select_reps([int(x) for x in h], v == 0, phase_seed)
    assert rep[:nrep].cpu().tolist() == want_reps
    assert rej[:nrej].cpu().tolist() == want_rej


@pytest.mark.parametrize("name", ["unsharp", "harris"])
def test_c2_beam_step_64k(name, dev):
    from paper_2012_07145_b200 import gen
    from paper_2012_07145_b200.engine import Scorer
    graph = _graph(name)
    info = gen.GraphInfo(graph)
    # enough parents for >= 64K children
    recs, owner, _ = gen.beam_step(graph, 64, seed=3)
    per = len(recs) / 64
    recs, owner, _ = gen.beam_step(graph, int(np.ceil(65536 / per)), seed=3)
    recs = recs[:65536]
    assert len(recs) == 65536
    sc = Scorer(graph, PARAMS, None, weights())
    dec = sc.to_device(recs)
    f = sc.featurize(dec)
    total, _, _ = sc.cost(f)
    st = sc.stats()
    sc.set_reuse(False)
    f2 = sc.featurize(dec)
    total2, _, _ = sc.cost(f2)
    sc.set_reuse(True)
    sc.check()
    assert st["incremental"] > 0.9 * len(recs)
    nr = f["n_rows"]
    assert torch.equal(nr, f2["n_rows"]) and torch.equal(f["verdict"], f2["verdict"])
    mask = torch.arange(sc.R, device=dev)[None, :] < nr[:, None]
    assert torch.equal(f["feats"][mask], f2["feats"][mask])
    assert torch.equal(total, total2)
    sample = list(range(0, len(recs), len(recs) // 24))
    _check_sample(sc, graph, info, recs, f, total, sample)
    h = sc.struct_hash(dec, 3)
    _check_select(sc, graph, info, recs, h, f["verdict"], 3 * 101 + 7, sample)


def test_c4_resnet_block_262k(dev):
    from oracle import costing
    from paper_2012_07145_b200 import gen
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS
    graph = _graph("resnet_block")
    recs, decs, info = gen.random_schedules(graph, 262144, seed=0)
    sc = Scorer(graph, PARAMS, None, weights())
    dec = sc.to_device(recs)
    f = sc.featurize(dec)
    total, _, _ = sc.cost(f)
    sc.check()
    assert torch.isfinite(total).all()
    v = f["verdict"].cpu().numpy()
    sample = list(range(0, len(recs), len(recs) // 64))
    for i in sample:
        want = costing.prune_reason(graph, decs[i], PARAMS, DEFAULT_THRESHOLDS)
        code = 0 if want is None else 1 + ("excessive_recompute", "idle_sms", "poor_warp_utilization",
                                           "serial_too_large", "thread_alloc_dynamic_or_large",
                                           "hardware_limit").index(want)
        assert v[i] == code, (i, v[i], want)
    # random schedules have no siblings: reuse must not change anything
    sc.set_reuse(False)
    g = sc.featurize(dec[:4096])
    sc.set_reuse(True)
    nr = g["n_rows"]
    mask = torch.arange(sc.R, device=dev)[None, :] < nr[:, None]
    assert torch.equal(f["feats"][:4096][mask], g["feats"][mask])
    h = sc.struct_hash(dec, 3)
    _check_select(sc, graph, info, recs, h, f["verdict"], 1 * 101 + 2, sample[:16])


def test_c4_resnet_small_vs_oracle(dev):
    from paper_2012_07145_b200 import gen
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.params import OPEN_THRESHOLDS
    graph = _graph("resnet_small")
    recs, decs, info = gen.random_schedules(graph, 4096, seed=1)
    sc = Scorer(graph, PARAMS, OPEN_THRESHOLDS, weights())
    dec = sc.to_device(recs)
    f = sc.featurize(dec)
    total, _, _ = sc.cost(f)
    sc.check()
    _check_sample(sc, graph, info, recs, f, total, list(range(0, 4096, 128)))
