"""GPU parity: the sm_100a path (through the C ABI) against vectors produced
by the unmodified reference (tests/golden) and against the CPU oracle.

Bars: features, row order, prune verdicts and structural hashes bit-exact;
per-row and total predicted costs within 1e-9 relative (north-star bar is
1e-5; fp64 on both sides, only summation order differs)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import PARAMS, available_sets, candidate_set, weights  # noqa: E402

pytestmark = pytest.mark.gpu

COST_RTOL = 1e-9
PRUNE_CODE = {None: 0, "excessive_recompute": 1, "idle_sms": 2, "poor_warp_utilization": 3,
              "serial_too_large": 4, "thread_alloc_dynamic_or_large": 5, "hardware_limit": 6}


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _scorer(cs, thresholds=None):
    from paper_2012_07145_b200.engine import Scorer
    return Scorer(cs.graph, PARAMS, thresholds or cs.thresholds, weights())


@pytest.mark.parametrize("name", available_sets())
def test_features_costs_hashes_match_reference(name, dev):
    cs = candidate_set(name)
    sc = _scorer(cs)
    dec = sc.upload(cs.decisions)
    f = sc.featurize(dec)
    total, rowc, gh = sc.cost(f, rows=True, basis=True)
    sc.check()
    feats = f["feats"].cpu().numpy()
    keys = f["row_key"].cpu().numpy()
    nrows = f["n_rows"].cpu().numpy()
    verdict = f["verdict"].cpu().numpy()
    total, rowc, gh = total.cpu().numpy(), rowc.cpu().numpy(), gh.cpu().numpy()
    for i in range(len(cs)):
        c = cs.cand(i)
        R = len(c["rows"])
        assert nrows[i] == R, (name, i)
        assert sc.packed.row_keys(keys[i, :R]) == c["rows"], (name, i)
        bad = np.argwhere(feats[i, :R] != c["feats"])
        assert bad.size == 0, (name, i, [(c["rows"][r], k, feats[i, r, k], c["feats"][r, k])
                                         for r, k in bad[:6]])
        assert np.array_equal(gh[i, :R, :30], c["g"]), (name, i)
        assert np.array_equal(gh[i, :R, 30], c["h"]), (name, i)
        np.testing.assert_allclose(rowc[i, :R], c["rowcost"], rtol=COST_RTOL)
        assert total[i] == pytest.approx(c["total"], rel=COST_RTOL)
        assert verdict[i] == PRUNE_CODE[c["prune"]], (name, i, verdict[i], c["prune"])
    for depth in range(6):
        h = sc.struct_hash(dec, depth).cpu().numpy().view(np.uint64)
        want = np.array([cs.hashes[i][depth] for i in range(len(cs))], dtype=np.uint64)
        assert np.array_equal(h, want), (name, depth)
    # several depths in one K3 pass (the beam step's pass + memo depths)
    for depths in ([0, 1, 2, 3], [5, 1, 4]):
        H = sc.struct_hash_depths(dec, depths).cpu().numpy().view(np.uint64)
        for row, depth in enumerate(depths):
            want = np.array([cs.hashes[i][depth] for i in range(len(cs))], dtype=np.uint64)
            assert np.array_equal(H[row], want), (name, depths, depth)


@pytest.mark.parametrize("name", ["chain3", "diamond", "stencil_chain"])
def test_open_thresholds_prune(name, dev):
    from paper_2012_07145_b200.params import OPEN_THRESHOLDS
    cs = candidate_set(name)
    sc = _scorer(cs, OPEN_THRESHOLDS)
    f = sc.featurize(sc.upload(cs.decisions))
    sc.check()
    v = f["verdict"].cpu().numpy()
    assert [int(x) for x in v] == [PRUNE_CODE[p] for p in cs.prune_open]


def test_small_tower_weights(dev):
    """Network dims other than 32/64 (reference test_costmodel.py:123-131)."""
    from oracle import costing
    cs = candidate_set("stencil_chain")
    w = weights("small")
    from paper_2012_07145_b200.engine import Scorer
    sc = Scorer(cs.graph, PARAMS, cs.thresholds, w)
    f = sc.featurize(sc.upload(cs.decisions[:10]))
    total, _, _ = sc.cost(f)
    sc.check()
    for i in range(10):
        want, _, _ = costing.score(cs.graph, cs.decisions[i], PARAMS, w.tensors)
        assert total[i].item() == pytest.approx(want, rel=COST_RTOL)
