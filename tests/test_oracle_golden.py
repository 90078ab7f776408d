"""Pin the CPU oracle against vectors produced by the unmodified reference.

Features and structural hashes must match exactly; per-row and total costs
to 1e-12 relative (the reference's fp64 values depend on the OpenBLAS kernel
order, see tests/golden/provenance.json); prune verdicts exactly.
"""

import numpy as np
import pytest

from golden_io import PARAMS, available_sets, candidate_set, search_trace, weights, SEARCHES
from oracle import costing, features, structure
from paper_2012_07145_b200.params import OPEN_THRESHOLDS


@pytest.mark.parametrize("name", available_sets())
def test_oracle_features_and_costs(name):
    cs = candidate_set(name)
    w = weights().tensors
    limit = 4 if name in ("chain100", "camera_pipe", "local_laplacian") else len(cs)
    for i in range(min(limit, len(cs))):
        c = cs.cand(i)
        total, per, rows = costing.score(cs.graph, c["decisions"], PARAMS, w)
        assert [k for k, _, _ in rows] == c["rows"], (name, i)
        got = np.array([f for _, f, _ in rows])
        bad = np.argwhere(got != c["feats"])
        assert bad.size == 0, (name, i, [(c["rows"][r], features.FEATURES[k], got[r, k],
                                          c["feats"][r, k]) for r, k in bad[:5]])
        assert np.array_equal(np.array([a for _, _, a in rows]), c["algo"])
        for r, (_, f, _) in enumerate(rows):
            g, h = costing.basis(f)
            assert np.array_equal(g, c["g"][r]) and h == c["h"][r]
        np.testing.assert_allclose([x for _, x in per], c["rowcost"], rtol=1e-12)
        assert total == pytest.approx(c["total"], rel=1e-12)


@pytest.mark.parametrize("name", available_sets())
def test_oracle_hash_and_prune(name):
    cs = candidate_set(name)
    for i in range(len(cs)):
        c = cs.cand(i)
        for d in range(6):
            assert structure.structural_hash(c["decisions"], d) == c["hashes"][d]
        assert costing.prune_reason(cs.graph, c["decisions"], PARAMS, cs.thresholds) == c["prune"]
        assert (costing.prune_reason(cs.graph, c["decisions"], PARAMS, OPEN_THRESHOLDS)
                == cs.prune_open[i])


def test_canonical_bytes_appendix_c():
    """SURVEY Appendix C / loopnest.py:131-165 example bytes and digests."""
    from paper_2012_07145_b200.schedule import Decision
    dec = (("blur_y", Decision("compute_root", serial=(1, 2), thread=(32, 4))),
           ("blur_x", Decision("fuse_at_block", consumer="blur_y", serial=(1, 2))))
    assert structure.canonical_bytes(dec, 0) == b"('kernels', ('blur_y',))"
    assert structure.structural_hash(dec, 0) == 0xf6e861dab17d3835
    assert structure.structural_hash(dec, 1) == 0x7da3fd4469713486
    assert structure.structural_hash(dec, 2) == 0x2464d1e18b8acc15
    assert structure.structural_hash(dec, 3) == 0x483e59bfb27ab5ff


@pytest.mark.parametrize("tag", [t for t in SEARCHES if t != "stencil_chain"])
def test_oracle_cut_matches_reference_trace(tag):
    """Replay every traced _cut of a real reference search with the oracle."""
    tr = search_trace(tag)
    cfg = tr["config"]
    th = cfg["thresholds"]
    from paper_2012_07145_b200.params import Thresholds
    th = Thresholds(**th)
    graph = tr["graph"]
    w = weights().tensors
    for call in tr["calls"][:12]:
        cands = call["candidates"]
        p = call["pass_index"]
        hashes = [structure.structural_hash(c, p) for c in cands]
        valid = [costing.prune_reason(graph, c, PARAMS, th) is None for c in cands]
        reps, rejects = structure.select_reps(hashes, valid, call["phase_seed"])
        assert len(rejects) == call["n_reports"]
        if not reps:
            assert call["beam"] == []
            continue
        costs = [costing.score(graph, cands[i], PARAMS, w)[0] for i in reps]
        flagged = {h for d, h in call["memo_before"] if d == p}
        keep, bottom = structure.cut(reps, costs, [hashes[i] for i in reps], flagged,
                                     cfg["penalty_factor"], cfg["beam_size"],
                                     cfg["explore_temperature"], call["phase_seed"])
        assert [cands[reps[k]] for k in keep] == call["beam"]
        memo = set(call["memo_before"])
        for k in bottom:
            for d in range(1, cfg["num_passes"] + 1):
                memo.add((d, structure.structural_hash(cands[reps[k]], d)))
        assert memo == call["memo_after"]
