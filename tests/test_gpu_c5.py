"""Parity at the headline scale: the 1,000,080-candidate C5 beam step the
bench times (bench.py), checked against fixtures the UNMODIFIED reference
wrote for that exact step (tests/golden/make_c5_golden.py):

* 1,024 candidates strided over the step: features (sha256 of each
  candidate's fp64 [R, 56] block, full blocks for every 16th), row keys,
  row costs and totals, prune verdicts and hashes at depths 0-5 — taken
  from the bench-mode step itself (two-phase K1, reuse mode 2: the rows are
  gathered through row_src), not from a separate small batch;
* the reference `_cut` over the whole step (beam 32, pass 3) in three
  variants — the bench's (empty memo, T = 0), a seeded memo (T = 0) and the
  same memo at T = 0.5: representatives and drawn rejects in order, every
  representative's cost, the beam, its costs and the memo after the call,
  through `StepPlan.run` (the cut `gpu_cut` and the bench use)."""

import gzip
import hashlib
import json
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLD = os.path.join(ROOT, "tests", "golden")
REL = 1e-9   # fp64 cost tolerance (north-star bar: 1e-5)


@pytest.fixture(scope="module")
def golden():
    with gzip.open(os.path.join(GOLD, "c5_step.json.gz"), "rt") as fh:
        meta = json.load(fh)
    arr = np.load(os.path.join(GOLD, "c5_step.npz"))
    return meta, arr


@pytest.fixture(scope="module")
def step(golden):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    import bench
    from paper_2012_07145_b200 import shard
    from paper_2012_07145_b200.engine import TIE_BAND, Scorer
    from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights
    meta, _ = golden
    graph, recs, _ = bench._workload(meta["parents"])
    assert len(recs) == meta["n_candidates"]
    sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
    dec = sc.to_device(recs)
    plan = shard.StepPlan(sc, len(recs), 1, 0, bench.PASS_INDEX, bench.PHASE_SEED, bench.BEAM, 2.0,
                          bench.NUM_PASSES, TIE_BAND)
    return sc, dec, plan


def _u64(x):
    return int(x) & 0xFFFFFFFFFFFFFFFF


def test_sample_features_costs_verdicts_hashes(golden, step):
    meta, arr = golden
    sc, dec, plan = step
    out = plan.run(dec)
    sc.check()
    f = plan.fbuf
    idx = torch.as_tensor(arr["sample_index"], device=sc.device)
    n_rows = f["n_rows"].index_select(0, idx).cpu().numpy()
    src = f["row_src"].index_select(0, idx).cpu().numpy()
    keys = f["row_key"].index_select(0, idx).cpu().numpy()
    tot = out["total"].index_select(0, idx).cpu().numpy()
    ver = out["verdict"].index_select(0, idx).cpu().numpy()
    from paper_2012_07145_b200.descriptor import PRUNE_REASONS
    off = arr["row_offsets"]
    # the bench-mode rows of candidate i: row r was written by candidate src[i, r]
    R = sc.R
    r_ix = np.arange(R)[None, :]
    flat = np.where(r_ix < n_rows[:, None], src, 0).astype(np.int64) * R + r_ix
    gathered = f["feats"].view(-1, f["feats"].shape[-1]).index_select(
        0, torch.as_tensor(flat.reshape(-1), device=sc.device)).view(len(flat), R, -1).cpu().numpy()
    full_i = 0
    for j, i in enumerate(arr["sample_index"]):
        n = int(n_rows[j])
        assert n == off[j + 1] - off[j], i
        rows = gathered[j, :n]
        assert hashlib.sha256(np.ascontiguousarray(rows).tobytes()).hexdigest() == meta["feat_sha256"][j], i
        if j % meta["full_features_every"] == 0:
            fo = arr["full_offsets"]
            assert np.array_equal(rows, arr["full_feats"][fo[full_i]:fo[full_i + 1]])
            full_i += 1
        assert [list(k) for k in sc.packed.row_keys(keys[j, :n])] == meta["rows"][j], i
        want = arr["total"][j]
        assert abs(tot[j] - want) <= REL * abs(want), i
        reason = PRUNE_REASONS[ver[j] - 1] if ver[j] else None
        assert reason == meta["prune"][j], i
    # per-row costs of the sample (K2 rows through row_src)
    _, rc, _ = sc.cost(plan.fbuf, rows=True, scratch=plan.rcbuf)
    rc = rc.index_select(0, idx).cpu().numpy()
    want_rc = arr["rowcost"]
    for j in range(len(arr["sample_index"])):
        a, b = off[j], off[j + 1]
        np.testing.assert_allclose(rc[j, :b - a], want_rc[a:b], rtol=REL, atol=0)
    # hashes at depths 0-5 of the sampled candidates, on the step's records
    d = dec.index_select(0, idx)
    for depth in range(6):
        hs = sc.struct_hash(d, depth).cpu().numpy().view(np.uint64)
        assert [str(int(x)) for x in hs] == [h[depth] for h in meta["hashes"]], depth


def test_multi_depth_hash_on_full_step(step):
    """One K3 pass at the pass depth and the memo depths equals one pass per
    depth over the whole 1M-candidate step (run heads hashed, followers
    filled at every depth)."""
    sc, dec, _ = step
    depths = [3, 1, 2]
    H = sc.struct_hash_depths(dec, depths)
    for row, depth in enumerate(depths):
        assert torch.equal(H[row], sc.struct_hash(dec, depth)), depth


@pytest.mark.parametrize("variant", ["bench", "memo", "memo_T05"])
def test_full_step_cut_equals_reference(golden, step, variant):
    meta, arr = golden
    sc, dec, plan = step
    cut = meta["cut"]
    v = cut["variants"][variant]
    before = {(int(dd), _u64(h)) for dd, h in v["memo_before"]}
    flagged = [h for dd, h in before if dd == cut["pass_index"]]
    out = plan.run(dec, flagged=flagged, temperature=v["temperature"], rejects=True)
    sc.check()
    reps = out["reps"].cpu().numpy()
    assert out["n_reps"] == cut["n_reps"]
    assert np.array_equal(reps, arr["rep_idx"])                   # bucket order + PCG64 walk
    assert [i for i, _ in out["rejects"]] == arr["rej_idx"].tolist()
    assert [r for _, r in out["rejects"]] == cut["reject_reasons"]
    rep_cost = out["total"].index_select(0, out["reps"]).cpu().numpy()
    np.testing.assert_allclose(rep_cost, arr["rep_cost"], rtol=REL, atol=0)
    assert out["beam"] == v["beam"]                               # bit-exact beam, in order
    np.testing.assert_allclose(out["beam_costs"], v["beam_costs"], rtol=REL, atol=0)
    new = {(depth, _u64(x)) for depth, hs in enumerate(out["memo"], start=1)
           for x in hs.cpu().numpy().view(np.uint64)}
    assert before | new == {(int(dd), _u64(h)) for dd, h in v["memo_after"]}
