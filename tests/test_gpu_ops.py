"""GPU: the torch.ops.gsched custom ops pass torch.library.opcheck (schema,
fake kernels against the real ones, AOT dispatch) and equal the Scorer's
direct C-ABI calls; one whole phase cut captured in a CUDA graph
(graph.CapturedStep) replays bit-exact against StepPlan.run — on the batch it
was captured with and on a different batch copied into its static input —
and against the reference's own cut of the 1,000,080-candidate C5 step."""

import gzip
import json
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import PARAMS, candidate_set, weights  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
REL = 1e-9


@pytest.fixture(scope="module")
def small():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2012_07145_b200 import ops  # noqa: F401
    from paper_2012_07145_b200.engine import Scorer
    cs = candidate_set("stencil_chain")
    sc = Scorer(cs.graph, PARAMS, cs.thresholds, weights())
    return cs, sc, sc.upload(cs.decisions)


def test_opcheck_all_ops(small):
    from paper_2012_07145_b200 import ops
    cs, sc, dec = small
    h = sc.handle.value
    feats, row_key, n_rows, verdict, row_src = torch.ops.gsched.featurize(h, dec, sc.R, 1)
    hashes = torch.ops.gsched.struct_hash(h, dec, 2)
    total, _, _ = torch.ops.gsched.cost(h, feats, row_key, n_rows, row_src)
    rep, _, cnt = torch.ops.gsched.select_reps(hashes, verdict, 11)
    cases = [
        (torch.ops.gsched.featurize.default, (h, dec, sc.R, 1)),
        (torch.ops.gsched.cost.default, (h, feats, row_key, n_rows, row_src)),
        (torch.ops.gsched.cost.default, (h, feats, row_key, n_rows, None, True)),
        (torch.ops.gsched.struct_hash.default, (h, dec, 3)),
        (torch.ops.gsched.select_reps.default, (hashes, verdict, 11)),
        (torch.ops.gsched.beam_topk.default, (total, hashes, rep, cnt[:1].clone(), None, 2.0, 0.0, 11, 4, 1e-14)),
        (torch.ops.gsched.beam_topk.default, (total, hashes, rep, cnt[:1].clone(), None, 2.0, 0.5, 11, 4, 1e-14)),
    ]
    for op, args in cases:
        torch.library.opcheck(op, args)
    # expand_step on phase-2 parents of the C5 chain
    import bench
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams
    z = np.load(bench.PARENTS_FILE)
    graph, _, _ = bench._workload(2)
    sc5 = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS)
    par = torch.as_tensor(np.ascontiguousarray(z["parents"][:3]), device="cuda")
    st = torch.as_tensor(z["steps"][:3].astype(np.int32), device="cuda")
    torch.library.opcheck(torch.ops.gsched.expand_step.default, (sc5.handle.value, par, st, 720, *ops.menu_args()))


def test_ops_equal_direct_calls(small):
    cs, sc, dec = small
    h = sc.handle.value
    f = sc.featurize(dec)
    t_direct, _, _ = sc.cost(f)
    feats, row_key, n_rows, verdict, row_src = torch.ops.gsched.featurize(h, dec, sc.R, 1)
    total, _, _ = torch.ops.gsched.cost(h, feats, row_key, n_rows, row_src)
    sc.check()
    assert torch.equal(verdict, f["verdict"]) and torch.equal(n_rows, f["n_rows"])
    for i in range(dec.shape[0]):
        r = int(n_rows[i])
        assert torch.equal(feats[i, :r], f["feats"][i, :r])
    assert torch.equal(total, t_direct)
    for depth in range(5):
        assert torch.equal(torch.ops.gsched.struct_hash(h, dec, depth), sc.struct_hash(dec, depth))


def _c5(parents, offset=0):
    import bench
    from paper_2012_07145_b200.descriptor import DECISION_DTYPE
    from paper_2012_07145_b200.gen import expand_step
    graph, _, _ = bench._workload(1)
    z = np.load(bench.PARENTS_FILE)
    par = np.ascontiguousarray(z["parents"]).view(DECISION_DTYPE).reshape(len(z["parents"]), -1)
    recs, _ = expand_step(par[offset:offset + parents], z["steps"][offset:offset + parents], graph)
    return graph, recs


def _same(a, b):
    from paper_2012_07145_b200.graph import memo_set
    assert a["beam"] == b["beam"]
    np.testing.assert_allclose(a["beam_costs"], b["beam_costs"], rtol=0, atol=0)
    assert torch.equal(a["reps"], b["reps"])
    assert a["rejects"] == b["rejects"]
    assert memo_set(a["memo"]) == memo_set(b["memo"])


@pytest.mark.parametrize("temperature", [0.0, 0.5])
def test_captured_step_replays_bit_exact(temperature):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench
    from paper_2012_07145_b200 import shard
    from paper_2012_07145_b200.engine import TIE_BAND, Scorer
    from paper_2012_07145_b200.graph import CapturedStep
    from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights
    graph, recs_a = _c5(60, 0)
    _, recs_b = _c5(60, 200)
    sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
    da, db = sc.to_device(recs_a), sc.to_device(recs_b)
    n, S = da.shape[0], da.shape[1] // 16
    plan = shard.StepPlan(sc, n, 1, 0, bench.PASS_INDEX, bench.PHASE_SEED, 8, 2.0, bench.NUM_PASSES, TIE_BAND)
    ref_a = plan.run(da, temperature=temperature, rejects=True)
    flagged = [int(x) for x in ref_a["memo"][bench.PASS_INDEX - 1].cpu().numpy().view(np.uint64)[:7]]
    ref_a = plan.run(da, flagged=flagged, temperature=temperature, rejects=True)
    ref_b = plan.run(db, flagged=flagged, temperature=temperature, rejects=True)
    cap = CapturedStep(sc, n, S, bench.PASS_INDEX, bench.PHASE_SEED, 8, 2.0, bench.NUM_PASSES, flagged=flagged,
                       temperature=temperature)
    cap.dec.copy_(da)
    cap.capture()
    cap.replay()
    _same(cap.result(), ref_a)
    cap.replay(db)
    _same(cap.result(), ref_b)
    cap.replay(da)
    _same(cap.result(), ref_a)


def test_captured_c5_step_equals_reference_cut():
    """The full bench step (memo variant) replayed from a CUDA graph against
    the unmodified reference's `_cut` (tests/golden/c5_step)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.graph import CapturedStep, memo_set
    from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights
    gold = os.path.join(ROOT, "tests", "golden")
    with gzip.open(os.path.join(gold, "c5_step.json.gz"), "rt") as fh:
        meta = json.load(fh)
    arr = np.load(os.path.join(gold, "c5_step.npz"))
    cut = meta["cut"]
    v = cut["variants"]["memo"]
    graph, recs, _ = bench._workload(meta["parents"])
    sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
    before = {(int(d), int(h) & 0xFFFFFFFFFFFFFFFF) for d, h in v["memo_before"]}
    flagged = [h for d, h in before if d == cut["pass_index"]]
    cap = CapturedStep(sc, len(recs), recs.shape[1], cut["pass_index"], bench.PHASE_SEED, bench.BEAM, 2.0,
                       bench.NUM_PASSES, flagged=flagged, temperature=v["temperature"])
    cap.dec.copy_(sc.to_device(recs))
    cap.capture()
    cap.replay()
    out = cap.result()
    assert out["n_reps"] == cut["n_reps"]
    assert np.array_equal(out["reps"].cpu().numpy(), arr["rep_idx"])
    assert [i for i, _ in out["rejects"]] == arr["rej_idx"].tolist()
    assert out["beam"] == v["beam"]
    np.testing.assert_allclose(out["beam_costs"], v["beam_costs"], rtol=REL, atol=0)
    assert before | memo_set(out["memo"]) == {(int(d), int(h) & 0xFFFFFFFFFFFFFFFF) for d, h in v["memo_after"]}
