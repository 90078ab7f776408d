"""GPU selection parity: every `_cut` call traced from real reference searches
(tests/golden/search_*.json.gz) is replayed through the B200 path (K1 prune,
K3 hash, K4 buckets + PCG64 representatives, K2 cost, K5 top-k); the beam,
its order, the bad-hash memo and the reject count must match bit-exactly."""

import os
import sys

import pytest

torch = pytest.importorskip("torch")

from golden_io import PARAMS, search_tags, search_trace, weights  # noqa: E402

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


@pytest.mark.parametrize("tag", search_tags())
def test_cut_replay_bit_exact(tag, dev):
    from paper_2012_07145_b200.cut import beam_cut
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.params import Thresholds
    tr = search_trace(tag)
    cfg = tr["config"]
    sc = Scorer(tr["graph"], PARAMS, Thresholds(**cfg["thresholds"]), weights())
    for ci, call in enumerate(tr["calls"]):
        cands = call["candidates"]
        p = call["pass_index"]
        flagged = [h for d, h in call["memo_before"] if d == p]
        res = beam_cut(sc, sc.upload(cands), p, call["phase_seed"], flagged, cfg["beam_size"],
                       cfg["penalty_factor"], cfg["explore_temperature"], cfg["num_passes"])
        assert len(res.rejects) == call["n_reports"], (tag, ci)
        assert [r for _, r in res.rejects] == call["report_reasons"], (tag, ci)
        got = [cands[i] for i in res.beam]
        assert got == call["beam"], (tag, ci)
        for c, want in zip(res.costs, call["beam_costs"]):
            assert c == pytest.approx(want, rel=1e-9)
        assert set(call["memo_before"]) | res.memo_new == call["memo_after"], (tag, ci)


def _reference_on_path():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "gpusched")) and ref not in sys.path:
        sys.path.append(ref)
    try:
        import gpusched  # noqa: F401
        return True
    except ImportError:
        return False


@pytest.mark.parametrize("expand", [False, True])
@pytest.mark.parametrize("tag", ["chain2", "diamond", "stencil_chain", "chain16_freeze"])
def test_reference_search_drives_gpu_path(tag, expand, dev):
    """The UNCHANGED reference search with the GPU evaluator + `_cut` hook
    returns the same final beam as the pure-CPU reference run — and with
    expand=True also with its candidate generation on the device (phase-1 /
    phase-2 groups expanded inside gpu_cut, host states only for beams)."""
    if not _reference_on_path():
        pytest.skip("reference package not installed (baseline/_ref)")
    import importlib
    import gpusched.search as gs
    from gpusched.costmodel import load_weights
    from gpusched.machine import MachineParams
    from gpusched.options import Thresholds, TilingConfig
    from gpusched.pipeline import parse_pipeline
    from gpusched.loopnest import schedule_dump
    ev_mod = importlib.import_module("paper_2012_07145_b200.evaluator")
    if not ev_mod.HAVE_REFERENCE:
        ev_mod = importlib.reload(ev_mod)
    tr = search_trace(tag)
    cfg = tr["config"]
    graph = parse_pipeline(tr["pipeline"], name=tag)
    scfg = gs.SearchConfig(beam_size=cfg["beam_size"], num_passes=cfg["num_passes"],
                           penalty_factor=cfg["penalty_factor"], seed=cfg["seed"],
                           explore_temperature=cfg["explore_temperature"],
                           freeze_enabled=cfg["freeze_enabled"],
                           thresholds=Thresholds(**cfg["thresholds"]),
                           tiling=TilingConfig(**{k: tuple(v) if isinstance(v, list) else v
                                                  for k, v in cfg["tiling"].items()}))
    w = load_weights(os.path.join(ROOT, "tests", "golden", "weights_seed0.txt"))
    params = MachineParams()
    ev = ev_mod.GpuCostEvaluator(w, params, scfg.thresholds)
    with ev_mod.installed(gs, expand=expand):
        if cfg["freeze_enabled"]:
            final = gs.schedule_with_freezing(graph, params, scfg, ev)
        else:
            final = gs.schedule_pipeline(graph, params, scfg, ev)
    from paper_2012_07145_b200.schedule import parse_dump
    assert [parse_dump(schedule_dump(s)) for s in final] == tr["final"]
    for s, c in zip(final, tr["final_costs"]):
        assert s.cost == pytest.approx(c, rel=1e-9)
