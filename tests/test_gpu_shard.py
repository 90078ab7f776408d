"""The sharded beam step (shard.StepPlan + exchange.sharded_cut, SURVEY
§8(e)) on the GPU: two ranks on the one device of a gpurun box (gloo
carries the window records and histograms; on a multi-GPU node the same
code runs one rank per GPU over NCCL) must cut exactly the beam a single
rank cuts, with every rank featurizing only its own buckets."""

import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as tmp  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
PARENTS = 40


def _plan(world, rank):
    sys.path.insert(0, ROOT)
    import bench
    from paper_2012_07145_b200 import shard
    from paper_2012_07145_b200.engine import TIE_BAND, Scorer
    from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights
    graph, recs, _ = bench._workload(PARENTS)
    sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
    dec = sc.to_device(recs)
    plan = shard.StepPlan(sc, len(recs), world, rank, bench.PASS_INDEX, bench.PHASE_SEED, bench.BEAM, 2.0,
                          bench.NUM_PASSES, TIE_BAND)
    return plan, dec


def _rank(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan, dec = _plan(world, rank)
        out = plan.run(dec)
        memo = [sorted(int(x) for x in m.cpu().tolist()) for m in out["memo"]]
        q.put((rank, out["beam"], plan.local_count, out["n_reps"], memo))
    finally:
        dist.destroy_process_group()


def test_two_rank_step_cuts_the_single_rank_beam():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    plan, dec = _plan(1, 0)
    want = plan.run(dec)
    want_memo = [sorted(int(x) for x in m.cpu().tolist()) for m in want["memo"]]
    n = dec.shape[0]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sum(g[2] for g in got) == n                 # buckets partition the step
    assert all(0 < g[2] < n for g in got)
    for rank, beam, _, n_reps, memo in got:
        assert beam == want["beam"], rank
        assert n_reps == want["n_reps"]
    # each rank records the memo entries of its own bottom-half reps; together
    # they are the single-rank memo
    for depth in range(len(want_memo)):
        assert sorted(set(x for g in got for x in g[4][depth])) == sorted(set(want_memo[depth])), depth


def _search_rank(rank, world, port, q, tag):
    import importlib
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
        ref = os.path.join(ROOT, "baseline", "_ref")
        if ref not in sys.path:
            sys.path.append(ref)
        import gpusched.search as gs
        from gpusched.costmodel import load_weights
        from gpusched.loopnest import schedule_dump
        from gpusched.machine import MachineParams
        from gpusched.options import Thresholds, TilingConfig
        from gpusched.pipeline import parse_pipeline
        from golden_io import search_trace
        ev_mod = importlib.import_module("paper_2012_07145_b200.evaluator")
        tr = search_trace(tag)
        cfg = tr["config"]
        graph = parse_pipeline(tr["pipeline"], name=tag)
        scfg = gs.SearchConfig(beam_size=cfg["beam_size"], num_passes=cfg["num_passes"],
                               penalty_factor=cfg["penalty_factor"], seed=cfg["seed"],
                               explore_temperature=cfg["explore_temperature"],
                               freeze_enabled=cfg["freeze_enabled"], thresholds=Thresholds(**cfg["thresholds"]),
                               tiling=TilingConfig(**{k: tuple(v) if isinstance(v, list) else v
                                                      for k, v in cfg["tiling"].items()}))
        w = load_weights(os.path.join(ROOT, "tests", "golden", "weights_seed0.txt"))
        ev = ev_mod.GpuCostEvaluator(w, MachineParams(), scfg.thresholds)
        ev_mod.configure_sharding(True)
        with ev_mod.installed(gs, expand=True):
            if cfg["freeze_enabled"]:
                final = gs.schedule_with_freezing(graph, MachineParams(), scfg, ev)
            else:
                final = gs.schedule_pipeline(graph, MachineParams(), scfg, ev)
        q.put((rank, [schedule_dump(s) for s in final], [s.cost for s in final]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tag", ["stencil_chain", "chain16_freeze"])
def test_two_rank_reference_search_through_the_seam(tag):
    """The unchanged reference search, run by two ranks with the sharded cut
    behind the seam (configure_sharding + install(expand=True)), returns the
    traced single-process reference beam on both ranks."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "gpusched")):
        pytest.skip("reference package not installed (baseline/_ref)")
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    from golden_io import search_trace
    from paper_2012_07145_b200.schedule import parse_dump
    tr = search_trace(tag)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_search_rank, args=(r, 2, port, q, tag)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, final, costs in got:
        assert [parse_dump(t) for t in final] == tr["final"], rank
        for c, want in zip(costs, tr["final_costs"]):
            assert c == pytest.approx(want, rel=1e-9)
