"""Generate golden parity fixtures by running the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports `gpusched` from /root/reference/pkg/src (and the reference test
helpers `conftest.make_chain_src`, `test_acceptance._random_schedule`) and
writes, per pipeline:

  <name>.json.gz — pipeline text, candidate decision logs (schedule_dump
                   format), row keys, prune verdicts, structural hashes
  <name>.npz     — fp64 features [rows, 56], algo [rows, 10], basis g/h,
                   per-row costs and per-candidate totals
  search_<name>.json.gz — every `_cut` call of real searches (inputs, memo,
                   representatives, costs, returned beam) and final beams

The NumPy / BLAS build that produced them is recorded in `provenance.json`.
"""

from __future__ import annotations

import gzip
import io
import json
import math
import os
import sys
import contextlib
import zlib

import numpy as np

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src"), os.path.join(REF, "tests")]
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import gpusched  # noqa: E402
import gpusched.search as gsearch  # noqa: E402
from gpusched.costmodel import init_weights, save_weights, stage_cost_basis, _forward  # noqa: E402
from gpusched.featurize import featurize  # noqa: E402
from gpusched.loopnest import schedule_dump, structural_hash  # noqa: E402
from gpusched.machine import MachineParams  # noqa: E402
from gpusched.options import DEFAULT_THRESHOLDS, TilingConfig, prune  # noqa: E402
from gpusched.pipeline import builtin_pipeline, parse_pipeline  # noqa: E402
from gpusched.search import CostEvaluator, SearchConfig  # noqa: E402

from conftest import CHAIN2_SRC, CHAIN3_SRC, DIAMOND_SRC, OPEN_THRESHOLDS, make_chain_src  # noqa: E402
from test_acceptance import SELF_READ_SRC, STRIDED_SRC, TINY_FORK_SRC, _random_schedule  # noqa: E402

from paper_2012_07145_b200.pipeline import graph_to_text  # noqa: E402

PIPE_DIR = os.path.join(HERE, "..", "..", "paper_2012_07145_b200", "pipelines")


def authored(name):
    with open(os.path.join(PIPE_DIR, f"{name}.txt")) as fh:
        return parse_pipeline(fh.read(), name=name)


def graphs():
    out = {
        "chain2": (parse_pipeline(CHAIN2_SRC, "chain2"), 40, OPEN_THRESHOLDS),
        "chain3": (parse_pipeline(CHAIN3_SRC, "chain3"), 40, OPEN_THRESHOLDS),
        "diamond": (parse_pipeline(DIAMOND_SRC, "diamond"), 40, OPEN_THRESHOLDS),
        "self_read": (parse_pipeline(SELF_READ_SRC, "self_read"), 30, OPEN_THRESHOLDS),
        "strided": (parse_pipeline(STRIDED_SRC, "strided"), 30, OPEN_THRESHOLDS),
        "tiny_fork": (parse_pipeline(TINY_FORK_SRC, "tiny_fork"), 20, OPEN_THRESHOLDS),
        "blur": (builtin_pipeline("blur"), 48, DEFAULT_THRESHOLDS),
        "conv": (builtin_pipeline("conv"), 12, DEFAULT_THRESHOLDS),
        "stencil_chain": (builtin_pipeline("stencil_chain"), 32, DEFAULT_THRESHOLDS),
        "chain20": (parse_pipeline(make_chain_src(20, extent=512), "chain20"), 12, DEFAULT_THRESHOLDS),
        "chain100": (parse_pipeline(make_chain_src(100, extent=1024), "chain100"), 6, DEFAULT_THRESHOLDS),
    }
    for name in ("unsharp", "harris", "resnet_small", "camera_pipe", "local_laplacian"):
        if os.path.exists(os.path.join(PIPE_DIR, f"{name}.txt")):
            n = 16 if name in ("unsharp", "harris", "resnet_small") else 4
            out[name] = (authored(name), n, DEFAULT_THRESHOLDS)
    return out


def _partial_states(graph, rng, k):
    """Phase-1 style partial states: a random prefix of a random schedule."""
    full = _random_schedule(graph, rng)
    out = []
    funcs = full.schedulable_funcs()
    for _ in range(k):
        n = int(rng.integers(1, len(funcs) + 1))
        st = gpusched.initial_state(graph)
        for f in funcs[:n]:
            d = full.decision(f)
            if d.kind == "compute_root":
                d = gpusched.Decision("compute_root")
            st = gpusched.apply_decision(st, f, d)
        out.append(st)
    return out


def record_candidates(name, graph, n_full, thresholds, params, weights):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    states = [_random_schedule(graph, rng) for _ in range(n_full)]
    states += _partial_states(graph, rng, max(2, n_full // 4))
    ev = CostEvaluator(weights, params)
    meta = {"pipeline": graph_to_text(graph), "name": name, "candidates": [],
            "rows": [], "prune": [], "prune_open": [], "hashes": [], "full": []}
    feats, algo, gs, hs, rc, tot, offs = [], [], [], [], [], [], [0]
    for st in states:
        meta["candidates"].append(schedule_dump(st))
        meta["full"].append(bool(st.fully_scheduled(graph)))
        basis = ev.stage_basis(st, graph)
        total, per = ev.cost(st, graph)
        meta["rows"].append([[k[0], k[1]] for k, *_ in basis])
        for (k, xa, xs, g, h) in basis:
            feats.append(xs)
            algo.append(xa)
            gs.append(g)
            hs.append(h)
            rc.append(per[k])
        tot.append(total)
        offs.append(offs[-1] + len(basis))
        r = prune(st, graph, params, thresholds)
        meta["prune"].append(r.reason if r else None)
        r = prune(st, graph, params, OPEN_THRESHOLDS)
        meta["prune_open"].append(r.reason if r else None)
        meta["hashes"].append([str(structural_hash(st, d)) for d in range(6)])
    meta["thresholds"] = thresholds.__dict__
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                        feats=np.array(feats), algo=np.array(algo), g=np.array(gs),
                        h=np.array(hs), rowcost=np.array(rc), total=np.array(tot),
                        offsets=np.array(offs))
    with gzip.open(os.path.join(HERE, f"{name}.json.gz"), "wt") as fh:
        json.dump(meta, fh)
    return len(states), offs[-1]


def record_search(tag, graph, cfg, params, weights, freeze=False):
    """Trace every _cut call of a real search."""
    calls = []
    orig_cut = gsearch._cut

    def traced(candidates, evaluator, graph_, config, pass_index, memo, phase_seed, validate):
        before = sorted([list(map(str, x)) for x in memo.flagged])
        beam, reports = orig_cut(candidates, evaluator, graph_, config, pass_index, memo,
                                 phase_seed, validate)
        after = sorted([list(map(str, x)) for x in memo.flagged])
        calls.append({
            "pass_index": pass_index, "phase_seed": phase_seed,
            "candidates": [schedule_dump(c) for c in candidates],
            "memo_before": before, "memo_after": after,
            "beam": [schedule_dump(s) for s in beam],
            "beam_costs": [s.cost for s in beam],
            "n_reports": len(reports),
            "report_reasons": [r.reason for r in reports],
        })
        return beam, reports

    gsearch._cut = traced
    try:
        ev = CostEvaluator(weights, params)
        if freeze:
            final = gsearch.schedule_with_freezing(graph, params, cfg, ev)
        else:
            final = gsearch.schedule_pipeline(graph, params, cfg, ev)
    finally:
        gsearch._cut = orig_cut
    out = {"pipeline": graph_to_text(graph), "config": {
        "beam_size": cfg.beam_size, "num_passes": cfg.num_passes,
        "penalty_factor": cfg.penalty_factor, "seed": cfg.seed,
        "explore_temperature": cfg.explore_temperature, "freeze_enabled": cfg.freeze_enabled,
        "thresholds": cfg.thresholds.__dict__, "tiling": cfg.tiling.__dict__},
        "calls": calls, "final": [schedule_dump(s) for s in final],
        "final_costs": [s.cost for s in final]}
    with gzip.open(os.path.join(HERE, f"search_{tag}.json.gz"), "wt") as fh:
        json.dump(out, fh)
    return len(calls), sum(len(c["candidates"]) for c in calls)


def record_search_beams(tag, graph, cfg, params, weights):
    """Trace a search too large to store its candidates (C3 at SURVEY §8(d)'s
    beam 32 x 5 passes): per `_cut` call the candidate count, the returned
    beam and costs and the memo size; plus the final beam and the wall time."""
    import time
    calls = []
    orig_cut = gsearch._cut

    def traced(candidates, evaluator, graph_, config, pass_index, memo, phase_seed, validate):
        beam, reports = orig_cut(candidates, evaluator, graph_, config, pass_index, memo,
                                 phase_seed, validate)
        calls.append({"pass_index": pass_index, "phase_seed": phase_seed, "n_candidates": len(candidates),
                      "beam": [schedule_dump(s) for s in beam], "beam_costs": [s.cost for s in beam],
                      "memo_size": len(memo.flagged), "n_reports": len(reports)})
        return beam, reports

    gsearch._cut = traced
    t = time.perf_counter()
    try:
        final = gsearch.schedule_with_freezing(graph, params, cfg, CostEvaluator(weights, params))
    finally:
        gsearch._cut = orig_cut
    wall = time.perf_counter() - t
    out = {"pipeline": graph_to_text(graph), "config": {
        "beam_size": cfg.beam_size, "num_passes": cfg.num_passes, "seed": cfg.seed,
        "freeze_enabled": cfg.freeze_enabled}, "calls": calls,
        "final": [schedule_dump(s) for s in final], "final_costs": [s.cost for s in final],
        "reference_wall_s": wall, "reference_cores": 1}
    with gzip.open(os.path.join(HERE, f"search_{tag}.json.gz"), "wt") as fh:
        json.dump(out, fh)
    return len(calls), sum(c["n_candidates"] for c in calls), wall


def main():
    params = MachineParams()
    if "--c3-full" in sys.argv:   # C3 at beam 32 x 5 passes (beams only; candidates regenerate on the GPU)
        print(record_search_beams("local_laplacian_b32p5", authored("local_laplacian"),
                                  SearchConfig(beam_size=32, num_passes=5, seed=0, freeze_enabled=True),
                                  params, init_weights(seed=0)), flush=True)
        return
    w0 = init_weights(seed=0)
    save_weights(w0, os.path.join(HERE, "weights_seed0.txt"))
    w1 = init_weights(seed=3, embed_dim=16, hidden_dim=48)
    save_weights(w1, os.path.join(HERE, "weights_small.txt"))
    if "--c3" in sys.argv:   # C3: full search with the freeze pre-pass on a ~100-func pipeline
        for tag in [a for a in sys.argv[1:] if not a.startswith("-")] or ["camera_pipe"]:
            print("s", tag, record_search(f"{tag}_freeze", authored(tag),
                                          SearchConfig(beam_size=2, num_passes=1, seed=0, freeze_enabled=True),
                                          params, w0, freeze=True), flush=True)
        return
    only = [a for a in sys.argv[1:] if not a.startswith("-")]
    for name, (graph, n, th) in graphs().items():
        if only and name not in only:
            continue
        print(name, record_candidates(name, graph, n, th, params, w0), flush=True)
    if only:
        return
    small = TilingConfig(serial_powers=(1, 2), odd_serial=(), innermost_thread=(16, 32),
                         outer_thread=(1, 4), unroll_budget=64)
    print("s chain2", record_search("chain2", parse_pipeline(CHAIN2_SRC, "chain2"),
                                    SearchConfig(beam_size=8, num_passes=2, seed=0,
                                                 thresholds=OPEN_THRESHOLDS), params, w0))
    print("s diamond", record_search("diamond", parse_pipeline(DIAMOND_SRC, "diamond"),
                                     SearchConfig(beam_size=6, num_passes=3, seed=5,
                                                  thresholds=OPEN_THRESHOLDS), params, w0))
    print("s diamond_T", record_search("diamond_T", parse_pipeline(DIAMOND_SRC, "diamond"),
                                       SearchConfig(beam_size=6, num_passes=2, seed=2,
                                                    explore_temperature=0.5,
                                                    thresholds=OPEN_THRESHOLDS), params, w0))
    print("s stencil", record_search("stencil_chain", builtin_pipeline("stencil_chain"),
                                     SearchConfig(beam_size=8, num_passes=2, seed=0), params, w0))
    print("s chain16f", record_search("chain16_freeze",
                                      parse_pipeline(make_chain_src(16, extent=32), "chain16"),
                                      SearchConfig(beam_size=4, num_passes=2, seed=0, tiling=small,
                                                   thresholds=OPEN_THRESHOLDS, freeze_enabled=True),
                                      params, w0, freeze=True))
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        np.show_config()
    with open(os.path.join(HERE, "provenance.json"), "w") as fh:
        json.dump({"numpy": np.__version__, "python": sys.version,
                   "reference": REF, "np_show_config": buf.getvalue()}, fh, indent=1)


if __name__ == "__main__":
    main()
