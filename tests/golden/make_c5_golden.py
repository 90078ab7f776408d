"""C5-scale parity fixtures, written by the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_c5_golden.py [--parents P] [--sample K] [--procs J]

The workload is exactly the bench step (bench.py): the
committed parents `bench_data/c5_parents_seed0.npz` of
`make_chain_src(100, extent=1024)`, each expanded by the reference
`_phase2_candidates` (search.py:223-235) to every tiling of its step root —
1,000,080 candidates at the full 4,167 parents.

Two fixtures (`tests/golden/c5_step.npz`, `c5_step.json.gz`):

* sample — K candidates evenly strided over the step: per-row features
  (sha256 of the fp64 [R, 56] block, plus the full block for every 16th),
  row costs, totals, row keys, prune verdicts and structural hashes at
  depths 0-5, from `CostEvaluator.stage_basis/.cost`, `prune` and
  `structural_hash`.
* cut — the reference `_cut` (search.py:168-201) over the WHOLE step at
  beam 32, pass 3, phase seed = 0*10007 + 3*101 + 57 (bench.py), in three
  memo/temperature variants: (empty memo, T = 0) = the bench config;
  (a seeded memo, T = 0) to exercise the bad-hash penalty at scale; (the
  same memo, T = 0.5) for the Gumbel cut.  Recorded: representatives and
  prune rejects in draw order, every representative's cost, the returned
  beam and its costs, and the memo after the call.

The reference `_cut` runs in this process, unmodified.  Two things are
computed ahead of it in a fork pool and handed to it through its own
parameters, because the whole step would take hours on one core: `validate`
(a closure the reference search passes in, search.py:246-247) answers from
a table of reference `prune` results, and the evaluator is a
`CostEvaluator` subclass whose `cost` answers from a table of reference
`CostEvaluator.cost` totals.  Both fall back to the reference functions on
a miss, so a table that missed a member cannot change the result.
"""

from __future__ import annotations

import argparse
import gzip
import hashlib
import json
import math
import multiprocessing as mp
import os
import sys
import time
import zlib

import numpy as np

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src"), os.path.join(REF, "tests")]
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

import gpusched  # noqa: E402
import gpusched.search as gsearch  # noqa: E402
from gpusched.costmodel import init_weights  # noqa: E402
from gpusched.loopnest import Decision, apply_decision, initial_state  # noqa: E402
from gpusched.machine import MachineParams  # noqa: E402
from gpusched.options import DEFAULT_THRESHOLDS, prune  # noqa: E402
from gpusched.search import BadHashMemo, CostEvaluator, SearchConfig  # noqa: E402

from conftest import make_chain_src  # noqa: E402

PASS_INDEX = 3
PHASE_SEED = 0 * 10007 + PASS_INDEX * 101 + 57
KINDS = ("compute_root", "fuse_at_block", "fuse_at_thread", "inline")
REASONS = ("excessive_recompute", "idle_sms", "poor_warp_utilization", "serial_too_large",
           "thread_alloc_dynamic_or_large", "hardware_limit")

_G = {}


def parent_states(graph, parents, steps):
    """Reference LoopNestStates of the committed parents (records -> apply_decision)."""
    out = []
    for rec, st in zip(parents, steps):
        s = initial_state(graph)
        for r in rec:
            if r["func"] == 0xFFFF:
                break
            f = _G["fnames"][int(r["func"])]
            nd = graph.func(f).ndim
            kind = KINDS[int(r["kind"])]
            cons = None if r["consumer"] == 0xFFFF else _G["fnames"][int(r["consumer"])]
            ser = tuple(int(x) for x in r["serial"][:nd]) if r["flags"] & 1 else None
            thr = tuple(int(x) for x in r["thread"][:nd]) if r["flags"] & 2 else None
            if kind == "compute_root" and ser is not None:
                s = apply_decision(s, f, Decision("compute_root"))
            s = apply_decision(s, f, Decision(kind, cons, ser, thr))
        out.append((s, _G["fnames"][int(rec[st]["func"])]))
    return out


def children(p):
    """Reference phase-2 children of parent p (cached per worker)."""
    c = _G.setdefault("kids", {})
    if p not in c:
        if len(c) > 64:
            c.clear()
        s, f = _G["parents"][p]
        c[p] = gsearch._phase2_candidates(s, f, _G["graph"], _G["cfg"])
    return c[p]


def _sample_one(i):
    p, t = divmod(int(i), _G["per"])
    st = children(p)[t]
    g, prm, w = _G["graph"], _G["params"], _G["w"]
    ev = CostEvaluator(w, prm)
    basis = ev.stage_basis(st, g)
    total, per = ev.cost(st, g)
    feats = np.array([xs for _, _, xs, _, _ in basis], dtype=np.float64)
    rows = [k for k, *_ in basis]
    rc = np.array([per[k] for k in rows], dtype=np.float64)
    r = prune(st, g, prm, DEFAULT_THRESHOLDS)
    hashes = [st.structural_hash(d) for d in range(6)]
    return int(i), feats, rc, float(total), [[k[0], k[1]] for k in rows], (r.reason if r else None), hashes


def _walk_bucket(job):
    """The reference's per-bucket draw (search.py:151-164) with reference
    prune; returns the drawn members' reports.  Only a lookup table: the
    reference _cut below makes the actual draws."""
    h, members = job
    quota = max(1, int(math.floor(math.log2(len(members)))))
    stream = np.random.default_rng((PHASE_SEED, h))
    out = []
    taken = 0
    for j in stream.permutation(len(members)):
        gi = members[int(j)]
        p, t = divmod(gi, _G["per"])
        r = prune(children(p)[t], _G["graph"], _G["params"], DEFAULT_THRESHOLDS)
        out.append((gi, None if r is None else (r.reason, r.detail)))
        if r is None:
            taken += 1
            if taken == quota:
                break
    return out


def _cost_many(idx):
    out = []
    for gi in idx:
        p, t = divmod(gi, _G["per"])
        total, _ = CostEvaluator(_G["w"], _G["params"]).cost(children(p)[t], _G["graph"])
        out.append((gi, total))
    return out


class TableEvaluator(CostEvaluator):
    """Reference evaluator whose cost() first consults reference totals
    computed ahead in the pool (keyed by the decision tuple)."""

    def __init__(self, weights, params, table):
        super().__init__(weights, params)
        self.table, self.misses = table, 0

    def cost(self, state, graph):
        t = self.table.get(state.decisions)
        if t is None:
            self.misses += 1
            return super().cost(state, graph)
        return t, {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parents", type=int, default=4167)
    ap.add_argument("--sample", type=int, default=1024)
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default="c5_step")
    args = ap.parse_args()
    from gpusched.pipeline import parse_pipeline
    graph = parse_pipeline(make_chain_src(100, extent=1024), "chain100")
    z = np.load(os.path.join(ROOT, "bench_data", "c5_parents_seed0.npz"))
    from paper_2012_07145_b200.descriptor import DECISION_DTYPE
    par = np.ascontiguousarray(z["parents"]).view(DECISION_DTYPE).reshape(len(z["parents"]), -1)
    par, steps = par[:args.parents], z["steps"][:args.parents]
    # func index -> name: the packed records number funcs in graph order
    from paper_2012_07145_b200.pipeline import parse_pipeline as our_parse
    ours = our_parse(make_chain_src(100, extent=1024), "chain100")
    _G["fnames"] = [f.name for f in ours.funcs]
    cfg = SearchConfig(beam_size=32, num_passes=5, seed=0)
    _G.update(graph=graph, params=MachineParams(), w=init_weights(0), cfg=cfg)
    t0 = time.time()
    _G["parents"] = parent_states(graph, par, steps)
    k0 = children(0)
    _G["per"] = per = len(k0)
    assert per == 240, per
    N = per * len(par)
    print(f"{len(par)} parents, {N} candidates ({time.time() - t0:.1f}s)", flush=True)

    # --- strided sample ------------------------------------------------------
    ctx = mp.get_context("fork")
    sidx = np.linspace(0, N - 1, args.sample).astype(np.int64)
    t0 = time.time()
    with ctx.Pool(args.procs) as pool:
        res = pool.map(_sample_one, sidx.tolist(), chunksize=4)
    print(f"sample of {len(res)} in {time.time() - t0:.1f}s", flush=True)
    res.sort(key=lambda r: r[0])
    offs = np.cumsum([0] + [len(r[2]) for r in res])
    full_every = 16
    meta = {"pipeline": "make_chain_src(100, extent=1024)", "n_candidates": N,
            "parents": len(par), "per_parent": per, "sample_index": sidx.tolist(),
            "rows": [r[4] for r in res], "prune": [r[5] for r in res],
            "hashes": [[str(h) for h in r[6]] for r in res],
            "feat_sha256": [hashlib.sha256(np.ascontiguousarray(r[1]).tobytes()).hexdigest() for r in res],
            "full_features_every": full_every}
    full = np.concatenate([r[1] for r in res[::full_every]])
    full_offs = np.cumsum([0] + [len(r[1]) for r in res[::full_every]])

    # --- buckets at the pass depth (siblings share every hash: extents are
    # never hashed, loopnest.py:158-164; checked on the sample above) --------
    for r in res:
        p = r[0] // per
        assert [str(h) for h in r[6]] == [str(children(p)[0].structural_hash(d)) for d in range(6)]
    phash = [children(p)[0].structural_hash(PASS_INDEX) for p in range(len(par))]
    buckets = {}
    for p, h in enumerate(phash):
        buckets.setdefault(h, []).extend(range(p * per, (p + 1) * per))
    print(f"{len(buckets)} buckets", flush=True)

    t0 = time.time()
    jobs = [(h, buckets[h]) for h in sorted(buckets)]
    with ctx.Pool(args.procs) as pool:
        walks = pool.map(_walk_bucket, jobs, chunksize=8)
    verdict_table = {}
    valid = []
    for w in walks:
        for gi, rep in w:
            verdict_table[gi] = rep
            if rep is None:
                valid.append(gi)
    print(f"walk: {len(verdict_table)} drawn, {len(valid)} valid ({time.time() - t0:.1f}s)", flush=True)
    t0 = time.time()
    chunks = [valid[i:i + 64] for i in range(0, len(valid), 64)]
    with ctx.Pool(args.procs) as pool:
        costed = pool.map(_cost_many, chunks, chunksize=1)
    cost_of = {gi: c for ch in costed for gi, c in ch}
    print(f"costs of {len(cost_of)} reps ({time.time() - t0:.1f}s)", flush=True)

    # --- the reference _cut over the whole step ------------------------------
    t0 = time.time()
    _G.pop("kids", None)
    allc = []
    for s, f in _G["parents"]:
        allc.extend(gsearch._phase2_candidates(s, f, graph, cfg))
    assert len(allc) == N
    index_of = {c.decisions: i for i, c in enumerate(allc)}
    assert len(index_of) == N, "duplicate candidates in the step"
    print(f"built {N} states ({time.time() - t0:.1f}s)", flush=True)
    from gpusched.options import PruneReport
    vt = {allc[gi].decisions: rep for gi, rep in verdict_table.items()}
    misses = [0]

    def validate(c):
        if c.decisions in vt:
            rep = vt[c.decisions]
            return None if rep is None else PruneReport(*rep)
        misses[0] += 1
        return prune(c, graph, _G["params"], cfg.thresholds)

    table = {allc[gi].decisions: c for gi, c in cost_of.items()}
    reps, reports = gsearch._select_representatives(allc, cfg, PASS_INDEX, PHASE_SEED, validate)
    rep_idx = np.array([index_of[s.decisions] for s in reps], dtype=np.int64)
    rep_cost = np.array([table[s.decisions] for s in reps], dtype=np.float64)
    # memo seeds for variants 2/3: every 3rd distinct pass-depth bucket hash
    # (the penalty looks up (pass_index, hash), search.py:84) plus entries at
    # other depths, which must not penalize
    seed_memo = set()
    for j, h in enumerate(sorted(buckets)):
        if j % 3 == 0:
            seed_memo.add((PASS_INDEX, h))
        if j % 5 == 1:
            seed_memo.add((2, h))
    variants = [("bench", set(), 0.0), ("memo", seed_memo, 0.0), ("memo_T05", seed_memo, 0.5)]
    cuts = {}
    for tag, mset, T in variants:
        c2 = SearchConfig(beam_size=32, num_passes=5, seed=0, explore_temperature=T)
        memo = BadHashMemo(flagged=set(mset))
        ev = TableEvaluator(_G["w"], _G["params"], table)
        t1 = time.time()
        beam, reps2 = gsearch._cut(allc, ev, graph, c2, PASS_INDEX, memo, PHASE_SEED, validate)
        el = time.time() - t1
        assert len(reps2) == len(reports)
        cuts[tag] = {"temperature": T, "memo_before": sorted([[d, str(h)] for d, h in mset]),
                     "beam": [index_of[s.decisions] for s in beam], "beam_costs": [s.cost for s in beam],
                     "memo_after": sorted([[d, str(h)] for d, h in memo.flagged]),
                     "evaluator_misses": ev.misses, "cut_wall_s": el}
        print(tag, "beam", cuts[tag]["beam"][:8], "memo", len(memo.flagged), f"{el:.1f}s", flush=True)
    meta["cut"] = {"pass_index": PASS_INDEX, "phase_seed": PHASE_SEED, "beam_size": 32, "num_passes": 5,
                   "penalty_factor": 2.0, "n_reps": int(len(reps)), "n_rejects": int(len(reports)),
                   "reject_reasons": [r.reason for r in reports], "validate_misses": misses[0],
                   "variants": cuts}
    # rejects in draw order: the reference reports follow the walk order
    draw_rej = []
    for w in walks:
        draw_rej.extend(gi for gi, rep in w if rep is not None)
    assert len(draw_rej) == len(reports)
    assert [verdict_table[gi][0] for gi in draw_rej] == [r.reason for r in reports]
    np.savez_compressed(os.path.join(HERE, f"{args.out}.npz"),
                        sample_index=sidx, row_offsets=offs, rowcost=np.concatenate([r[2] for r in res]),
                        total=np.array([r[3] for r in res]), full_feats=full, full_offsets=full_offs,
                        rep_idx=rep_idx, rep_cost=rep_cost, rej_idx=np.array(draw_rej, dtype=np.int64))
    with gzip.open(os.path.join(HERE, f"{args.out}.json.gz"), "wt") as fh:
        json.dump(meta, fh)
    print("wrote", args.out, flush=True)


if __name__ == "__main__":
    main()
