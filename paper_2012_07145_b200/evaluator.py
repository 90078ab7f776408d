"""Drop-in surface for the reference search (`gpusched`).

* `GpuCostEvaluator` — subclass of `gpusched.search.CostEvaluator`
  (search.py:90-124; the search type-checks with isinstance at
  search.py:302-303, 331-332, 351-352) whose `stage_basis` / `cost` run the
  sm_100a path.  When `gpusched` is not importable it derives from a local
  mirror with the same surface, so this package also stands alone.
* `gpu_cut` — same signature and results as `gpusched.search._cut`
  (search.py:168-201); `install()` swaps it into the module global the
  search resolves at call time (search.py:254), so the unchanged search,
  freeze pre-pass and driver batch whole phases onto the GPU.
"""

from __future__ import annotations

import contextlib

import numpy as np
import torch

from . import ops  # noqa: F401  (registers torch.ops.gsched)
from .cut import beam_cut
from .engine import Scorer
from .params import DEFAULT_THRESHOLDS

try:  # the reference is the user's own installation; optional here
    from gpusched.search import CostEvaluator as _Base  # type: ignore
    from gpusched.options import PruneReport as _PruneReport  # type: ignore
    from gpusched.machine import OracleResult as _OracleResult  # type: ignore
    HAVE_REFERENCE = True
except Exception:  # pragma: no cover - standalone use
    HAVE_REFERENCE = False

    class _OracleResult:  # mirror of machine.py:71-82
        def __init__(self, runtime, spilled_registers, spill_bytes):
            if runtime <= 0:
                raise ValueError("oracle runtime must be positive")
            if (spill_bytes > 0) != spilled_registers:
                raise ValueError("spill_bytes > 0 iff spilled_registers")
            self.runtime, self.spilled_registers, self.spill_bytes = runtime, spilled_registers, spill_bytes

    class _Base:  # mirror of search.py:90-101
        def __init__(self, weights, params):
            self.weights = weights
            self.params = params
            self._basis_cache = {}

    class _PruneReport:  # mirror of options.py:44-57
        REASONS = ("excessive_recompute", "idle_sms", "poor_warp_utilization",
                   "serial_too_large", "thread_alloc_dynamic_or_large", "hardware_limit")

        def __init__(self, reason, detail):
            if reason not in self.REASONS:
                raise ValueError(f"unknown prune reason {reason!r}")
            self.reason, self.detail = reason, detail


_SCORERS: dict = {}
_SHARDING = {"on": False, "group": None}


def configure_sharding(enable: bool = True, group=None):
    """Shard every phase cut's buckets across the ranks of `group` (default:
    the initialised torch.distributed world; one process per GPU, NCCL), as
    SURVEY §8(e) splits a beam step.  Every rank runs the same search; each
    featurizes and costs only its buckets' candidates, and the ranks agree on
    the beam through the top-k / memo-window exchange (exchange.py)."""
    _SHARDING["on"], _SHARDING["group"] = enable, group


def scorer_for(graph, params, thresholds, weights) -> Scorer:
    """One device pipeline per (graph, machine, thresholds); weights are
    re-uploaded whenever the weights object changes (driver.py:110, 219)."""
    key = (id(graph), params, thresholds)
    sc = _SCORERS.get(key)
    if sc is None or sc.packed.graph is not graph:
        sc = Scorer(graph, params, thresholds)
        _SCORERS[key] = sc
    if weights is not None:
        sc.set_weights(weights)
    return sc


def simulate_runtime(state, graph, params):
    """Drop-in for the reference machine oracle `simulate_runtime`
    (machine.py:108-167; the driver's `oracle=` hook, driver.py:120, 158,
    183): K1 + K6 on the B200.  Returns an OracleResult and raises
    ValueError in the two cases the reference raises for."""
    key = (id(graph), params, "oracle")
    sc = _SCORERS.get(key)
    if sc is None or sc.packed.graph is not graph:
        sc = Scorer(graph, params, DEFAULT_THRESHOLDS)
        _SCORERS[key] = sc
    rt, sp, st = sc.simulate(sc.upload([state]), params)
    sc.check()
    status = int(st[0].item())
    if status == 2:
        raise ValueError("oracle requires a fully scheduled state")
    if status == 1:
        raise ValueError("hardware limit violation")
    spill = int(sp[0].item())
    return _OracleResult(runtime=float(rt[0].item()), spilled_registers=spill > 0, spill_bytes=spill)


class GpuCostEvaluator(_Base):
    """`CostEvaluator` whose featurization and costing run on the B200."""

    def __init__(self, weights, params, thresholds=None):
        _Base.__init__(self, weights, params)
        self.thresholds = thresholds or DEFAULT_THRESHOLDS
        self._cost_cache = {}    # (id(graph), decisions) -> (weights key, total, per-stage dict)
        self._last_beam = None   # (id(graph), states) of the last gpu_cut

    def _batch_costs(self, states, graph):
        """K1 + K2 (with the basis) for several states in one launch each;
        fills the cost and basis caches (search.py:103-124 semantics)."""
        sc = scorer_for(graph, self.params, self.thresholds, self.weights)
        dec = sc.upload(states)
        h = sc.handle.value
        feats, row_key, n_rows, verdict, row_src = torch.ops.gsched.featurize(h, dec, sc.R, 1)
        total, rows, gh = torch.ops.gsched.cost(h, feats, row_key, n_rows, None, True)
        sc.check()
        f_all = feats.cpu().numpy()
        keys_all, nr = row_key.cpu().numpy(), n_rows.cpu().numpy()
        tot, rc, g = total.cpu().numpy(), rows.cpu().numpy(), gh.cpu().numpy()
        algo = sc.packed.algo
        for i, st in enumerate(states):
            n = int(nr[i])
            keys = sc.packed.row_keys(keys_all[i, :n])
            ck = (id(graph), st.decisions)
            self._cost_cache[ck] = (sc._weights_key, float(tot[i]), {k: float(c) for k, c in zip(keys, rc[i, :n])})
            if ck not in self._basis_cache:
                self._basis_cache[ck] = [(k, algo[sc.packed.stage_index[k]].copy(), f_all[i, r].copy(),
                                          g[i, r, :30].copy(), float(g[i, r, 30])) for r, k in enumerate(keys)]

    def _run(self, state, graph):
        # through the registered custom ops (ops.py): K1 then K2 with the basis
        sc = scorer_for(graph, self.params, self.thresholds, self.weights)
        dec = sc.upload([state])
        h = sc.handle.value
        feats, row_key, n_rows, verdict, row_src = torch.ops.gsched.featurize(h, dec, sc.R, 1)
        total, rows, gh = torch.ops.gsched.cost(h, feats, row_key, n_rows, None, True)
        sc.check()
        f = {"feats": feats, "row_key": row_key, "n_rows": n_rows, "verdict": verdict, "row_src": row_src}
        n = int(n_rows[0].item())
        keys = sc.packed.row_keys(row_key[0, :n].cpu().numpy())
        return sc, f, n, keys, float(total[0].item()), rows[0, :n].cpu().numpy(), gh[0, :n].cpu().numpy()

    def _fill_cache(self, sc, f, n, keys, gh, state, graph):
        key = (id(graph), state.decisions)
        if key in self._basis_cache:
            return self._basis_cache[key]
        feats = f["feats"][0, :n].cpu().numpy()
        algo = sc.packed.algo
        hit = []
        for r, k in enumerate(keys):
            xa = algo[sc.packed.stage_index[k]].copy()
            hit.append((k, xa, feats[r].copy(), gh[r, :30].copy(), float(gh[r, 30])))
        self._basis_cache[key] = hit
        return hit

    def stage_basis(self, state, graph):
        key = (id(graph), state.decisions)
        hit = self._basis_cache.get(key)
        if hit is None:
            sc, f, n, keys, _t, _r, gh = self._run(state, graph)
            hit = self._fill_cache(sc, f, n, keys, gh, state, graph)
        return hit

    def cost(self, state, graph):
        # The search re-costs its final beam one state at a time
        # (search.py:312-317, and the freeze pre-pass's best, 335): the first
        # such call costs the whole last beam in one batch, the rest are hits.
        ck = (id(graph), state.decisions)
        wk = scorer_for(graph, self.params, self.thresholds, self.weights)._weights_key
        hit = self._cost_cache.get(ck)
        if hit is None and self._last_beam is not None and self._last_beam[0] == id(graph):
            beam = self._last_beam[1]
            if any(s.decisions == state.decisions for s in beam):
                self._batch_costs(beam, graph)
                self._last_beam = None
                hit = self._cost_cache.get(ck)
        if hit is not None and hit[0] == wk:
            return hit[1], dict(hit[2])
        sc, f, n, keys, total, rows, gh = self._run(state, graph)
        self._fill_cache(sc, f, n, keys, gh, state, graph)
        per = {k: float(c) for k, c in zip(keys, rows)}
        self._cost_cache[ck] = (sc._weights_key, total, per)
        return total, dict(per)

    def cost_batch(self, states, graph):
        """Totals (np.float64[N]) and prune verdicts for a list of states."""
        sc = scorer_for(graph, self.params, self.thresholds, self.weights)
        dec = sc.upload(states)
        h = sc.handle.value
        feats, row_key, n_rows, verdict, row_src = torch.ops.gsched.featurize(h, dec, sc.R, 1)
        total, _, _ = torch.ops.gsched.cost(h, feats, row_key, n_rows, row_src, False)
        sc.check()
        return total.cpu().numpy(), verdict.cpu().numpy()


class CandidateGroup:
    """Every phase-1 (or phase-2) candidate of one beam state, left
    unexpanded: `gpu_cut` generates them on the device
    (gs_expand_phase1 / gs_expand_step) and builds host states only for the
    beam it returns.  Produced by `phase1_candidates` / `phase2_candidates`,
    the drop-ins for search.py:204-220 / 223-235 that `install(expand=True)`
    puts into the search module."""

    __slots__ = ("parent", "func", "phase", "config")

    def __init__(self, parent, func, phase, config):
        self.parent, self.func, self.phase, self.config = parent, func, phase, config


def phase1_candidates(state, func, graph, config):
    """Drop-in for `gpusched.search._phase1_candidates` (search.py:204-220)."""
    return [CandidateGroup(state, func, 1, config)]


def phase2_candidates(state, func, graph, config):
    """Drop-in for `gpusched.search._phase2_candidates` (search.py:223-235)."""
    return [CandidateGroup(state, func, 2, config)]


def _expand_items(sc, candidates):
    """Device records of a phase's candidate list, in the list's order, where
    items are states or CandidateGroups.  Returns (records [N, S*16], where:
    per item (kind, a, b) — ('state', state, row) or ('group', group, first
    row, count))."""
    groups = [c for c in candidates if isinstance(c, CandidateGroup)]
    plain = [c for c in candidates if not isinstance(c, CandidateGroup)]
    parts, counts = [], []
    if groups:
        g0 = groups[0]
        if any(g.phase != g0.phase or g.func != g0.func for g in groups):
            raise ValueError("one phase expands one func")
        par = sc.upload([g.parent for g in groups])
        if g0.phase == 1:
            restrict = g0.config.restrict_placements
            recs, _, offs = sc.expand_phase1(par, g0.func, restrict=restrict, menus=g0.config.tiling)
        else:
            steps = []
            for g in groups:
                pos = [i for i, (f, _d) in enumerate(g.parent.decisions) if f == g0.func]
                steps.append(pos[0])
            st = torch.tensor(steps, dtype=torch.int32, device=sc.device)
            recs, _, offs = sc.expand_step(par, st, menus=g0.config.tiling)
        sc.check()
        counts = np.diff(offs.cpu().numpy()).tolist()
        parts.append(recs)
    n_exp = sum(counts)
    if plain:
        parts.append(sc.upload(plain))
    allr = torch.cat(parts) if len(parts) > 1 else parts[0]
    order, where = [], []
    gi = pi = 0
    first = 0
    starts = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64) if counts else [0]
    for c in candidates:
        if isinstance(c, CandidateGroup):
            k = counts[gi]
            start = int(starts[gi])
            order.extend(range(start, start + k))
            where.append(("group", c, first, k))
            first += k
            gi += 1
        else:
            order.append(n_exp + pi)
            where.append(("state", c, first, 1))
            first += 1
            pi += 1
    idx = torch.tensor(order, dtype=torch.int64, device=sc.device)
    dec = allr.index_select(0, idx) if order != list(range(len(order))) else allr
    return dec, where


def _materialize(sc, rows, where, idx):
    """Host states of candidates `idx` (their device records already read
    back as `rows`, one per index): the item itself, or — for a group — the
    reference's own apply_decision of the record's decision on the parent
    (what the reference's _phase1/2_candidates would have built)."""
    import bisect
    from .descriptor import DECISION_DTYPE, KIND_NAME
    firsts = [w[2] for w in where]
    out = []
    for i, raw in zip(idx, rows):
        k = bisect.bisect_right(firsts, i) - 1
        kind, item, first, _ = where[k]
        if kind == "state":
            out.append(item)
            continue
        from gpusched.loopnest import Decision, apply_decision  # type: ignore
        rec = raw.view(DECISION_DTYPE)
        fi = sc.packed.index[item.func]
        r = rec[rec["func"] == fi][0]
        nd = sc.packed.graph.func(item.func).ndim
        d = Decision(KIND_NAME[int(r["kind"])],
                     consumer=None if r["consumer"] == 0xFFFF else sc.packed.names[int(r["consumer"])],
                     serial=tuple(int(x) for x in r["serial"][:nd]) if r["flags"] & 1 else None,
                     thread=tuple(int(x) for x in r["thread"][:nd]) if r["flags"] & 2 else None)
        out.append(apply_decision(item.parent, item.func, d))
    return out


def gpu_cut(candidates, evaluator, graph, config, pass_index, memo, phase_seed, validate):
    """Drop-in for `gpusched.search._cut` (search.py:168-201).

    `validate` is the reference prune closure over `config.thresholds`
    (search.py:246-247); the same rules run on the GPU with those thresholds.
    Candidates may be states or CandidateGroups (install(expand=True)): a
    group's candidates are generated on the device and only the returned
    beam becomes host states.
    """
    if not candidates:
        return [], []
    weights = getattr(evaluator, "weights", None)
    sc = scorer_for(graph, evaluator.params, config.thresholds, weights)
    lazy = any(isinstance(c, CandidateGroup) for c in candidates)
    if lazy:
        dec, where = _expand_items(sc, candidates)
    else:
        dec, where = sc.upload(candidates), None
    flagged = [h for d, h in memo.flagged if d == pass_index]
    world, rank, group = 1, 0, None
    if _SHARDING["on"]:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            group = _SHARDING["group"]
            world, rank = dist.get_world_size(group), dist.get_rank(group)
    res = beam_cut(sc, dec, pass_index, phase_seed, flagged, config.beam_size,
                   config.penalty_factor, config.explore_temperature, config.num_passes,
                   sampling=config.sampling, world=world, rank=rank, group=group)
    reports = [_PruneReport(reason, f"GPU prune verdict for candidate {i} of this phase")
               for i, reason in res.rejects]
    for depth, h in res.memo_new:
        memo.record(depth, h)
    if lazy:
        bi = torch.tensor(res.beam, dtype=torch.int64, device=dec.device)
        rows = dec.index_select(0, bi).cpu().numpy() if res.beam else []   # one read-back for the beam
        states = _materialize(sc, rows, where, res.beam)
        beam = [st.with_cost(c) for st, c in zip(states, res.costs)]
    else:
        beam = [candidates[i].with_cost(c) for i, c in zip(res.beam, res.costs)]
    if isinstance(evaluator, GpuCostEvaluator):
        evaluator._last_beam = (id(graph), beam)   # batched final re-cost (GpuCostEvaluator.cost)
    return beam, reports


def install(search_module=None, expand=False):
    """Route the reference search's phase cuts through the GPU; with
    expand=True also its candidate generation (`_phase1_candidates`,
    `_phase2_candidates` -> device expansion inside gpu_cut).  Returns the
    previous functions so callers can restore them."""
    if search_module is None:
        import gpusched.search as search_module  # type: ignore
    prev = (search_module._cut, search_module._phase1_candidates, search_module._phase2_candidates)
    search_module._cut = gpu_cut
    if expand:
        search_module._phase1_candidates = phase1_candidates
        search_module._phase2_candidates = phase2_candidates
    return prev


@contextlib.contextmanager
def installed(search_module=None, expand=False):
    if search_module is None:
        import gpusched.search as search_module  # type: ignore
    prev = install(search_module, expand=expand)
    try:
        yield
    finally:
        search_module._cut, search_module._phase1_candidates, search_module._phase2_candidates = prev


def as_numpy(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()
