"""Synthetic candidate generation (SURVEY §8(d) beam-step generator).

Mirrors the reference menus (`enumerate_compute_locations`,
`enumerate_serial_tilings`, `enumerate_thread_tilings`,
options.py:103-183) and the random-schedule procedure of the reference
tests (`_random_schedule`, tests/test_acceptance.py:136-160), with array
bookkeeping instead of persistent state objects so a million candidates
can be produced in seconds.  Output is the packed 16-byte decision record
array consumed by the C ABI.

Beam-step workload (config C5): P random parent states at a phase-2 step —
every func placed, roots before the step root tiled, the step root and the
roots after it untiled — each expanded to all tilings of the step root.
"""

from __future__ import annotations

import math

import numpy as np

from .descriptor import DECISION_DTYPE, KIND_CODE
from .schedule import Decision

CHEAP_INLINE_OPS = 8  # options.py:22


class Menus:
    serial_powers = (1, 2, 4, 8)
    odd_serial = (3, 5, 7)
    innermost_thread = (16, 32, 64)
    outer_thread = (1, 2, 4, 8, 16)
    unroll_budget = 64
    warp_size = 32


def serial_tilings(extents, m=Menus):
    """options.py:144-162."""
    per = []
    for e in extents:
        opts = sorted({s for s in m.serial_powers if s <= e})
        for o in m.odd_serial:
            if o <= e and e % o == 0 and (e // o) % m.warp_size == 0:
                opts.append(o)
        per.append(sorted(set(opts)) or [1])
    out = [()]
    for o in per:
        out = [v + (x,) for v in out for x in o]
    return [v for v in out if math.prod(v) <= m.unroll_budget]


def thread_tilings(extents, m=Menus):
    """options.py:165-183."""
    if not extents:
        return []
    inner = next((i for i, e in enumerate(extents) if e >= 16), 0)
    per = [sorted({min(t, e) for t in (m.innermost_thread if i == inner else m.outer_thread)})
           for i, e in enumerate(extents)]
    out = [()]
    for o in per:
        out = [v + (x,) for v in out for x in o]
    return out


def root_tilings(extents, m=Menus):
    """All (serial, thread) phase-2 tilings of a root func (search.py:223-235)."""
    out = []
    for s in serial_tilings(extents, m):
        post = tuple(-(-e // x) for e, x in zip(extents, s))
        for t in thread_tilings(post, m):
            out.append((s, t))
    return out


class GraphInfo:
    def __init__(self, graph, menus=Menus):
        self.graph = graph
        self.m = menus
        self.names = [f.name for f in graph.funcs]
        self.idx = {n: i for i, n in enumerate(self.names)}
        self.order = [self.idx[f] for f in reversed(graph.topo_order)
                      if not graph.func(f).is_external_input]
        self.consumers = {}
        self.pointwise = {}
        for f in graph.funcs:
            cons, found, pw = [], False, True
            for c in graph.funcs:
                if c.name == f.name:
                    continue
                hit = False
                for st in c.stages:
                    for a in st.accesses:
                        if a.producer == f.name:
                            hit = found = True
                            if not a.is_pointwise():
                                pw = False
                if hit:
                    cons.append(self.idx[c.name])
            self.consumers[self.idx[f.name]] = cons
            self.pointwise[self.idx[f.name]] = found and pw
        self.outputs = {self.idx[o] for o in graph.outputs}
        self.inline_ok = {}
        self.cheap = {}
        for f in graph.funcs:
            i = self.idx[f.name]
            self.inline_ok[i] = (i not in self.outputs and len(f.stages) == 1 and not any(
                a.producer == f.name for st in f.stages for a in st.accesses))
            self.cheap[i] = sum(sum(st.op_histogram.values()) for st in f.stages) <= CHEAP_INLINE_OPS
        self.extents = {self.idx[f.name]: f.extents for f in graph.funcs}
        self.n_stages = {self.idx[f.name]: len(f.stages) for f in graph.funcs}
        self._serial = {}
        self._roots = {}

    def serials(self, f):
        if f not in self._serial:
            self._serial[f] = serial_tilings(self.extents[f], self.m)
        return self._serial[f]

    def tilings(self, f):
        if f not in self._roots:
            self._roots[f] = root_tilings(self.extents[f], self.m)
        return self._roots[f]

    def random_placement(self, rng):
        """Phase 1 of `_random_schedule`: (func, kind, consumer, serial) in order."""
        kind, kern, eff = {}, {}, {}
        out = []
        for f in self.order:
            e = set()
            for c in self.consumers[f]:
                if kind.get(c) == 3:
                    e |= eff[c]
                else:
                    e.add(c)
            eff[f] = e
            if f in self.outputs:
                menu = [(0, None)]
            elif self.n_stages[f] == 1 and self.pointwise[f] and self.inline_ok[f]:
                menu = [(3, None)]
            else:
                menu = [(0, None)]
                for c in sorted(e, key=lambda i: self.names[i]):
                    if c not in kind or kind[c] == 3:
                        continue
                    menu.append((1, c)) if all(kern.get(o) == kern[c] for o in e) else None
                    if e == {c}:
                        menu.append((2, c))
                if self.cheap[f] and self.inline_ok[f]:
                    menu.append((3, None))
            k, c = menu[int(rng.integers(len(menu)))]
            serial = None
            if k == 1:
                ss = self.serials(f)
                serial = ss[int(rng.integers(len(ss)))]
            kind[f] = k
            kern[f] = f if k == 0 else (kern[c] if k in (1, 2) else None)
            out.append([f, k, c, serial, None])
        return out

    def random_full(self, rng):
        """`_random_schedule` (tests/test_acceptance.py:136-160)."""
        dec = self.random_placement(rng)
        for d in dec:
            if d[1] == 0:
                s, t = self._draw_tiling(rng, d[0])
                d[3], d[4] = s, t
        return dec

    def _draw_tiling(self, rng, f):
        ss = self.serials(f)
        s = ss[int(rng.integers(len(ss)))]
        post = tuple(-(-e // x) for e, x in zip(self.extents[f], s))
        ts = thread_tilings(post, self.m)
        return s, ts[int(rng.integers(len(ts)))]

    def random_step_parent(self, rng):
        """A parent at a phase-2 step: roots before the step root tiled."""
        dec = self.random_placement(rng)
        roots = [i for i, d in enumerate(dec) if d[1] == 0]
        step = roots[int(rng.integers(len(roots)))]
        for i in roots:
            if i < step:
                dec[i][3], dec[i][4] = self._draw_tiling(rng, dec[i][0])
        return dec, step

    def to_decisions(self, dec):
        kinds = {v: k for k, v in KIND_CODE.items()}
        return tuple((self.names[f], Decision(kinds[k], self.names[c] if c is not None else None,
                                              s, t)) for f, k, c, s, t in dec)

    def pack_rows(self, decs, S):
        out = np.zeros((len(decs), S), dtype=DECISION_DTYPE)
        out["func"] = 0xFFFF
        out["consumer"] = 0xFFFF
        for r, dec in enumerate(decs):
            for i, (f, k, c, s, t) in enumerate(dec):
                rec = out[r, i]
                rec["func"], rec["kind"] = f, k
                rec["consumer"] = 0xFFFF if c is None else c
                fl = 0
                if s is not None:
                    fl |= 1
                    rec["serial"][:len(s)] = s
                if t is not None:
                    fl |= 2
                    rec["thread"][:len(t)] = t
                rec["flags"] = fl
        return out


def _menu(info, f, kind, kern, eff):
    """`enumerate_compute_locations` for func f given the placements so far."""
    e = set()
    for c in info.consumers[f]:
        if kind.get(c) == 3:
            e |= eff[c]
        else:
            e.add(c)
    eff[f] = e
    if f in info.outputs:
        return [(0, None)]
    if info.n_stages[f] == 1 and info.pointwise[f] and info.inline_ok[f]:
        return [(3, None)]
    menu = [(0, None)]
    for c in sorted(e, key=lambda i: info.names[i]):
        if c not in kind or kind[c] == 3:
            continue
        if all(kern.get(o) == kern[c] for o in e):
            menu.append((1, c))
        if e == {c}:
            menu.append((2, c))
    if info.cheap[f] and info.inline_ok[f]:
        menu.append((3, None))
    return menu


def _set_record(arr, row, col, f, k, c, s, t):
    r = arr[row, col]
    r["func"], r["kind"] = f, k
    r["consumer"] = 0xFFFF if c is None else c
    fl = 0
    r["serial"][:] = 0
    r["thread"][:] = 0
    if s is not None:
        fl |= 1
        r["serial"][:len(s)] = s
    if t is not None:
        fl |= 2
        r["thread"][:len(t)] = t
    r["flags"] = fl
    arr[row, col] = r


def valid_step_parents(graph, prune, n_parents, seed=0, menus=Menus, tries=6):
    """Parents of a phase-2 beam step that survive pruning, built the way a
    beam search builds them: every placement (search.py:261-271) and every
    earlier root tiling (search.py:274-290) is drawn uniformly among the
    options whose partial state passes `prune` (a batched verdict function:
    packed records -> np.uint8 verdicts, 0 = valid).  Parent i draws from
    its own stream default_rng((seed, i)).  Returns (records [n, S], step
    decision index per parent)."""
    info = GraphInfo(graph, menus)
    S = len(info.order)
    P0 = int(n_parents * 1.25) + 16
    rngs = [np.random.default_rng((seed, i)) for i in range(P0)]
    cur = np.zeros((P0, S), dtype=DECISION_DTYPE)
    cur["func"] = 0xFFFF
    cur["consumer"] = 0xFFFF
    kinds = [dict() for _ in range(P0)]
    kerns = [dict() for _ in range(P0)]
    effs = [dict() for _ in range(P0)]
    bad = np.zeros(P0, dtype=bool)
    for j, f in enumerate(info.order):
        opts, owner = [], []
        for p in range(P0):
            for k, c in _menu(info, f, kinds[p], kerns[p], effs[p]):
                s = None
                if k == 1:
                    ss = info.serials(f)
                    s = ss[int(rngs[p].integers(len(ss)))]
                opts.append((k, c, s))
                owner.append(p)
        owner = np.array(owner)
        cand = cur[owner].copy()
        for i, (k, c, s) in enumerate(opts):
            _set_record(cand, i, j, f, k, c, s, None)
        ver = prune(cand)
        start = 0
        for p in range(P0):
            end = start
            while end < len(owner) and owner[end] == p:
                end += 1
            ok = [i for i in range(start, end) if ver[i] == 0]
            pick = ok if ok else list(range(start, end))
            if not ok:
                bad[p] = True
            i = pick[int(rngs[p].integers(len(pick)))]
            k, c, s = opts[i]
            cur[p, j] = cand[i, j]
            kinds[p][f] = k
            kerns[p][f] = f if k == 0 else (kerns[p][c] if k in (1, 2) else None)
            start = end
    # phase 2: tile the roots placed before each parent's step root
    steps = np.zeros(P0, dtype=np.int64)
    todo = []
    for p in range(P0):
        roots = [i for i in range(S) if cur[p, i]["kind"] == 0]
        steps[p] = roots[int(rngs[p].integers(len(roots)))]
        todo.append([i for i in roots if i < steps[p]])
    rounds = max(len(t) for t in todo) if todo else 0
    for r in range(rounds):
        ps = [p for p in range(P0) if r < len(todo[p]) and not bad[p]]
        if not ps:
            continue
        cand, own, props = [], [], []
        for p in ps:
            col = todo[p][r]
            f = int(cur[p, col]["func"])
            for _ in range(tries):
                s, t = info._draw_tiling(rngs[p], f)
                props.append((col, f, s, t))
                own.append(p)
        own = np.array(own)
        cand = cur[own].copy()
        for i, (col, f, s, t) in enumerate(props):
            _set_record(cand, i, col, f, 0, None, s, t)
        ver = prune(cand)
        for q, p in enumerate(ps):
            ok = [q * tries + x for x in range(tries) if ver[q * tries + x] == 0]
            if not ok:
                bad[p] = True
                continue
            i = ok[0]
            col = props[i][0]
            cur[p, col] = cand[i, col]
    final = prune(cur)
    good = np.nonzero((~bad) & (final == 0))[0][:n_parents]
    if len(good) < n_parents:
        raise RuntimeError(f"only {len(good)} valid parents of {P0} drawn")
    return cur[good], steps[good]


def expand_step(parents, steps, graph, menus=Menus):
    """Children of a beam step: every phase-2 tiling of each parent's step
    root (search.py:223-235).  Returns (records [N, S], parent of each)."""
    info = GraphInfo(graph, menus)
    tilings = [info.tilings(int(parents[p, steps[p]]["func"])) for p in range(len(parents))]
    counts = np.array([len(t) for t in tilings])
    out = np.repeat(parents, counts, axis=0)
    owner = np.repeat(np.arange(len(parents)), counts)
    pos = 0
    for p in range(len(parents)):
        st = int(steps[p])
        blk = out[pos:pos + counts[p], st]
        ser = np.array([s for s, _ in tilings[p]], dtype=np.uint8)
        thr = np.array([t for _, t in tilings[p]], dtype=np.uint8)
        nd = ser.shape[1]
        blk["serial"][:, :nd] = ser
        blk["thread"][:, :nd] = thr
        blk["flags"] = 3
        out[pos:pos + counts[p], st] = blk
        pos += counts[p]
    return out, owner


def beam_step(graph, n_parents, seed=0, S=None, menus=Menus):
    """Packed C5-style beam-step batch: n_parents x (all step-root tilings).

    Returns (records [N, S], parent index per candidate, info)."""
    info = GraphInfo(graph, menus)
    S = S or len(info.order)
    rng = np.random.default_rng(seed)
    parents, steps, tilings = [], [], []
    for _ in range(n_parents):
        d, st = info.random_step_parent(rng)
        parents.append(d)
        steps.append(st)
        tilings.append(info.tilings(d[st][0]))
    base = info.pack_rows(parents, S)
    counts = np.array([len(t) for t in tilings])
    out = np.repeat(base, counts, axis=0)
    owner = np.repeat(np.arange(n_parents), counts)
    pos = 0
    for p in range(n_parents):
        st = steps[p]
        blk = out[pos:pos + counts[p], st]
        ser = np.array([s for s, _ in tilings[p]], dtype=np.uint8)
        thr = np.array([t for _, t in tilings[p]], dtype=np.uint8)
        nd = ser.shape[1]
        blk["serial"][:, :nd] = ser
        blk["thread"][:, :nd] = thr
        blk["flags"] = 3
        out[pos:pos + counts[p], st] = blk
        pos += counts[p]
    return out, owner, info


def random_schedules(graph, n, seed=0, S=None, menus=Menus):
    """n fully scheduled random candidates (packed) + their decision tuples."""
    info = GraphInfo(graph, menus)
    S = S or len(info.order)
    rng = np.random.default_rng(seed)
    decs = [info.random_full(rng) for _ in range(n)]
    return info.pack_rows(decs, S), [info.to_decisions(d) for d in decs], info
