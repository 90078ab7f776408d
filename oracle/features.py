"""56 schedule features per (func, stage) row (restates reference `featurize.py`).

Transaction counts are computed the brute-force way the reference does
(materialize every lane address of block 0 for every warp instruction and
count segments / bank conflicts per row, featurize.py:173-196, 508-571), so
this checker shares no shortcut with the CUDA path, which counts only the
distinct per-instruction address residues.
"""

from __future__ import annotations

import math

import numpy as np

from .boxes import through_links, union_count
from .geometry import resolve_geometry

FEATURES = (
    "num_scalars", "points_computed_per_thread",
    "unique_global_bytes_read_per_realization", "unique_shared_bytes_read_per_realization",
    "unique_register_bytes_read_per_realization", "unique_global_lines_read_per_realization",
    "unique_shared_lines_read_per_realization", "unique_register_lines_read_per_realization",
    "unique_global_bytes_read_per_thread", "unique_shared_bytes_read_per_thread",
    "unique_register_bytes_read_per_thread", "unique_global_lines_read_per_thread",
    "unique_shared_lines_read_per_thread", "unique_register_lines_read_per_thread",
    "global_allocation_bytes_read_per_realization", "shared_allocation_bytes_read_per_realization",
    "register_allocation_bytes_read_per_realization",
    "global_bytes_at_task", "shared_bytes_at_task", "register_bytes_at_task",
    "global_innermost_bytes_at_task", "shared_innermost_bytes_at_task",
    "register_innermost_bytes_at_task",
    "num_blocks", "num_warps_per_block", "num_active_warps_per_block", "num_threads_per_block",
    "expr_branching", "block_occupancy", "warp_lane_utilization", "idle_lane_wastage",
    "num_shared_mem_loads_per_block", "num_global_mem_loads_per_block",
    "num_shared_mem_stores_per_block", "num_global_mem_stores_per_block",
    "shared_mem_store_efficiency", "shared_mem_load_efficiency",
    "global_mem_store_efficiency", "global_mem_load_efficiency",
    "working_set_at_thread", "shared_mem_occupancy", "shared_mem_block_limit_factor",
    "max_warp_occupancy", "max_block_occupancy",
    "num_realizations", "num_productions", "num_tasks", "inner_parallelism",
    "tasks_per_core", "num_cores", "inlined_calls",
    "unique_bytes_read_per_point", "unique_lines_read_per_point",
    "unique_bytes_read_per_task", "unique_lines_read_per_task", "working_set",
)  # featurize.py:78-155 field order
FIDX = {n: i for i, n in enumerate(FEATURES)}
OPS = ("add", "mul", "div", "minmax", "transcendental", "cast", "compare")
_DEFAULTS = {"expr_branching": 1.0, "block_occupancy": 1.0, "warp_lane_utilization": 1.0,
             "shared_mem_store_efficiency": 1.0, "shared_mem_load_efficiency": 1.0,
             "global_mem_store_efficiency": 1.0, "global_mem_load_efficiency": 1.0,
             "shared_mem_block_limit_factor": 1.0, "max_warp_occupancy": 1.0,
             "max_block_occupancy": 1.0, "inner_parallelism": 1.0, "num_cores": 1.0}
TIERS = ("global", "shared", "register")


def strahler(tree) -> int:
    """featurize.py:31-39."""
    if tree is None:
        return 1
    v = [strahler(c) for c in tree]
    if not v:
        return 1
    m = max(v)
    return m + 1 if v.count(m) > 1 else m


def stage_branching(stage) -> int:
    """featurize.py:306-309."""
    if stage.expr_tree is not None:
        return strahler(stage.expr_tree)
    return 2 if sum(stage.op_histogram.values()) >= 2 else 1


def algo_vector(func_node, si):
    """featurize.py:64-75 (order of `AlgorithmFeatures.to_vector`)."""
    st = func_node.stages[si]
    vols = [a.window_volume for a in st.accesses]
    return np.array([float(st.op_histogram.get(o, 0)) for o in OPS]
                    + [float(len(st.accesses)), float(np.mean(vols)) if vols else 0.0,
                       float(func_node.elem_bytes)], dtype=np.float64)


# ---------------------------------------------------------------------------
# transaction counting: brute force over block 0
# ---------------------------------------------------------------------------

_BIAS = 1 << 40


def _count(addr_rows, tier, mp):
    """addr_rows int64 [rows, warp]; -1 = inactive lane."""
    if addr_rows.size == 0:
        return 0
    if tier == "global":
        seg = np.where(addr_rows >= 0, addr_rows // mp.global_transaction_bytes, -1)
        seg.sort(axis=1)
        new = np.ones_like(seg, dtype=bool)
        new[:, 1:] = seg[:, 1:] != seg[:, :-1]
        return int((new & (seg >= 0)).sum())
    word = np.where(addr_rows >= 0, addr_rows // mp.bank_width_bytes, -1)
    word.sort(axis=1)
    new = np.ones_like(word, dtype=bool)
    new[:, 1:] = word[:, 1:] != word[:, :-1]
    new &= word >= 0
    rows = word.shape[0]
    r_idx = np.broadcast_to(np.arange(rows)[:, None], word.shape)
    bank = np.mod(word, mp.shared_banks)
    hist = np.zeros((rows, mp.shared_banks), dtype=np.int64)
    np.add.at(hist, (r_idx[new], bank[new]), 1)
    return int(hist.max(axis=1).sum())


def _layout(geo, eb):
    los = [lo for lo, _ in geo.region]
    strides, acc = [], eb
    for lo, hi in geo.region:
        strides.append(acc)
        acc *= hi - lo + 1
    return los, strides


def _tids(n, ctx):
    t = np.arange(n, dtype=np.int64)
    cols = []
    for e in ctx:
        cols.append(t % e)
        t = t // e
    return cols


def _instr_offsets(chain, ext, unrolled):
    """Per-dim relative producer coordinates touched by one lane, one entry
    per emitted load (featurize.py:211-232)."""
    nd = len(ext)
    per = []
    for d in range(nd):
        links = [link[d] for link in chain]
        if unrolled:
            ivs = through_links([(0, ext[d] - 1)], links)
            per.append(np.concatenate([np.arange(lo, hi + 1, dtype=np.int64) for lo, hi in ivs]))
        else:
            v = np.arange(ext[d], dtype=np.int64)
            for s, lo, hi in links:
                v = (v[:, None] * s + np.arange(lo, hi + 1, dtype=np.int64)[None, :]).ravel()
            per.append(v)
    return per


def _rel_addresses(per_dim, strides):
    # cross product, dim 0 fastest (order irrelevant for counts)
    rel = np.zeros(1, dtype=np.int64)
    for d in range(len(per_dim)):
        rel = (per_dim[d][:, None] * strides[d] + rel[None, :]).ravel()
    return rel


def _warp_count(origins, rel, n_threads, tier, mp):
    ws = mp.warp_size
    warps = -(-n_threads // ws)
    base = np.full(warps * ws, -1, dtype=np.int64)
    base[:n_threads] = origins + _BIAS
    base = base.reshape(warps, ws)
    active = base >= 0
    total = 0
    chunk = max(1, (1 << 21) // (warps * ws))
    for i in range(0, rel.size, chunk):
        r = rel[i:i + chunk]
        a = base[None, :, :] + r[:, None, None]
        a = np.where(active[None], a, -1)
        total += _count(a.reshape(-1, ws), tier, mp)
    return total


def loads_for(geos, host, reads, mp):
    """Load transactions of block 0 per tier (featurize.py:527-554)."""
    out = {"global": 0, "shared": 0}
    tc = _tids(host.n_threads, host.ctx)
    for r in reads:
        if r.tier not in out:
            continue
        pg = geos[r.producer]
        los, strides = _layout(pg, r.elem_bytes)
        ts = r.total_stride
        org = np.zeros(host.n_threads, dtype=np.int64)
        for d in range(len(host.ext)):
            org += (tc[d] * (host.coeff[d] * ts[d]) + host.base[d] * ts[d] - los[d]) * strides[d]
        rel = _rel_addresses(_instr_offsets(r.chain, host.ext, host.unrolled), strides)
        out[r.tier] += _warp_count(org, rel, host.n_threads, r.tier, mp)
    return out


def stores_for(g, eb, mp):
    """Store transactions of block 0 into the func's own allocation
    (featurize.py:557-571)."""
    if g.tier not in ("global", "shared"):
        return 0
    los, strides = _layout(g, eb)
    tc = _tids(g.n_threads, g.ctx)
    org = np.zeros(g.n_threads, dtype=np.int64)
    for d in range(len(g.ext)):
        org += (tc[d] * g.coeff[d] + g.base[d] - los[d]) * strides[d]
    rel = _rel_addresses([np.arange(e, dtype=np.int64) for e in g.ext], strides)
    return _warp_count(org, rel, g.n_threads, g.tier, mp)


# ---------------------------------------------------------------------------
# unique bytes / lines over a box
# ---------------------------------------------------------------------------

def uniques(graph, reads, box):
    """Per-tier (bytes, lines) of the union of the reads' footprints over a
    box, grouped by (tier, producer) (featurize.py:393-412)."""
    groups = {}
    for r in reads:
        prod = [through_links([iv], [link[d] for link in r.chain]) for d, iv in enumerate(box)]
        groups.setdefault((r.tier, r.producer), []).append(prod)
    b = {t: 0 for t in TIERS}
    ln = {t: 0 for t in TIERS}
    for (tier, producer), prods in groups.items():
        b[tier] += union_count(prods, False) * graph.func(producer).elem_bytes
        ln[tier] += union_count(prods, True)
    return b, ln, groups


# ---------------------------------------------------------------------------
# rows
# ---------------------------------------------------------------------------

def _parallel(v, mp, n, kern):
    """featurize.py:317-363."""
    kt = kern.threads
    ws = mp.warp_size
    aw = -(-n // ws)
    v["num_blocks"] = float(kern.n_blocks)
    v["num_warps_per_block"] = float(-(-kt // ws))
    v["num_active_warps_per_block"] = float(aw)
    v["num_threads_per_block"] = float(n)
    v["warp_lane_utilization"] = n / (ws * aw)
    v["idle_lane_wastage"] = (ws * aw - n) / mp.max_threads_per_block
    v["block_occupancy"] = kt / mp.max_threads_per_block
    wpb = max(1, -(-kt // ws))
    if kern.shared_bytes > 0:
        by_shared = max(1, mp.shared_mem_per_sm // kern.shared_bytes)
        v["shared_mem_occupancy"] = min(1.0, kern.shared_bytes / mp.shared_mem_per_block_limit)
    else:
        by_shared = mp.max_active_blocks_per_sm
        v["shared_mem_occupancy"] = 0.0
    v["shared_mem_block_limit_factor"] = (min(by_shared, mp.max_active_blocks_per_sm)
                                          / mp.max_active_blocks_per_sm)
    act = max(1, min(mp.max_active_blocks_per_sm, by_shared, mp.max_active_warps_per_sm // wpb))
    aw_sm = min(mp.max_active_warps_per_sm, act * wpb)
    v["max_warp_occupancy"] = aw_sm / mp.max_active_warps_per_sm
    v["max_block_occupancy"] = act / mp.max_active_blocks_per_sm
    v["num_tasks"] = float(kern.n_blocks)
    v["inner_parallelism"] = float(n)
    v["num_cores"] = float(mp.num_sms)
    v["tasks_per_core"] = kern.n_blocks / mp.num_sms


def _efficiencies(v, mp, used, stored, store_tier, store_tx):
    """featurize.py:366-390."""
    gtx = mp.global_transaction_bytes
    stx = mp.shared_banks * mp.bank_width_bytes
    if v["num_global_mem_loads_per_block"] > 0:
        v["global_mem_load_efficiency"] = min(1.0, used["global"] / (v["num_global_mem_loads_per_block"] * gtx))
    if v["num_shared_mem_loads_per_block"] > 0:
        v["shared_mem_load_efficiency"] = min(1.0, used["shared"] / (v["num_shared_mem_loads_per_block"] * stx))
    if store_tier == "global" and store_tx > 0:
        v["global_mem_store_efficiency"] = min(1.0, stored / (store_tx * gtx))
    elif store_tier == "shared" and store_tx > 0:
        v["shared_mem_store_efficiency"] = min(1.0, stored / (store_tx * stx))


def _blank():
    v = {n: 0.0 for n in FEATURES}
    v.update(_DEFAULTS)
    return v


def _set_thread_uniques(v, b, ln):
    for t in TIERS:
        v[f"unique_{t}_bytes_read_per_thread"] = float(b[t])
        v[f"unique_{t}_lines_read_per_thread"] = float(ln[t])


def _used(groups_blk, graph):
    used = {"global": 0, "shared": 0}
    for (tier, producer), prods in groups_blk.items():
        if tier in used:
            used[tier] += union_count(prods, False) * graph.func(producer).elem_bytes
    return used


def stage_row(graph, geos, kernels, mp, g, si):
    """featurize.py:415-505."""
    node = graph.func(g.name)
    kern = kernels[g.kernel]
    v = _blank()
    _parallel(v, mp, g.n_threads, kern)
    v["num_scalars"] = float(g.pts_block * kern.n_blocks)
    v["points_computed_per_thread"] = float(g.pts_thread)
    v["num_realizations"] = v["num_productions"] = float(g.realizations)
    reads = [r for r in (g.reads[si] if si < len(g.reads) else []) if r.owner == g.name]

    b, ln, groups = uniques(graph, reads, g.region)
    for t in TIERS:
        v[f"unique_{t}_bytes_read_per_realization"] = float(b[t])
        v[f"unique_{t}_lines_read_per_realization"] = float(ln[t])
    bt, lt, _ = uniques(graph, reads, g.lane_box())
    _set_thread_uniques(v, bt, lt)
    alloc = {t: 0 for t in TIERS}
    for tier, producer in groups:
        alloc[tier] += geos[producer].alloc * graph.func(producer).elem_bytes
    for t in TIERS:
        v[f"{t}_allocation_bytes_read_per_realization"] = float(alloc[t])

    eb = node.elem_bytes
    written = g.pts_block * eb
    blk = g.block_box()
    v[f"{g.tier}_bytes_at_task"] = float(written)
    v[f"{g.tier}_innermost_bytes_at_task"] = float((blk[0][1] - blk[0][0] + 1) * eb)

    bb, lb, groups_blk = uniques(graph, reads, blk)
    loads = loads_for(geos, g, reads, mp)
    v["num_global_mem_loads_per_block"] = float(loads["global"])
    v["num_shared_mem_loads_per_block"] = float(loads["shared"])
    st = stores_for(g, eb, mp)
    if g.tier in ("global", "shared"):
        v[f"num_{g.tier}_mem_stores_per_block"] = float(st)
    _efficiencies(v, mp, _used(groups_blk, graph), written, g.tier, st)

    wst = g.alloc * eb if g.tier == "register" else 0
    for o in geos.values():
        if o.kind == "fuse_at_thread" and o.consumer == g.name:
            wst += o.alloc * graph.func(o.name).elem_bytes
    if g.unrolled:
        wst += v["unique_global_bytes_read_per_thread"] + v["unique_shared_bytes_read_per_thread"]
    v["working_set_at_thread"] = float(wst)
    v["working_set"] = float(g.alloc * eb)

    bp, lp, _ = uniques(graph, reads, [(b0, b0) for b0 in g.base])
    v["unique_bytes_read_per_point"] = float(sum(bp.values()))
    v["unique_lines_read_per_point"] = float(sum(lp.values()))
    v["unique_bytes_read_per_task"] = float(sum(bb.values()))
    v["unique_lines_read_per_task"] = float(sum(lb.values()))
    return v


def inline_row(graph, geos, kernels, mp, g):
    """featurize.py:574-617."""
    v = _blank()
    host = geos.get(g.primary) if g.primary else None
    if host is None:
        v["inlined_calls"] = float(max(1, g.calls))
        v["num_scalars"] = float(g.calls)
        return v
    kern = kernels[host.kernel]
    _parallel(v, mp, host.n_threads, kern)
    v["inlined_calls"] = float(g.calls)
    v["num_scalars"] = float(g.calls)
    den = kern.n_blocks * host.n_threads
    v["points_computed_per_thread"] = g.calls / den if den else 0.0
    reads = g.reads[0] if g.reads else []
    bt, lt, _ = uniques(graph, reads, host.lane_box())
    _set_thread_uniques(v, bt, lt)
    loads = loads_for(geos, host, reads, mp)
    v["num_global_mem_loads_per_block"] = float(loads["global"])
    v["num_shared_mem_loads_per_block"] = float(loads["shared"])
    bb, lb, groups_blk = uniques(graph, reads, host.block_box())
    _efficiencies(v, mp, _used(groups_blk, graph), 0.0, None, 0)
    v["unique_bytes_read_per_task"] = float(sum(bb.values()))
    v["unique_lines_read_per_task"] = float(sum(lb.values()))
    bp, lp, _ = uniques(graph, reads, [(b0, b0) for b0 in host.base])
    v["unique_bytes_read_per_point"] = float(sum(bp.values()))
    v["unique_lines_read_per_point"] = float(sum(lp.values()))
    return v


def featurize_rows(graph, decisions, mp):
    """Ordered rows [(func, stage), feature vector f64[56], algo f64[10]]
    (featurize.py:275-303).  Row order = geometry insertion order."""
    geos, kernels = resolve_geometry(graph, decisions)
    rows = []
    for name, g in geos.items():
        if g.kind == "external":
            continue
        node = graph.func(name)
        if g.kind == "inline":
            v = inline_row(graph, geos, kernels, mp, g)
            v["expr_branching"] = float(stage_branching(node.stages[0]))
            rows.append(((name, 0), np.array([v[n] for n in FEATURES]), algo_vector(node, 0)))
            continue
        for si in range(len(node.stages)):
            v = stage_row(graph, geos, kernels, mp, g, si)
            v["expr_branching"] = float(stage_branching(node.stages[si]))
            rows.append(((name, si), np.array([v[n] for n in FEATURES]), algo_vector(node, si)))
    return rows
