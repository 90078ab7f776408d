"""Cost basis, coefficient network, stage/total cost and prune verdicts
(restates reference `costmodel.py:118-176, 271-293`, `search.py:90-124`,
`options.py:200-255`, `machine.py:91-105`)."""

from __future__ import annotations

import math

import numpy as np

from .features import FIDX, featurize_rows
from .geometry import resolve_geometry

NUM_COEFFS = 30
_EPS = 1e-8


def basis(f):
    """(g[30], h) with stage cost = g . c + h (costmodel.py:118-176)."""
    F = lambda n: f[FIDX[n]]  # noqa: E731
    g = np.zeros(NUM_COEFFS)
    inl = F("inlined_calls") > 0
    scale = math.ceil(F("num_tasks") / F("num_cores")) / max(1.0, F("tasks_per_core"))
    if not inl:
        scale /= 1.0 - F("idle_lane_wastage")
    pts = F("num_blocks") * F("num_threads_per_block") * F("points_computed_per_thread")
    g[3 if inl else 1] += F("num_scalars") * scale
    g[4 if inl else 19] += pts * scale
    r = F("num_realizations")
    for idx, name in ((5, "unique_global_lines_read_per_realization"),
                      (16, "unique_shared_lines_read_per_realization"),
                      (8, "unique_register_lines_read_per_realization"),
                      (6, "unique_global_bytes_read_per_realization"),
                      (20, "unique_shared_bytes_read_per_realization"),
                      (7, "unique_register_bytes_read_per_realization"),
                      (18, "unique_global_lines_read_per_thread"),
                      (17, "unique_shared_lines_read_per_thread"),
                      (2, "unique_register_lines_read_per_thread"),
                      (13, "unique_global_bytes_read_per_thread"),
                      (11, "unique_shared_bytes_read_per_thread"),
                      (0, "unique_register_bytes_read_per_thread")):
        g[idx] += r * F(name)
    g[10] += F("num_scalars") * F("unique_bytes_read_per_point")
    g[12] += F("num_scalars") * F("unique_lines_read_per_point")
    g[14] += F("num_tasks") * F("unique_bytes_read_per_task")
    g[15] += F("num_tasks") * F("unique_lines_read_per_task")
    gl = F("num_blocks") * F("num_global_mem_loads_per_block")
    sl = F("num_blocks") * F("num_shared_mem_loads_per_block")
    if not inl:
        gl /= F("global_mem_load_efficiency")
        sl /= F("shared_mem_load_efficiency")
    h = 0.0 + gl + sl
    g[29] += F("num_blocks") * F("num_shared_mem_stores_per_block")
    gs = F("num_blocks") * F("num_global_mem_stores_per_block")
    if not inl:
        gs /= F("global_mem_store_efficiency")
    g[21] += gs
    if F("inner_parallelism") > 1:
        g[22] += F("num_scalars") / max(1.0, F("global_innermost_bytes_at_task"))
    g[24] += F("num_realizations")
    if F("inner_parallelism") > 1:
        g[25] += F("num_productions")
    g[26] += F("num_productions") * (F("inner_parallelism") - 1)
    g[9] += F("working_set")
    return g, h


def coefficients(w, xa, xs):
    """Two-tower forward in fp64 (costmodel.py:275-293).  `w` maps the eight
    tensor names to arrays."""
    xs = np.log1p(np.asarray(xs, dtype=np.float64))
    ea = np.maximum(np.asarray(xa, dtype=np.float64) @ w["algo_w"] + w["algo_b"], 0.0)
    es = np.maximum(xs @ w["sched_w"] + w["sched_b"], 0.0)
    eh = np.maximum(np.concatenate([ea, es]) @ w["head_w"] + w["head_b"], 0.0)
    return np.logaddexp(0.0, eh @ w["out_w"] + w["out_b"]) + _EPS


def score(graph, decisions, mp, w):
    """(total, [(key, row cost)], rows) — `CostEvaluator.cost` (search.py:115-124):
    per-row c = g . coeffs + h, total = sequential sum in row order."""
    rows = featurize_rows(graph, decisions, mp)
    total, per = 0.0, []
    for key, f, xa in rows:
        g, h = basis(f)
        c = float(g @ coefficients(w, xa, f)) + h
        per.append((key, c))
        total += c
    return total, per, rows


PRUNE_REASONS = ("excessive_recompute", "idle_sms", "poor_warp_utilization",
                 "serial_too_large", "thread_alloc_dynamic_or_large", "hardware_limit")


def prune_reason(graph, decisions, mp, th):
    """First failing prune rule or None (options.py:200-255, machine.py:91-105)."""
    geos, kernels = resolve_geometry(graph, decisions)
    computed = needed = 0
    for name, g in geos.items():
        if g.kind == "external":
            continue
        needed += graph.func(name).domain_size
        computed += g.calls if g.kind == "inline" else g.pts_block * kernels[g.kernel].n_blocks
    if needed and computed > th.recompute_factor * needed:
        return "excessive_recompute"
    floor_blocks = th.min_blocks_per_sm_factor * mp.num_sms
    for k in kernels.values():
        if k.n_blocks < floor_blocks:
            return "idle_sms"
    for name, g in geos.items():
        if g.kind in ("external", "inline"):
            continue
        warps = -(-g.n_threads // mp.warp_size)
        if g.n_threads / (warps * mp.warp_size) < th.warp_utilization_floor:
            return "poor_warp_utilization"
        if g.serial is not None and math.prod(g.serial) > th.unroll_budget:
            return "serial_too_large"
        if g.kind == "fuse_at_thread" and g.alloc * graph.func(name).elem_bytes > th.thread_alloc_bytes:
            return "thread_alloc_dynamic_or_large"
    for k in kernels.values():
        if k.threads > mp.max_threads_per_block or k.shared_bytes > mp.shared_mem_per_block_limit:
            return "hardware_limit"
    return None
