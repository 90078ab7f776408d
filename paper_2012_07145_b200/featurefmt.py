"""Feature text v1: the versioned `name=value` dump of a candidate's feature
rows (reference `featurize.py:620-628`, `format_features`), produced from the
GPU feature tensor (K1) so a dump diffs directly against the reference's.

Rows are `((func name, stage), 56 values)`; the dump sorts them by
(func name, stage) and prints every value with 17 significant digits, in
FEATURE_ORDER (reference `featurize.py:153`)."""

from __future__ import annotations

FEATURE_VERSION = 1   # featurize.py:28

FEATURE_ORDER = (
    "num_scalars", "points_computed_per_thread",
    "unique_global_bytes_read_per_realization", "unique_shared_bytes_read_per_realization",
    "unique_register_bytes_read_per_realization", "unique_global_lines_read_per_realization",
    "unique_shared_lines_read_per_realization", "unique_register_lines_read_per_realization",
    "unique_global_bytes_read_per_thread", "unique_shared_bytes_read_per_thread",
    "unique_register_bytes_read_per_thread", "unique_global_lines_read_per_thread",
    "unique_shared_lines_read_per_thread", "unique_register_lines_read_per_thread",
    "global_allocation_bytes_read_per_realization", "shared_allocation_bytes_read_per_realization",
    "register_allocation_bytes_read_per_realization", "global_bytes_at_task", "shared_bytes_at_task",
    "register_bytes_at_task", "global_innermost_bytes_at_task", "shared_innermost_bytes_at_task",
    "register_innermost_bytes_at_task", "num_blocks", "num_warps_per_block",
    "num_active_warps_per_block", "num_threads_per_block", "expr_branching", "block_occupancy",
    "warp_lane_utilization", "idle_lane_wastage", "num_shared_mem_loads_per_block",
    "num_global_mem_loads_per_block", "num_shared_mem_stores_per_block",
    "num_global_mem_stores_per_block", "shared_mem_store_efficiency", "shared_mem_load_efficiency",
    "global_mem_store_efficiency", "global_mem_load_efficiency", "working_set_at_thread",
    "shared_mem_occupancy", "shared_mem_block_limit_factor", "max_warp_occupancy",
    "max_block_occupancy", "num_realizations", "num_productions", "num_tasks", "inner_parallelism",
    "tasks_per_core", "num_cores", "inlined_calls", "unique_bytes_read_per_point",
    "unique_lines_read_per_point", "unique_bytes_read_per_task", "unique_lines_read_per_task",
    "working_set")
assert len(FEATURE_ORDER) == 56


def format_features(rows) -> str:
    """Text dump of feature rows `((func, stage), values[56])`."""
    out = [f"# feature_version={FEATURE_VERSION}"]
    for (func, si), vals in sorted(rows, key=lambda r: r[0]):
        if len(vals) != len(FEATURE_ORDER):
            raise ValueError(f"row ({func}, {si}) has {len(vals)} features, expected {len(FEATURE_ORDER)}")
        out.append(f"[{func} stage {si}]")
        out.extend(f"{name}={float(v):.17g}" for name, v in zip(FEATURE_ORDER, vals))
    return "\n".join(out) + "\n"


def parse_features(text: str) -> dict:
    """Inverse of format_features: {(func, stage): [56 floats]}."""
    lines = [ln.strip() for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] != f"# feature_version={FEATURE_VERSION}":
        raise ValueError("not a feature text v1 dump")
    rows, key, vals = {}, None, []
    for ln in lines[1:]:
        if ln.startswith("["):
            if key is not None:
                rows[key] = vals
            func, _, si = ln[1:-1].rpartition(" stage ")
            key, vals = (func, int(si)), []
        else:
            name, _, v = ln.partition("=")
            if name != FEATURE_ORDER[len(vals)]:
                raise ValueError(f"feature {name!r} out of order in row {key}")
            vals.append(float(v))
    if key is not None:
        rows[key] = vals
    return rows


def candidate_rows(scorer, f, i):
    """Feature rows of candidate i of a `Scorer.featurize` output, as
    `((func name, stage), values)`.  In reuse mode 2 a repeated row is read
    from the candidate that computed it (`row_src`)."""
    n = int(f["n_rows"][i])
    keys = scorer.packed.row_keys(f["row_key"][i, :n].cpu().numpy())
    feats = f["feats"]
    if f.get("rows_only"):
        src = f["row_src"][i, :n].cpu().numpy()
        vals = [feats[int(s), r].cpu().numpy() for r, s in enumerate(src)]
    else:
        vals = list(feats[i, :n].cpu().numpy())
    return list(zip(keys, vals))
