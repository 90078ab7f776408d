"""ctypes binding of libgs_sched.so (the C ABI in include/gs_sched.h).

The library is built in-tree by `_build.build()`; importing this module
never falls back to anything else: a missing library or a failing call
raises `GsError`.
"""

from __future__ import annotations

import ctypes as C
import os

from .descriptor import GsPipelineDesc

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GS_LIB_PATH") or os.path.join(HERE, "libgs_sched.so")   # override: diagnostics builds

EXPORTS = ("gs_last_error", "gs_version", "gs_launch_count", "gs_pipeline_create", "gs_pipeline_destroy",
           "gs_pipeline_max_rows", "gs_set_weights", "gs_set_reuse", "gs_featurize", "gs_cost", "gs_cost_totals",
           "gs_struct_hash", "gs_select_workspace_bytes", "gs_select_reps",
           "gs_topk_workspace_bytes", "gs_beam_topk", "gs_check", "gs_stats", "gs_debug_phases",
           "gs_expand_workspace_bytes", "gs_expand_step", "gs_simulate", "gs_featurize_workspace_bytes",
           "gs_featurize_ws", "gs_struct_hash_workspace_bytes", "gs_struct_hash_ws", "gs_beam_topk_reps",
           "gs_model_params", "gs_predict", "gs_train_workspace_bytes", "gs_train",
           "gs_set_placement_info", "gs_phase1_workspace_bytes", "gs_expand_phase1",
           "gs_random_schedules", "gs_get_reuse", "gs_struct_hash_depths_ws")


class GsError(RuntimeError):
    pass


_lib = None


def load(path: str = LIB_PATH):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise GsError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(or paper_2012_07145_b200/_build.py); there is no CPU fallback")
    lib = C.CDLL(path)
    P, V, i32, i64, u64, dbl = C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
    sig = {
        "gs_last_error": (C.c_char_p, []),
        "gs_version": (i32, []),
        "gs_launch_count": (i64, []),
        "gs_pipeline_create": (i32, [C.POINTER(GsPipelineDesc), C.POINTER(P)]),
        "gs_pipeline_destroy": (i32, [P]),
        "gs_pipeline_max_rows": (i32, [P]),
        "gs_set_weights": (i32, [P, i32, i32] + [V] * 8),
        "gs_set_reuse": (i32, [P, i32]),
        "gs_get_reuse": (i32, [P]),
        "gs_featurize": (i32, [P, V, i64, i32, V, V, V, V, V, V]),
        "gs_cost": (i32, [P, V, V, V, V, i64, V, V, V, V]),
        "gs_cost_totals": (i32, [P, V, V, V, V, i64, V, V, V]),
        "gs_struct_hash": (i32, [P, V, i64, i32, i32, V, V]),
        "gs_select_workspace_bytes": (i64, [i64]),
        "gs_select_reps": (i32, [V, V, i64, u64, V, i64, V, V, V, V, V]),
        "gs_topk_workspace_bytes": (i64, [i64]),
        "gs_beam_topk": (i32, [V, V, i64, V, i64, dbl, dbl, u64, i64, dbl, V, i64, V, V, V, V]),
        "gs_check": (i32, [P, V]),
        "gs_stats": (i32, [P, V, V]),
        "gs_debug_phases": (i32, [V]),
        "gs_expand_workspace_bytes": (i64, [i64]),
        "gs_expand_step": (i32, [P, V, i64, i32, V, V, V, V, i64, V, i64, V, V]),
        "gs_simulate": (i32, [P, V, i64, i32, V, V, V, V, V]),
        "gs_featurize_workspace_bytes": (i64, [P, i64, i32, i64]),
        "gs_featurize_ws": (i32, [P, V, i64, i32, V, V, V, V, V, i64, V, i64, V]),
        "gs_struct_hash_workspace_bytes": (i64, [i64]),
        "gs_model_params": (i32, [i32, i32]),
        "gs_set_placement_info": (i32, [P, V, V, V, V, i32]),
        "gs_random_schedules": (i32, [P, u64, i64, i64, i32, V, V, V]),
        "gs_phase1_workspace_bytes": (i64, [i64]),
        "gs_expand_phase1": (i32, [P, V, i64, i32, i32, i32, V, V, V, i64, V, i64, V, V]),
        "gs_predict": (i32, [V, i32, i32, V, V, V, i64, V, V, V]),
        "gs_train_workspace_bytes": (i64, [i32, i32, i32]),
        "gs_train": (i32, [V, i32, i32, V, V, V, V, V, V, V, i32, i32, dbl, dbl, i32, V, i64, V, V, V]),
        "gs_beam_topk_reps": (i32, [V, V, V, i64, V, V, i64, dbl, dbl, u64, i64, dbl, V, i64, V, V, V, V]),
        "gs_struct_hash_ws": (i32, [P, V, i64, i32, i32, V, V, i64, V]),
        "gs_struct_hash_depths_ws": (i32, [P, V, i64, i32, i32, V, V, V, i64, V]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int):
    if rc != 0:
        msg = _lib.gs_last_error().decode(errors="replace") if _lib else "library not loaded"
        raise GsError(f"gs_sched error {rc}: {msg}")
    return rc
