"""Pack pipelines, machine params and candidate decision logs into the
C-ABI structures of include/gs_sched.h.

Works on reference `gpusched` objects and on this package's own
(duck-typed: see pipeline.py / schedule.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

MAX_NDIM = 4
KIND_CODE = {"compute_root": 0, "fuse_at_block": 1, "fuse_at_thread": 2, "inline": 3}
KIND_NAME = {v: k for k, v in KIND_CODE.items()}
OPS = ("add", "mul", "div", "minmax", "transcendental", "cast", "compare")
PRUNE_REASONS = ("excessive_recompute", "idle_sms", "poor_warp_utilization",
                 "serial_too_large", "thread_alloc_dynamic_or_large", "hardware_limit")
DECISION_DTYPE = np.dtype([("func", "<u2"), ("consumer", "<u2"), ("kind", "u1"), ("flags", "u1"),
                           ("serial", "u1", (4,)), ("thread", "u1", (4,)), ("pad", "<u2")])
assert DECISION_DTYPE.itemsize == 16


class GsFunc(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("extent", C.c_int32 * 4), ("elem_bytes", C.c_int32),
                ("is_external", C.c_int32), ("is_output", C.c_int32), ("n_stages", C.c_int32),
                ("stage_begin", C.c_int32), ("name_rank", C.c_int32), ("pad", C.c_int32)]


class GsStage(C.Structure):
    _fields_ = [("func", C.c_int32), ("n_access", C.c_int32), ("access_begin", C.c_int32),
                ("branching", C.c_int32)]


class GsAccess(C.Structure):
    _fields_ = [("producer", C.c_int32), ("consumer", C.c_int32), ("stage", C.c_int32),
                ("window", C.c_int32), ("s", C.c_int32 * 4), ("lo", C.c_int32 * 4),
                ("hi", C.c_int32 * 4)]


class GsMachine(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "warp_size", "num_sms", "max_threads_per_block", "max_active_warps_per_sm",
        "max_active_blocks_per_sm", "shared_mem_per_block_limit", "shared_mem_per_sm",
        "global_transaction_bytes", "shared_banks", "bank_width_bytes")]


class GsThresholds(C.Structure):
    _fields_ = [("recompute_factor", C.c_double), ("min_blocks_per_sm_factor", C.c_double),
                ("warp_utilization_floor", C.c_double), ("unroll_budget", C.c_int64),
                ("thread_alloc_bytes", C.c_int64)]


class GsTilingMenus(C.Structure):
    _fields_ = [("serial_powers", C.c_int32 * 8), ("n_serial_powers", C.c_int32),
                ("odd_serial", C.c_int32 * 8), ("n_odd_serial", C.c_int32),
                ("innermost_thread", C.c_int32 * 8), ("n_innermost", C.c_int32),
                ("outer_thread", C.c_int32 * 8), ("n_outer", C.c_int32),
                ("unroll_budget", C.c_int32), ("warp_size", C.c_int32)]


class GsOracleParams(C.Structure):
    """Machine-oracle throughput knobs (reference machine.py:24-31)."""
    _fields_ = [("registers_per_thread_budget", C.c_int32), ("pad", C.c_int32),
                ("compute_throughput", C.c_double), ("global_bandwidth", C.c_double),
                ("shared_bandwidth", C.c_double), ("kernel_launch_overhead", C.c_double)]


def oracle_params(mp) -> GsOracleParams:
    """Pack the oracle knobs of a MachineParams-like object."""
    return GsOracleParams(int(mp.registers_per_thread_budget), 0, float(mp.compute_throughput),
                          float(mp.global_bandwidth), float(mp.shared_bandwidth),
                          float(mp.kernel_launch_overhead))


def tiling_menus(menus) -> GsTilingMenus:
    """Pack a TilingConfig-like object (reference options.py:25-37)."""
    m = GsTilingMenus()
    for name, cnt in (("serial_powers", "n_serial_powers"), ("odd_serial", "n_odd_serial"),
                      ("innermost_thread", "n_innermost"), ("outer_thread", "n_outer")):
        vals = tuple(getattr(menus, name))
        if len(vals) > 8:
            raise ValueError(f"{name}: at most 8 menu values")
        arr = getattr(m, name)
        for i, v in enumerate(vals):
            arr[i] = int(v)
        setattr(m, cnt, len(vals))
    m.unroll_budget = int(menus.unroll_budget)
    m.warp_size = int(menus.warp_size)
    return m


class GsPipelineDesc(C.Structure):
    _fields_ = [("n_funcs", C.c_int32), ("n_stages", C.c_int32), ("n_access", C.c_int32),
                ("funcs", C.POINTER(GsFunc)), ("stages", C.POINTER(GsStage)),
                ("access", C.POINTER(GsAccess)), ("algo", C.POINTER(C.c_double)),
                ("name_repr", C.POINTER(C.c_uint8)), ("name_off", C.POINTER(C.c_int32)),
                ("machine", GsMachine), ("thresholds", GsThresholds)]


def strahler(tree) -> int:
    """Strahler number of an expression-tree shape (featurize.py:31-39)."""
    if tree is None:
        return 1
    v = [strahler(c) for c in tree]
    if not v:
        return 1
    m = max(v)
    return m + 1 if v.count(m) > 1 else m


def _branching(stage) -> int:
    if stage.expr_tree is not None:
        return strahler(stage.expr_tree)
    return 2 if sum(stage.op_histogram.values()) >= 2 else 1


class PackedPipeline:
    """Flat, C-ABI-ready description of one pipeline + machine + thresholds.

    Keeps the ctypes arrays alive for as long as the descriptor is in use.
    """

    def __init__(self, graph, params, thresholds):
        self.graph = graph
        funcs = list(graph.funcs)
        self.names = [f.name for f in funcs]
        self.index = {n: i for i, n in enumerate(self.names)}
        nf = len(funcs)
        if nf > 0x7FFF:
            raise ValueError("too many funcs")
        ranks = {n: r for r, n in enumerate(sorted(self.names))}
        stages, access, algo = [], [], []
        self.funcs = (GsFunc * nf)()
        self.stage_of = []   # global stage index -> (func, stage)
        for fi, f in enumerate(funcs):
            if f.ndim > MAX_NDIM:
                raise ValueError(f"func {f.name}: ndim {f.ndim} > {MAX_NDIM}")
            g = self.funcs[fi]
            g.ndim = f.ndim
            for d in range(MAX_NDIM):
                g.extent[d] = f.extents[d] if d < f.ndim else 1
            g.elem_bytes = f.elem_bytes
            g.is_external = int(bool(f.is_external_input))
            g.is_output = int(f.name in graph.outputs)
            g.n_stages = len(f.stages)
            g.stage_begin = len(stages)
            g.name_rank = ranks[f.name]
            for si, st in enumerate(f.stages):
                sd = GsStage()
                sd.func = fi
                sd.n_access = len(st.accesses)
                sd.access_begin = len(access)
                sd.branching = _branching(st)
                gsi = len(stages)
                stages.append(sd)
                self.stage_of.append((f.name, si))
                vols = []
                for a in st.accesses:
                    ad = GsAccess()
                    ad.producer = self.index[a.producer]
                    ad.consumer = fi
                    ad.stage = gsi
                    w = 1
                    for d, (s, lo, hi) in enumerate(a.dims):
                        ad.s[d], ad.lo[d], ad.hi[d] = s, lo, hi
                        w *= hi - lo + 1
                    ad.window = w
                    vols.append(w)
                    access.append(ad)
                algo.append([float(st.op_histogram.get(o, 0)) for o in OPS]
                            + [float(len(st.accesses)), float(np.mean(vols)) if vols else 0.0,
                               float(f.elem_bytes)])
        self.n_funcs, self.n_stages, self.n_access = nf, len(stages), len(access)
        self.stages = (GsStage * max(1, len(stages)))(*stages)
        self.access = (GsAccess * max(1, len(access)))(*access)
        self.algo = np.ascontiguousarray(np.array(algo, dtype=np.float64).reshape(-1, 10))
        reprs = [repr(n).encode("utf-8") for n in self.names]
        self.name_blob = np.frombuffer(b"".join(reprs) or b"\0", dtype=np.uint8).copy()
        self.name_off = np.cumsum([0] + [len(r) for r in reprs]).astype(np.int32)
        self.max_rows = sum(len(f.stages) for f in funcs if not f.is_external_input)
        self.desc = GsPipelineDesc()
        d = self.desc
        d.n_funcs, d.n_stages, d.n_access = nf, len(stages), len(access)
        d.funcs = C.cast(self.funcs, C.POINTER(GsFunc))
        d.stages = C.cast(self.stages, C.POINTER(GsStage))
        d.access = C.cast(self.access, C.POINTER(GsAccess))
        d.algo = self.algo.ctypes.data_as(C.POINTER(C.c_double))
        d.name_repr = self.name_blob.ctypes.data_as(C.POINTER(C.c_uint8))
        d.name_off = self.name_off.ctypes.data_as(C.POINTER(C.c_int32))
        for n, _ in GsMachine._fields_:
            setattr(d.machine, n, int(getattr(params, n)))
        t = thresholds
        d.thresholds.recompute_factor = float(t.recompute_factor)
        d.thresholds.min_blocks_per_sm_factor = float(t.min_blocks_per_sm_factor)
        d.thresholds.warp_utilization_floor = float(t.warp_utilization_floor)
        d.thresholds.unroll_budget = int(t.unroll_budget)
        d.thresholds.thread_alloc_bytes = int(t.thread_alloc_bytes)
        self.stage_index = {k: i for i, k in enumerate(self.stage_of)}

    def placement_info(self):
        """Static per-func facts of the phase-1 menus (gs_set_placement_info),
        with the reference's definitions: consumers_of (pipeline.py:127-134),
        _is_pointwise_called (options.py:74-86), apply_decision's inline rules
        (loopnest.py:199-205) and CHEAP_INLINE_OPS = 8 (options.py:22)."""
        g = self.graph
        funcs = list(g.funcs)
        flags = np.zeros(len(funcs), dtype=np.uint8)
        off, cons = [0], []
        for fi, f in enumerate(funcs):
            cs = g.consumers_of(f.name)
            cons.extend(self.index[c] for c in cs)
            off.append(len(cons))
            single = len(f.stages) == 1
            self_read = any(a.producer == f.name for st in f.stages for a in st.accesses)
            is_out = f.name in g.outputs
            found, pointwise = False, True
            for c in cs:
                for st in g.func(c).stages:
                    for a in st.accesses:
                        if a.producer == f.name:
                            found = True
                            if not a.is_pointwise():
                                pointwise = False
            ops = sum(sum(st.op_histogram.values()) for st in f.stages)
            flags[fi] = ((1 if is_out else 0) | (2 if single else 0) | (4 if found and pointwise else 0)
                         | (8 if (not is_out and single and not self_read and not f.is_external_input) else 0)
                         | (16 if ops <= 8 else 0))
        order = np.array([self.index[f] for f in reversed(g.topo_order)
                          if not g.func(f).is_external_input], dtype=np.int32)
        return flags, np.array(off, dtype=np.int32), np.array(cons or [0], dtype=np.int32), order

    def max_decisions(self) -> int:
        return sum(1 for f in self.graph.funcs if not f.is_external_input)

    # -- candidates ---------------------------------------------------------
    def pack(self, candidates, stride: int | None = None) -> np.ndarray:
        """Decision logs -> structured array [N, S] of 16-byte records.
        `candidates` holds decision tuples or objects with `.decisions`."""
        S = stride or max(1, self.max_decisions())
        out = np.zeros((len(candidates), S), dtype=DECISION_DTYPE)
        out["func"] = 0xFFFF
        out["consumer"] = 0xFFFF
        idx = self.index
        for c, cand in enumerate(candidates):
            decs = getattr(cand, "decisions", cand)
            if len(decs) > S:
                raise ValueError(f"candidate {c} has {len(decs)} decisions > stride {S}")
            row = out[c]
            for i, (f, d) in enumerate(decs):
                r = row[i]
                r["func"] = idx[f]
                r["kind"] = KIND_CODE[d.kind]
                r["consumer"] = idx[d.consumer] if d.consumer is not None else 0xFFFF
                flags = 0
                if d.serial is not None:
                    flags |= 1
                    if max(d.serial) > 255 or len(d.serial) > MAX_NDIM:
                        raise ValueError("serial extents must be <= 255 (16-byte records)")
                    r["serial"][:len(d.serial)] = d.serial
                if d.thread is not None:
                    flags |= 2
                    if max(d.thread) > 255 or len(d.thread) > MAX_NDIM:
                        raise ValueError("thread extents must be <= 255 (16-byte records)")
                    r["thread"][:len(d.thread)] = d.thread
                r["flags"] = flags
        return out

    def row_keys(self, keys) -> list:
        """Device row keys (func << 8 | stage) -> reference (func, stage) keys."""
        return [(self.names[int(k) >> 8], int(k) & 255) for k in keys]
