"""`torch.ops.gsched.*`: the C-ABI entry points registered as PyTorch custom
operators, each with a fake (meta) kernel for shape inference.

The reference has no operator layer (its seam is Python); the
north star asks for the Python cost-model / featurizer surface to reach the
GPU through PyTorch-registered custom ops over the thin C-ABI.  These are
those ops.  They are functional (fresh outputs, no data-dependent shapes:
counts come back as device scalars), so they can be traced, captured in CUDA
graphs and checked with `torch.library.opcheck`.

The pipeline handle (a `Scorer`) is passed as its integer address
(`Scorer.handle.value`); the ops are registered for CUDA only, so a CPU
tensor fails at dispatch — there is no CPU fallback.

| op | C-ABI (include/gs_sched.h) | reference interface it replaces |
|---|---|---|
| featurize    | gs_featurize          | featurize.py:275-303 + options.py:200-255 |
| cost         | gs_cost               | search.py:115-124 (CostEvaluator.cost) |
| struct_hash  | gs_struct_hash        | loopnest.py:131-165, 254 |
| select_reps  | gs_select_reps        | sampling.py:45-59, search.py:127-165 |
| beam_topk    | gs_beam_topk_reps     | search.py:76-87, 168-201 |
| expand_step  | gs_expand_step        | search.py:223-235 |
"""

from __future__ import annotations

import ctypes as C

import torch
from torch import Tensor

from . import _lib

NF = 56
_U64 = 0xFFFFFFFFFFFFFFFF


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _h(handle: int):
    if not handle:
        raise _lib.GsError("null pipeline handle")
    return C.c_void_p(handle)


def _st():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise _lib.GsError("gsched ops run only on CUDA tensors (no CPU fallback)")


# ---------------------------------------------------------------- featurize --
@torch.library.custom_op("gsched::featurize", mutates_args=(), device_types="cuda")
def featurize(handle: int, dec: Tensor, R: int, reuse: int) -> tuple[Tensor, Tensor, Tensor, Tensor, Tensor]:
    """K1: (feats f64 [N, R, 56], row_key i32 [N, R], n_rows i32 [N],
    verdict u8 [N], row_src i32 [N, R]).  reuse 0/1 write every row; 2 only
    the computed ones (see gs_set_reuse)."""
    _need_cuda(dec)
    lib = _lib.load()
    n, S = dec.shape[0], dec.shape[1] // 16
    dev = dec.device
    # zero-filled: rows past n_rows (and, in reuse mode 2, repeated rows)
    # are not written by K1, and a functional op's outputs must be defined
    feats = torch.zeros((n, R, NF), dtype=torch.float64, device=dev)
    row_key = torch.zeros((n, R), dtype=torch.int32, device=dev)
    n_rows = torch.empty((n,), dtype=torch.int32, device=dev)
    verdict = torch.empty((n,), dtype=torch.uint8, device=dev)
    row_src = torch.zeros((n, R), dtype=torch.int32, device=dev)
    h = _h(handle)
    prev = lib.gs_get_reuse(h)
    _lib.check(lib.gs_set_reuse(h, reuse))
    try:
        _lib.check(lib.gs_featurize(h, _p(dec), n, S, _p(feats), _p(row_key), _p(n_rows), _p(verdict),
                                    _p(row_src), _st()))
    finally:
        lib.gs_set_reuse(h, prev)   # the handle's mode is the caller's state: restore it
    return feats, row_key, n_rows, verdict, row_src


@featurize.register_fake
def _(handle, dec, R, reuse):
    n = dec.shape[0]
    return (dec.new_empty((n, R, NF), dtype=torch.float64), dec.new_empty((n, R), dtype=torch.int32),
            dec.new_empty((n,), dtype=torch.int32), dec.new_empty((n,), dtype=torch.uint8),
            dec.new_empty((n, R), dtype=torch.int32))


# --------------------------------------------------------------------- cost --
@torch.library.custom_op("gsched::cost", mutates_args=(), device_types="cuda")
def cost(handle: int, feats: Tensor, row_key: Tensor, n_rows: Tensor, row_src: Tensor | None,
         basis: bool = False) -> tuple[Tensor, Tensor, Tensor]:
    """K2: (total f64 [N], row_cost f64 [N, R], basis f64 [N, R, 31] = g[30], h
    when `basis`, else an empty [0, R, 31]).  With row_src (and no basis) the
    network runs once per distinct row; every row's cost is still returned."""
    _need_cuda(feats, row_key, n_rows, row_src)
    lib = _lib.load()
    n, R = feats.shape[0], feats.shape[1]
    total = torch.empty((n,), dtype=torch.float64, device=feats.device)
    rc = torch.zeros((n, R), dtype=torch.float64, device=feats.device)   # rows past n_rows stay 0
    gh = torch.zeros((n if basis else 0, R, 31), dtype=torch.float64, device=feats.device)
    _lib.check(lib.gs_cost(_h(handle), _p(feats), _p(row_key), _p(n_rows), None if basis else _p(row_src), n,
                           _p(total), _p(rc), _p(gh) if basis else C.c_void_p(0), _st()))
    return total, rc, gh


@cost.register_fake
def _(handle, feats, row_key, n_rows, row_src, basis=False):
    n, R = feats.shape[0], feats.shape[1]
    return feats.new_empty((n,)), feats.new_empty((n, R)), feats.new_empty((n if basis else 0, R, 31))


# -------------------------------------------------------------- struct_hash --
@torch.library.custom_op("gsched::struct_hash", mutates_args=(), device_types="cuda")
def struct_hash(handle: int, dec: Tensor, depth: int) -> Tensor:
    """K3: blake2b-64 structural hash per candidate (uint64 bits in int64)."""
    _need_cuda(dec)
    if depth < 0:
        raise ValueError("depth must be >= 0")
    lib = _lib.load()
    n, S = dec.shape[0], dec.shape[1] // 16
    out = torch.empty((n,), dtype=torch.int64, device=dec.device)
    wsb = lib.gs_struct_hash_workspace_bytes(n)
    ws = torch.empty((wsb,), dtype=torch.uint8, device=dec.device)
    _lib.check(lib.gs_struct_hash_ws(_h(handle), _p(dec), n, S, depth, _p(out), _p(ws), wsb, _st()))
    return out


@struct_hash.register_fake
def _(handle, dec, depth):
    return dec.new_empty((dec.shape[0],), dtype=torch.int64)


# -------------------------------------------------------------- select_reps --
@torch.library.custom_op("gsched::select_reps", mutates_args=(), device_types="cuda")
def select_reps(hashes: Tensor, verdict: Tensor, phase_seed: int) -> tuple[Tensor, Tensor, Tensor]:
    """K4: (rep_idx i64 [N], rej_idx i64 [N], counts i64 [2] = (n_reps,
    n_rejects)); the first counts[0] / counts[1] entries are valid."""
    _need_cuda(hashes, verdict)
    lib = _lib.load()
    n = hashes.shape[0]
    dev = hashes.device
    wsb = lib.gs_select_workspace_bytes(n)
    ws = torch.empty((wsb,), dtype=torch.uint8, device=dev)
    rep = torch.full((max(1, n),), -1, dtype=torch.int64, device=dev)   # entries past the counts: -1
    rej = torch.full((max(1, n),), -1, dtype=torch.int64, device=dev)
    cnt = torch.zeros((2,), dtype=torch.int64, device=dev)
    _lib.check(lib.gs_select_reps(_p(hashes), _p(verdict), n, C.c_uint64(phase_seed & _U64), _p(ws), wsb, _p(rep),
                                  C.c_void_p(cnt.data_ptr()), _p(rej), C.c_void_p(cnt.data_ptr() + 8), _st()))
    return rep, rej, cnt


@select_reps.register_fake
def _(hashes, verdict, phase_seed):
    n = hashes.shape[0]
    m = torch.sym_max(1, n)
    return (hashes.new_empty((m,), dtype=torch.int64), hashes.new_empty((m,), dtype=torch.int64),
            hashes.new_empty((2,), dtype=torch.int64))


# ---------------------------------------------------------------- beam_topk --
@torch.library.custom_op("gsched::beam_topk", mutates_args=(), device_types="cuda")
def beam_topk(costs: Tensor, pass_hash: Tensor, rep_idx: Tensor, n_reps: Tensor, flagged: Tensor | None,
              penalty: float, temperature: float, phase_seed: int, k: int,
              tie_band: float) -> tuple[Tensor, Tensor, Tensor]:
    """K5 over the representatives K4 selected (costs / pass_hash per
    candidate, rep_idx + device count n_reps from select_reps): (positions
    i64 [k] in cut order, count i64 [1] (negative: a tie group wider than
    the cut window), bottom-half flags u8 [len(rep_idx)])."""
    _need_cuda(costs, pass_hash, rep_idx, n_reps, flagged)
    lib = _lib.load()
    m = rep_idx.shape[0]
    dev = costs.device
    wsb = lib.gs_topk_workspace_bytes(m)
    ws = torch.empty((wsb,), dtype=torch.uint8, device=dev)
    pos = torch.full((k,), -1, dtype=torch.int64, device=dev)   # entries past the count: -1
    cnt = torch.zeros((1,), dtype=torch.int64, device=dev)
    bot = torch.zeros((m,), dtype=torch.uint8, device=dev)
    fl = flagged if flagged is not None and flagged.numel() else None
    _lib.check(lib.gs_beam_topk_reps(_p(costs), _p(pass_hash), _p(rep_idx), m, _p(n_reps), _p(fl),
                                     0 if fl is None else fl.numel(), float(penalty), float(temperature),
                                     C.c_uint64(phase_seed & _U64), min(k, m), float(tie_band), _p(ws), wsb,
                                     _p(pos), _p(cnt), _p(bot), _st()))
    return pos, cnt, bot


@beam_topk.register_fake
def _(costs, pass_hash, rep_idx, n_reps, flagged, penalty, temperature, phase_seed, k, tie_band):
    return (costs.new_empty((k,), dtype=torch.int64), costs.new_empty((1,), dtype=torch.int64),
            costs.new_empty((rep_idx.shape[0],), dtype=torch.uint8))


# -------------------------------------------------------------- expand_step --
@torch.library.custom_op("gsched::expand_step", mutates_args=(), device_types="cuda")
def expand_step(handle: int, parents: Tensor, steps: Tensor, total: int, serial_powers: list[int],
                odd_serial: list[int], innermost_thread: list[int], outer_thread: list[int], unroll_budget: int,
                warp_size: int) -> tuple[Tensor, Tensor, Tensor]:
    """Every phase-2 tiling of each parent's step root: (records u8
    [total, S*16], owner i32 [total], offsets i64 [P+1]).  `total` is the
    caller-known candidate count; a mismatch with the device count raises
    at gs_check (nothing is written past `total`)."""
    _need_cuda(parents, steps)
    from .descriptor import GsTilingMenus
    lib = _lib.load()
    P, S = parents.shape[0], parents.shape[1] // 16
    m = GsTilingMenus()
    for name, vals in (("serial_powers", serial_powers), ("odd_serial", odd_serial),
                       ("innermost_thread", innermost_thread), ("outer_thread", outer_thread)):
        arr = getattr(m, name)
        for i, v in enumerate(vals):
            arr[i] = v
    m.n_serial_powers, m.n_odd_serial = len(serial_powers), len(odd_serial)
    m.n_innermost, m.n_outer = len(innermost_thread), len(outer_thread)
    m.unroll_budget, m.warp_size = unroll_budget, warp_size
    dev = parents.device
    wsb = lib.gs_expand_workspace_bytes(P)
    ws = torch.empty((max(1, wsb),), dtype=torch.uint8, device=dev)
    offsets = torch.empty((P + 1,), dtype=torch.int64, device=dev)
    out = torch.empty((total, S * 16), dtype=torch.uint8, device=dev)
    owner = torch.empty((total,), dtype=torch.int32, device=dev)
    _lib.check(lib.gs_expand_step(_h(handle), _p(parents), P, S, _p(steps), C.byref(m), _p(offsets), _p(ws), wsb,
                                  _p(out), total, _p(owner), _st()))
    return out, owner, offsets


@expand_step.register_fake
def _(handle, parents, steps, total, serial_powers, odd_serial, innermost_thread, outer_thread, unroll_budget,
      warp_size):
    P = parents.shape[0]
    return (parents.new_empty((total, parents.shape[1])), parents.new_empty((total,), dtype=torch.int32),
            parents.new_empty((P + 1,), dtype=torch.int64))


def menu_args(menus=None):
    """The expand_step menu arguments from a `gen.Menus`-like object."""
    from .descriptor import tiling_menus
    from .gen import Menus
    m = tiling_menus(menus or Menus)
    return ([m.serial_powers[i] for i in range(m.n_serial_powers)], [m.odd_serial[i] for i in range(m.n_odd_serial)],
            [m.innermost_thread[i] for i in range(m.n_innermost)], [m.outer_thread[i] for i in range(m.n_outer)],
            m.unroll_budget, m.warp_size)
