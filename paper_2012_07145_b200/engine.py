"""Device-side scoring engine: one object per (pipeline, machine, thresholds).

Thin stream-ordered wrappers around the C ABI.  Device memory and streams
come from PyTorch (plumbing only); all arithmetic happens in the sm_100a
kernels of libgs_sched.so.  Nothing here falls back to a CPU path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .descriptor import DECISION_DTYPE, PackedPipeline
from .params import DEFAULT_THRESHOLDS, MachineParams

NF = 56
# Relative gap under which adjacent cut keys fall into one band group and
# keep representative order (see csrc/select.cu cut_kernel).  Our fp64 totals
# sit within a few ulp (~1e-15 relative) of the reference's; its exact ties
# between permuted per-stage cost multisets are rounding coincidences we
# cannot reproduce bit for bit, so two keys the reference ties may differ by
# up to twice that here.  The band is a small multiple of it.
TIE_BAND = 1e-14


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class Scorer:
    """Featurize, cost, hash, bucket and cut candidate batches on one GPU."""

    def __init__(self, graph, params=None, thresholds=None, weights=None, device=None):
        if not torch.cuda.is_available():
            raise _lib.GsError("no CUDA device: the scoring path runs only on the GPU")
        self.lib = _lib.load()
        self.device = torch.device(device or "cuda")
        self.params = params or MachineParams()
        self.thresholds = thresholds or DEFAULT_THRESHOLDS
        self.packed = PackedPipeline(graph, self.params, self.thresholds)
        self.handle = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.gs_pipeline_create(C.byref(self.packed.desc), C.byref(self.handle)))
        self.R = max(1, self.lib.gs_pipeline_max_rows(self.handle))
        pf, po, pc, porder = self._placement = self.packed.placement_info()
        _lib.check(self.lib.gs_set_placement_info(self.handle, C.c_void_p(pf.ctypes.data),
                                                  C.c_void_p(po.ctypes.data), C.c_void_p(pc.ctypes.data),
                                                  C.c_void_p(porder.ctypes.data), len(porder)))
        self.S = max(1, self.packed.max_decisions())
        self._weights_key = None
        self.reuse_mode = 1   # gs_set_reuse default
        if weights is not None:
            self.set_weights(weights)

    def __del__(self):
        try:
            if self.handle:
                self.lib.gs_pipeline_destroy(self.handle)
        except Exception:
            pass

    def set_reuse(self, enable):
        """Exact sibling reuse in K1 (see gs_set_reuse in include/gs_sched.h):
        False/True, or 2 = reuse with only the computed rows materialised."""
        mode = enable if isinstance(enable, int) and not isinstance(enable, bool) else int(bool(enable))
        _lib.check(self.lib.gs_set_reuse(self.handle, mode))
        self.reuse_mode = mode

    # -- weights --------------------------------------------------------------
    def set_weights(self, weights):
        """Upload the cost-model weights when their CONTENT changed (the
        reference evaluator reads `.weights` on every call, search.py:117,
        so in-place updates must be seen too; a 66 KB digest per call)."""
        t = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in weights.tensors.items()}
        import hashlib
        hsh = hashlib.blake2b(digest_size=16)
        for name in sorted(t):
            hsh.update(name.encode())
            hsh.update(str(t[name].shape).encode())
            hsh.update(t[name].tobytes())
        key = hsh.digest()
        if key == self._weights_key:
            return
        E, H = t["algo_b"].shape[0], t["head_b"].shape[0]
        arrs = [t[n] for n in ("algo_w", "algo_b", "sched_w", "sched_b", "head_w", "head_b",
                               "out_w", "out_b")]
        with torch.cuda.device(self.device):
            _lib.check(self.lib.gs_set_weights(self.handle, E, H,
                                               *[C.c_void_p(a.ctypes.data) for a in arrs]))
        self._weights_key = key
        self._weights_ref = weights

    # -- inputs ---------------------------------------------------------------
    def upload(self, candidates, pin=False) -> torch.Tensor:
        arr = self.packed.pack(candidates, self.S)
        return self.to_device(arr, pin)

    def to_device(self, arr: np.ndarray, pin=False) -> torch.Tensor:
        assert arr.dtype == DECISION_DTYPE
        host = torch.from_numpy(arr.view(np.uint8).reshape(arr.shape[0], -1))
        if pin:
            host = host.pin_memory()
        return host.to(self.device, non_blocking=pin)

    # -- K1 -------------------------------------------------------------------
    def prune(self, dec: torch.Tensor) -> torch.Tensor:
        """Resolve + prune verdicts only (K1 without feature rows)."""
        n = dec.shape[0]
        verdict = torch.empty((n,), dtype=torch.uint8, device=self.device)
        nrows = torch.empty((n,), dtype=torch.int32, device=self.device)
        _lib.check(self.lib.gs_featurize(self.handle, _ptr(dec), n, dec.shape[1] // 16, C.c_void_p(0),
                                         C.c_void_p(0), _ptr(nrows), _ptr(verdict), C.c_void_p(0), _stream()))
        return verdict

    def featurize(self, dec: torch.Tensor, out=None):
        n = dec.shape[0]
        S = dec.shape[1] // 16
        if out is None:
            out = dict(
                feats=torch.empty((n, self.R, NF), dtype=torch.float64, device=self.device),
                row_key=torch.empty((n, self.R), dtype=torch.int32, device=self.device),
                n_rows=torch.empty((n,), dtype=torch.int32, device=self.device),
                verdict=torch.empty((n,), dtype=torch.uint8, device=self.device),
                row_src=torch.empty((n, self.R), dtype=torch.int32, device=self.device))
        _lib.check(self.lib.gs_featurize(self.handle, _ptr(dec), n, S, _ptr(out["feats"]),
                                         _ptr(out["row_key"]), _ptr(out["n_rows"]),
                                         _ptr(out["verdict"]), _ptr(out.get("row_src")), _stream()))
        out["rows_only"] = self.reuse_mode == 2
        return out

    def stats(self):
        """K1 work counters since the last call (see gs_stats)."""
        out = np.zeros(6, dtype=np.int64)
        _lib.check(self.lib.gs_stats(self.handle, C.c_void_p(out.ctypes.data), _stream()))
        d = dict(zip(("candidates", "incremental", "rows_computed", "rows", "geometries"), out[:5].tolist()))
        d["k1_warps"], d["k1_slice_bytes"] = int(out[5]) >> 32, int(out[5]) & 0xFFFFFFFF
        return d

    def check(self):
        """Synchronize and raise on any device-side capacity / schedule error."""
        _lib.check(self.lib.gs_check(self.handle, _stream()))

    # -- K2 -------------------------------------------------------------------
    def cost(self, f, rows=False, basis=False, total=None, reuse=None, scratch=None):
        """Totals (and optionally per-row costs / basis) of a featurized batch.

        reuse (default: when `f` carries K1's row_src and no basis is asked
        for) evaluates the network once per distinct row; `scratch` is an
        optional preallocated [N, R] fp64 row-cost buffer for that mode."""
        n = f["feats"].shape[0]
        if total is None:
            total = torch.empty((n,), dtype=torch.float64, device=self.device)
        src = f.get("row_src")
        if reuse is None:
            reuse = src is not None and not basis
        if not reuse:
            src = None
        if f.get("rows_only") and src is None:
            raise ValueError("features from reuse mode 2 hold only the computed rows: cost them with row_src")
        rc = None
        if rows or src is not None:
            rc = scratch if scratch is not None else torch.empty((n, self.R), dtype=torch.float64,
                                                                 device=self.device)
        gh = torch.empty((n, self.R, 31), dtype=torch.float64, device=self.device) if basis else None
        if src is not None and not rows and not basis:
            # totals only: the non-computed rows' costs are not written back
            _lib.check(self.lib.gs_cost_totals(self.handle, _ptr(f["feats"]), _ptr(f["row_key"]),
                                               _ptr(f["n_rows"]), _ptr(src), n, _ptr(total), _ptr(rc),
                                               _stream()))
            return total, None, None
        _lib.check(self.lib.gs_cost(self.handle, _ptr(f["feats"]), _ptr(f["row_key"]), _ptr(f["n_rows"]),
                                    _ptr(src), n, _ptr(total), _ptr(rc), _ptr(gh), _stream()))
        return total, (rc if rows else None), gh

    # -- K3 -------------------------------------------------------------------
    def struct_hash(self, dec: torch.Tensor, depth: int, out=None):
        if depth < 0:
            raise ValueError("depth must be >= 0")
        n = dec.shape[0]
        if out is None:
            out = torch.empty((n,), dtype=torch.int64, device=self.device)
        _lib.check(self.lib.gs_struct_hash(self.handle, _ptr(dec), n, dec.shape[1] // 16, depth,
                                           _ptr(out), _stream()))
        return out

    def struct_hash_depths(self, dec: torch.Tensor, depths):
        """K3 at several depths in one pass (gs_struct_hash_depths_ws):
        int64 [len(depths), N], row k = depth depths[k]."""
        depths = [int(d) for d in depths]
        if not 1 <= len(depths) <= 4 or min(depths) < 0:
            raise ValueError("1..4 depths, each >= 0")
        n = dec.shape[0]
        out = torch.empty((len(depths), n), dtype=torch.int64, device=self.device)
        wsb = self.lib.gs_struct_hash_workspace_bytes(n)
        ws = torch.empty((wsb,), dtype=torch.uint8, device=self.device)
        d = (C.c_int * len(depths))(*depths)
        _lib.check(self.lib.gs_struct_hash_depths_ws(self.handle, _ptr(dec), n, dec.shape[1] // 16, len(depths),
                                                     C.cast(d, C.c_void_p), _ptr(out), _ptr(ws), wsb, _stream()))
        return out

    def memo_hashes(self, dec: torch.Tensor, num_passes: int, h3=None):
        """Hashes at depths 1..num_passes (the bad-hash memo, search.py:196-200).
        The canonical key caps the depth at 3 (loopnest.py:137), so deeper
        depths reuse the depth-3 hashes (`h3`, when the caller has them)."""
        out = []
        for depth in range(1, num_passes + 1):
            if depth >= 3:
                h3 = self.struct_hash(dec, 3) if h3 is None else h3
                out.append(h3)
            else:
                out.append(self.struct_hash(dec, depth))
        return out

    # -- machine oracle (K6) -------------------------------------------------
    def simulate(self, dec: torch.Tensor, params=None):
        """Reference `simulate_runtime` (machine.py:108-167) for a batch of
        fully scheduled candidates: K1 features and row kernels, then K6.
        Returns (runtime f64 [N], spill_bytes i64 [N], status u8 [N]) with
        status 0 ok, 1 hardware-limit violation, 2 not fully scheduled (the
        two cases the reference raises ValueError for; runtime is NaN)."""
        from .descriptor import oracle_params
        n, S = dec.shape[0], dec.shape[1] // 16
        op = oracle_params(params or self.params)
        rt = torch.empty((n,), dtype=torch.float64, device=self.device)
        sp = torch.empty((n,), dtype=torch.int64, device=self.device)
        st = torch.empty((n,), dtype=torch.uint8, device=self.device)
        _lib.check(self.lib.gs_simulate(self.handle, _ptr(dec), n, S, C.byref(op), _ptr(rt), _ptr(sp), _ptr(st),
                                        _stream()))
        return rt, sp, st

    # -- beam-step expansion -------------------------------------------------
    def expand_step(self, parents: torch.Tensor, steps: torch.Tensor, menus=None, total=None):
        """Every phase-2 tiling of each parent's step root on the device
        (search.py:223-235).  parents: uint8 [P, S*16] decision records on the
        device; steps: int32 [P] record index of each parent's step root.
        Returns (records [N, S*16], owner int32 [N], offsets int64 [P+1]).
        `total` (N) skips the sizing pass when already known."""
        from .descriptor import tiling_menus
        from .gen import Menus
        P, S = parents.shape[0], parents.shape[1] // 16
        m = tiling_menus(menus or Menus)
        wsb = self.lib.gs_expand_workspace_bytes(P)
        ws = torch.empty((max(1, wsb),), dtype=torch.uint8, device=self.device)
        offsets = torch.empty((P + 1,), dtype=torch.int64, device=self.device)
        if total is None:
            _lib.check(self.lib.gs_expand_step(self.handle, _ptr(parents), P, S, _ptr(steps), C.byref(m),
                                               _ptr(offsets), _ptr(ws), wsb, C.c_void_p(0), 0, C.c_void_p(0),
                                               _stream()))
            total = int(offsets[-1].item())
        out = torch.empty((total, S * 16), dtype=torch.uint8, device=self.device)
        owner = torch.empty((max(1, total),), dtype=torch.int32, device=self.device)
        _lib.check(self.lib.gs_expand_step(self.handle, _ptr(parents), P, S, _ptr(steps), C.byref(m),
                                           _ptr(offsets), _ptr(ws), wsb, _ptr(out), total, _ptr(owner),
                                           _stream()))
        return out, owner[:total], offsets

    def expand_phase1(self, parents: torch.Tensor, func: str, restrict=None, menus=None, total=None):
        """Every phase-1 candidate of each parent for `func` on the device
        (search.py:204-220 `_phase1_candidates`): parents uint8 [P, S*16];
        restrict: the SearchConfig.restrict_placements kinds (None = all).
        Returns (records [N, S*16], owner int32 [N], offsets int64 [P+1])."""
        from .descriptor import KIND_CODE, tiling_menus
        from .gen import Menus
        P, S = parents.shape[0], parents.shape[1] // 16
        fi = self.packed.index[func]
        mask = 0xF if restrict is None else sum(1 << KIND_CODE[k] for k in set(restrict))
        m = tiling_menus(menus or Menus)
        wsb = self.lib.gs_phase1_workspace_bytes(P)
        ws = torch.empty((max(1, wsb),), dtype=torch.uint8, device=self.device)
        offsets = torch.empty((P + 1,), dtype=torch.int64, device=self.device)
        if total is None:
            _lib.check(self.lib.gs_expand_phase1(self.handle, _ptr(parents), P, S, fi, mask, C.byref(m),
                                                 _ptr(offsets), _ptr(ws), wsb, C.c_void_p(0), 0, C.c_void_p(0),
                                                 _stream()))
            total = int(offsets[-1].item())
        out = torch.empty((total, S * 16), dtype=torch.uint8, device=self.device)
        owner = torch.empty((max(1, total),), dtype=torch.int32, device=self.device)
        _lib.check(self.lib.gs_expand_phase1(self.handle, _ptr(parents), P, S, fi, mask, C.byref(m), _ptr(offsets),
                                             _ptr(ws), wsb, _ptr(out), total, _ptr(owner), _stream()))
        return out, owner[:total], offsets

    def random_schedules(self, n: int, seed: int, first: int = 0, menus=None) -> torch.Tensor:
        """n complete random schedules generated on the device; candidate i
        equals the reference `_random_schedule(graph, default_rng((seed,
        first + i)))` (tests/test_acceptance.py:136-160).  Returns uint8
        [n, S*16] decision records."""
        from .descriptor import tiling_menus
        from .gen import Menus
        m = tiling_menus(menus or Menus)
        out = torch.empty((n, self.S * 16), dtype=torch.uint8, device=self.device)
        _lib.check(self.lib.gs_random_schedules(self.handle, C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), first, n, self.S,
                                                C.byref(m), _ptr(out), _stream()))
        return out

    # -- K4 -------------------------------------------------------------------
    def select(self, hashes: torch.Tensor, verdict: torch.Tensor, phase_seed: int, rejects=True):
        n = hashes.shape[0]
        wsb = self.lib.gs_select_workspace_bytes(n)
        ws = torch.empty((wsb,), dtype=torch.uint8, device=self.device)
        rep = torch.empty((max(1, n),), dtype=torch.int64, device=self.device)
        rej = torch.empty((max(1, n),), dtype=torch.int64, device=self.device) if rejects else None
        cnt = torch.zeros((2,), dtype=torch.int64, device=self.device)
        _lib.check(self.lib.gs_select_reps(_ptr(hashes), _ptr(verdict), n,
                                           C.c_uint64(phase_seed & 0xFFFFFFFFFFFFFFFF), _ptr(ws), wsb,
                                           _ptr(rep), C.c_void_p(cnt.data_ptr()), _ptr(rej),
                                           C.c_void_p(cnt.data_ptr() + 8), _stream()))
        return rep, rej, cnt

    # -- K5 -------------------------------------------------------------------
    def beam_topk(self, costs, pass_hash, flagged, penalty, temperature, phase_seed, k,
                  bottom=True, tie_band=TIE_BAND):
        """K5 (search.py:76-87, 168-201).  Returns (positions [k] in cut
        order, count (device int64; negative if a tie group was wider than
        the cut window), bottom-half flags u8 [n] or None)."""
        n = costs.shape[0]
        wsb = self.lib.gs_topk_workspace_bytes(n)
        ws = torch.empty((wsb,), dtype=torch.uint8, device=self.device)
        pos = torch.empty((max(1, min(k, n)),), dtype=torch.int64, device=self.device)
        cnt = torch.zeros((1,), dtype=torch.int64, device=self.device)
        bot = torch.empty((max(1, n),), dtype=torch.uint8, device=self.device) if bottom else None
        fl = flagged if flagged is not None and flagged.numel() else None
        _lib.check(self.lib.gs_beam_topk(_ptr(costs), _ptr(pass_hash), n, _ptr(fl),
                                         0 if fl is None else fl.numel(), float(penalty),
                                         float(temperature),
                                         C.c_uint64(phase_seed & 0xFFFFFFFFFFFFFFFF), k,
                                         float(tie_band), _ptr(ws),
                                         wsb, _ptr(pos), _ptr(cnt), _ptr(bot), _stream()))
        return pos, cnt, bot


    def beam_topk_reps(self, total, pass_hash, rep, n_max, cnt, flagged, penalty, temperature, phase_seed, k,
                       tie_band=TIE_BAND):
        """K5 over K4's representatives without a host round trip
        (gs_beam_topk_reps): costs and pass hashes are the per-candidate
        arrays, `rep` the representative list and cnt[0] its device-side
        length.  Returns (positions into `rep` in cut order, count (device),
        bottom-half flags over the representative positions)."""
        wsb = self.lib.gs_topk_workspace_bytes(n_max)
        ws = torch.empty((wsb,), dtype=torch.uint8, device=self.device)
        pos = torch.empty((max(1, k),), dtype=torch.int64, device=self.device)
        kcnt = torch.zeros((1,), dtype=torch.int64, device=self.device)
        bot = torch.zeros((max(1, n_max),), dtype=torch.uint8, device=self.device)
        fl = flagged if flagged is not None and flagged.numel() else None
        _lib.check(self.lib.gs_beam_topk_reps(_ptr(total), _ptr(pass_hash), _ptr(rep), n_max,
                                              C.c_void_p(cnt.data_ptr()), _ptr(fl),
                                              0 if fl is None else fl.numel(), float(penalty), float(temperature),
                                              C.c_uint64(phase_seed & 0xFFFFFFFFFFFFFFFF), k, float(tie_band),
                                              _ptr(ws), wsb, _ptr(pos), _ptr(kcnt), _ptr(bot), _stream()))
        return pos, kcnt, bot


def u64_sorted_tensor(values, device) -> torch.Tensor:
    """Sorted uint64 values as an int64 tensor holding the same bits."""
    arr = np.array(sorted(int(v) & 0xFFFFFFFFFFFFFFFF for v in values), dtype=np.uint64)
    return torch.from_numpy(arr.view(np.int64)).to(device)


def as_u64(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)
