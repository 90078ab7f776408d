"""One beam-search phase cut as a replayable CUDA graph.

`StepPlan.run` (shard.py) is the cut the search and the bench call; it reads
the representative count back to the host once, between K4 and K5.  This
module issues the same kernels in the same order with every count kept on
the device, from static buffers and caller-sized workspaces, so the whole
phase — K3 at the pass depth (and the memo depths), K1 + prune, K2, K4
buckets + representatives, K5 penalty / Gumbel / tie-banded cut / bottom-half
flags — is captured once and replayed per batch of the same size with no
host round trip (`gs_featurize_ws`, `gs_struct_hash_ws`,
`gs_beam_topk_reps`: none of them allocates or synchronizes).

The host reads the results after a replay (`result()`): beam, costs,
representatives, drawn rejects and the memo hashes of the bottom half
(reference search.py:127-201 semantics; checked bit for bit against
StepPlan and the C5 reference fixture in tests/test_gpu_graph.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .descriptor import PRUNE_REASONS
from .engine import TIE_BAND
from .shard import flagged_tensor

_U64 = 0xFFFFFFFFFFFFFFFF


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


class CapturedStep:
    """Static-shape phase cut over `n` candidates of `S` records each.

    pass_index, phase_seed, beam, penalty, num_passes, temperature and the
    pass-depth flagged hashes are fixed at construction (they are kernel
    arguments baked into the graph)."""

    def __init__(self, scorer, n, S, pass_index, phase_seed, beam, penalty, num_passes,
                 flagged=None, temperature=0.0, tie_band=TIE_BAND):
        sc = self.sc = scorer
        lib = self.lib = sc.lib
        dev = sc.device
        self.n, self.S, self.R = n, S, sc.R
        self.pass_index, self.phase_seed, self.beam = pass_index, phase_seed, beam
        self.penalty, self.num_passes, self.temperature, self.tie_band = penalty, num_passes, temperature, tie_band
        self.flagged = flagged_tensor(flagged, dev)
        e = lambda shape, dt: torch.empty(shape, dtype=dt, device=dev)  # noqa: E731
        self.dec = torch.zeros((n, S * 16), dtype=torch.uint8, device=dev)
        # K3: pass depth + memo depths 1..min(num_passes, 3) (deeper keys cap at 3)
        self.depths = sorted({pass_index} | set(range(1, min(num_passes, 3) + 1)))
        self.H = e((len(self.depths), n), torch.int64)   # one K3 pass, every depth
        self.hash = {d: self.H[i] for i, d in enumerate(self.depths)}
        self._depths_c = (C.c_int * len(self.depths))(*self.depths)
        self.hws_b = lib.gs_struct_hash_workspace_bytes(n)
        self.hws = e((self.hws_b,), torch.uint8)
        # K1 (reuse mode 2: computed rows only; K2 gathers through row_src)
        self.feats = e((n, self.R, 56), torch.float64)
        self.row_key = e((n, self.R), torch.int32)
        self.n_rows = e((n,), torch.int32)
        self.verdict = e((n,), torch.uint8)
        self.row_src = e((n, self.R), torch.int32)
        prev = sc.reuse_mode
        sc.set_reuse(2)
        self.fws_b = lib.gs_featurize_workspace_bytes(sc.handle, n, S, 0)
        sc.set_reuse(prev)
        if self.fws_b < 0:
            raise _lib.GsError("gs_featurize_workspace_bytes failed")
        self.fws = e((max(1, self.fws_b),), torch.uint8)
        # K2
        self.total = e((n,), torch.float64)
        self.row_cost = e((n, self.R), torch.float64)
        # K4
        self.sws_b = lib.gs_select_workspace_bytes(n)
        self.sws = e((self.sws_b,), torch.uint8)
        self.rep = e((max(1, n),), torch.int64)
        self.rej = e((max(1, n),), torch.int64)
        self.cnt = torch.zeros((2,), dtype=torch.int64, device=dev)
        # K5
        self.k = max(1, min(beam, n))
        self.tws_b = lib.gs_topk_workspace_bytes(n)
        self.tws = e((self.tws_b,), torch.uint8)
        self.pos = e((self.k,), torch.int64)
        self.kcnt = torch.zeros((1,), dtype=torch.int64, device=dev)
        self.bottom = torch.zeros((max(1, n),), dtype=torch.uint8, device=dev)
        self.graph = None

    def _launch(self):
        sc, lib = self.sc, self.lib
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        h = sc.handle
        _lib.check(lib.gs_struct_hash_depths_ws(h, _p(self.dec), self.n, self.S, len(self.depths),
                                                C.cast(self._depths_c, C.c_void_p), _p(self.H), _p(self.hws),
                                                self.hws_b, st))
        prev = sc.reuse_mode
        sc.set_reuse(2)
        try:
            _lib.check(lib.gs_featurize_ws(h, _p(self.dec), self.n, self.S, _p(self.feats), _p(self.row_key),
                                           _p(self.n_rows), _p(self.verdict), _p(self.row_src), 0, _p(self.fws),
                                           self.fws_b, st))
        finally:
            sc.set_reuse(prev)
        _lib.check(lib.gs_cost(h, _p(self.feats), _p(self.row_key), _p(self.n_rows), _p(self.row_src), self.n,
                               _p(self.total), _p(self.row_cost), C.c_void_p(0), st))
        ph = self.hash[self.pass_index]
        _lib.check(lib.gs_select_reps(_p(ph), _p(self.verdict), self.n, C.c_uint64(self.phase_seed & _U64),
                                      _p(self.sws), self.sws_b, _p(self.rep), C.c_void_p(self.cnt.data_ptr()),
                                      _p(self.rej), C.c_void_p(self.cnt.data_ptr() + 8), st))
        fl = self.flagged
        _lib.check(lib.gs_beam_topk_reps(_p(self.total), _p(ph), _p(self.rep), self.n,
                                         C.c_void_p(self.cnt.data_ptr()), _p(fl), 0 if fl is None else fl.numel(),
                                         float(self.penalty), float(self.temperature),
                                         C.c_uint64(self.phase_seed & _U64), self.k, float(self.tie_band),
                                         _p(self.tws), self.tws_b, _p(self.pos), _p(self.kcnt), _p(self.bottom), st))

    def capture(self):
        """Warm up once eagerly (first-use kernel attributes), then capture."""
        s = torch.cuda.Stream(device=self.sc.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self._launch()
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._launch()
        return self

    def replay(self, dec=None):
        """Run the captured phase on `dec` (uint8 [n, S*16], copied into the
        static input) or on whatever the static input holds."""
        if dec is not None:
            if tuple(dec.shape) != tuple(self.dec.shape):
                raise ValueError(f"batch shape {tuple(dec.shape)} != captured {tuple(self.dec.shape)}")
            self.dec.copy_(dec, non_blocking=True)
        if self.graph is None:
            self._launch()
        else:
            self.graph.replay()

    def result(self):
        """Host-side results of the last replay (synchronizes)."""
        self.sc.check()
        kk = int(self.kcnt.item())
        if kk < 0:
            raise _lib.GsError("beam_topk: a tie group is wider than the cut window")
        nrep, nrej = (int(x) for x in self.cnt.cpu().tolist())
        reps = self.rep[:nrep]
        pos = self.pos[:kk]
        beam_idx = reps.index_select(0, pos)
        out = {"beam": beam_idx.cpu().tolist(),
               "beam_costs": self.total.index_select(0, beam_idx).cpu().tolist(),
               "reps": reps, "n_reps": nrep, "total": self.total, "verdict": self.verdict}
        ridx = self.rej[:nrej]
        codes = self.verdict.index_select(0, ridx).cpu().numpy()
        out["rejects"] = [(int(i), PRUNE_REASONS[int(c) - 1]) for i, c in zip(ridx.cpu().numpy(), codes)]
        memo = []
        if nrep > 1:
            bsel = reps.index_select(0, torch.nonzero(self.bottom[:nrep]).flatten())
            for depth in range(1, self.num_passes + 1):
                memo.append(self.hash[min(depth, 3)].index_select(0, bsel))
        out["memo"] = memo
        return out


def memo_set(memo):
    """{(depth, hash)} of a result's memo hashes."""
    return {(depth, int(x)) for depth, hs in enumerate(memo, start=1) for x in hs.cpu().numpy().view(np.uint64)}
