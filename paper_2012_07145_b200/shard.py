"""One beam-search phase cut over a candidate batch — the batched
replacement of the reference `_select_representatives` + `_cut`
(pkg/src/gpusched/search.py:127-201) — on one GPU or bucket-sharded over
several (one process per GPU, NCCL over NVLink for the exchange).

`StepPlan.run` is THE cut: `evaluator.gpu_cut` (the `_cut` drop-in the
search calls), the bench and the multi-GPU arm all go through it.

Per phase, on the device:
  K3 hash at the pass depth -> K1 featurize + prune (reuse mode 2: only the
  computed rows are written) -> K2 cost every candidate -> K4 buckets +
  PCG64 representatives (+ the drawn prune rejects) -> K5 penalty for
  memo-flagged hashes, optional Gumbel(T), tie-banded top-k and the
  bottom-half memo flags -> K3 memo hashes of the representatives.
The host syncs once, at the end, to read the beam.

Sharding: every rank holds the batch's decision records and
hashes all of them at the pass depth (cheap).  A structural-hash bucket is
owned by rank `hash % world`, so buckets never straddle ranks; each rank
featurizes, prunes and costs only its buckets' candidates (the expensive
part) and draws their representatives with the same per-bucket PCG64
streams the reference uses.  The ranks then agree on the cut through
`topk_exchange` (see its docstring): fixed-size all-gathers of each rank's
cut window, not of every representative.
"""

from __future__ import annotations

import numpy as np
import torch

from ._lib import GsError
from .descriptor import PRUNE_REASONS

SIGN = -0x8000000000000000  # flips int64 order into uint64 order


def flagged_tensor(flagged, device):
    """Pass-depth flagged hashes as a sorted-as-uint64 int64 tensor (or None)."""
    if flagged is None:
        return None
    if isinstance(flagged, torch.Tensor):
        return flagged.to(device) if flagged.numel() else None
    vals = sorted(int(v) & 0xFFFFFFFFFFFFFFFF for v in flagged)
    if not vals:
        return None
    return torch.from_numpy(np.array(vals, dtype=np.uint64).view(np.int64)).to(device)


class StepPlan:
    """Reusable buffers + the cut of one beam-search phase.

    pass_index / phase_seed / beam / penalty / num_passes / tie_band are the
    reference SearchConfig and `_cut` arguments (search.py:168-201);
    `sampling=False` is the reference test hook that keeps every valid
    candidate (search.py:142-150)."""

    def __init__(self, scorer, n, world, rank, pass_index, phase_seed, beam, penalty, num_passes,
                 tie_band, sampling=True, group=None, reuse=2):
        self.sc, self.n, self.world, self.rank = scorer, n, world, rank
        self.reuse = reuse   # K1 sibling reuse: 2 (computed rows only, the default), 1, or 0 (every row)
        self.pass_index, self.phase_seed, self.beam = pass_index, phase_seed, beam
        self.penalty, self.num_passes, self.tie_band = penalty, num_passes, tie_band
        self.sampling, self.group = sampling, group
        self.fbuf = None
        self.rcbuf = None
        self.local_count = n
        self.last_exchange_bytes = 0

    def _features(self, d):
        # the cut consumes features only through K2 with row_src, so K1
        # writes just the computed rows (reuse mode 2)
        prev = self.sc.reuse_mode
        if prev != self.reuse:
            self.sc.set_reuse(self.reuse)
        try:
            return self._features_into(d)
        finally:
            if prev != self.reuse:
                self.sc.set_reuse(prev)

    def _features_into(self, d):
        m = d.shape[0]
        if self.fbuf is None or self.fbuf["feats"].shape[0] != m:
            self.fbuf = self.rcbuf = None
            self.fbuf = self.sc.featurize(d)
            self.rcbuf = torch.empty((m, self.sc.R), dtype=torch.float64, device=self.sc.device)
        else:
            self.sc.featurize(d, out=self.fbuf)
        return self.fbuf

    def run(self, dec, flagged=None, temperature=0.0, times=None, rejects=False):
        """One phase cut over the decision records `dec` (uint8 [N, S*16] on
        the device).

        flagged: the memo's hashes at this pass depth (`memo.flagged` entries
        with depth == pass_index) — list/set of ints or a sorted uint64-as-
        int64 tensor; temperature: SearchConfig.explore_temperature.
        `times` (optional dict) accumulates device milliseconds per phase:
        hash, featurize (K1), cost (K2), select (K4 + exchange), cut (K5),
        memo (K3 at depths 1..num_passes).

        Returns a dict: beam (candidate indices, cut order), beam_costs
        (unpenalized), reps (candidate indices, the reference's rep order;
        world 1), rejects ([(candidate index, reason)] in draw order, when
        asked), memo (per depth 1..num_passes: int64 tensor of the bottom
        half's hashes), total / verdict (per local candidate, device),
        local (local -> batch candidate index, None on one rank), n_reps."""
        sc = self.sc
        ev = []

        def mark():
            if times is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev.append(e)

        mark()
        # K3 once over the records at the pass depth and every memo depth
        # (1..num_passes; keys cap at depth 3, loopnest.py:137): the memo
        # below gathers the bottom half's hashes instead of re-hashing them
        cap = lambda x: min(x, 3)  # noqa: E731
        depths = [self.pass_index] + sorted({cap(x) for x in range(1, self.num_passes + 1)} - {cap(self.pass_index)})
        H = sc.struct_hash_depths(dec, depths)
        row_of = {cap(x): i for i, x in enumerate(depths)}
        h = H[0]
        if self.world > 1:
            mine = torch.nonzero(torch.remainder(h, self.world) == self.rank).flatten()
            d = dec.index_select(0, mine)
            hl = h.index_select(0, mine)
        else:
            mine, d, hl = None, dec, h
        self.local_count = d.shape[0]
        mark()
        f = self._features(d)
        mark()
        total, _, _ = sc.cost(f, scratch=self.rcbuf, reuse=self.reuse != 0)
        mark()
        verdict = f["verdict"]
        rej = None
        if self.sampling:
            rep, rej, cnt = sc.select(hl, verdict, self.phase_seed, rejects=rejects)
            nrep_t, nrej_t = cnt[0], cnt[1]
        else:   # every valid candidate in order; every invalid one reported
            valid = verdict == 0
            rep = torch.nonzero(valid).flatten()
            rej = torch.nonzero(~valid).flatten() if rejects else None
            nrep_t = torch.tensor(rep.numel(), device=sc.device)
            nrej_t = torch.tensor(0 if rej is None else rej.numel(), device=sc.device)
        fl = flagged_tensor(flagged, sc.device)
        if self.world == 1 and self.sampling and hl.shape[0] > 0:
            # one rank: K5 reads the representative count K4 left on the
            # device (gs_beam_topk_reps), so the GPU goes from K4 to K5
            # without waiting for the host; the count is read once K5 is queued
            mark()
            n_loc = int(hl.shape[0])
            pos, kcnt, bot = sc.beam_topk_reps(total, hl, rep, n_loc, cnt, fl, self.penalty, temperature,
                                               self.phase_seed, max(1, min(self.beam, n_loc)),
                                               tie_band=self.tie_band)
            nrep = int(nrep_t.item())
            rep = rep[:nrep]
            cand = rep
            n_all = nrep
            if n_all:
                kk = int(kcnt.item())
                if kk < 0:
                    raise GsError("beam_topk: a tie group is wider than the cut window")
                beam = rep.index_select(0, pos[:kk])
                beam_costs = total.index_select(0, beam)
            else:
                beam = rep[:0]
                beam_costs = total[:0]
                bot = None
            mem_src = cand
        else:
            nrep = int(nrep_t.item())
            rep = rep[:nrep]
            costs = total.index_select(0, rep)
            ph = hl.index_select(0, rep)
            cand = rep if mine is None else mine.index_select(0, rep)
            mark()
            if self.world > 1:
                from . import exchange
                beam, beam_costs, bot_local, n_global = exchange.sharded_cut(
                    sc, costs, ph, cand, fl, self.penalty, temperature, self.phase_seed, self.beam,
                    self.tie_band, self.world, self.group)
                self.last_exchange_bytes = exchange.LAST_BYTES
                n_all = n_global
                bot = bot_local
            else:
                n_all = int(costs.shape[0])
                if n_all:
                    pos, kcnt, bot = sc.beam_topk(costs, ph, fl, self.penalty, temperature, self.phase_seed,
                                                  min(self.beam, n_all), tie_band=self.tie_band)
                    kk = int(kcnt.item())
                    if kk < 0:
                        raise GsError("beam_topk: a tie group is wider than the cut window")
                    beam = cand.index_select(0, pos[:kk])
                    beam_costs = costs.index_select(0, pos[:kk])
                else:
                    beam = cand[:0]
                    beam_costs = costs[:0]
                    bot = None
            mem_src = cand
        mark()
        # bad-hash memo (search.py:196-200): hashes of the bottom half at
        # every depth a later pass may bucket at.  At depth >= 3 the key
        # caps at 3 (loopnest.py:137), so the pass-depth bucket hashes serve
        # when pass_index >= 3.
        memo = []
        if n_all > 1 and mem_src.numel():
            keep = torch.nonzero(bot[:mem_src.numel()]).flatten()
            bsel = mem_src.index_select(0, keep)
            memo = [H[row_of[cap(x)]].index_select(0, bsel) for x in range(1, self.num_passes + 1)]
        mark()
        if times is not None:
            torch.cuda.synchronize()
            for name, a, b in zip(("hash", "featurize", "cost", "select", "cut", "memo"), ev[:-1], ev[1:]):
                times[name] = times.get(name, 0.0) + a.elapsed_time(b)
        out = {"beam": beam.cpu().tolist(), "beam_costs": beam_costs.cpu().tolist(), "memo": memo,
               "total": total, "verdict": verdict, "local": mine, "n_reps": n_all,
               "reps": cand if self.world == 1 else None}
        if rejects and rej is not None:
            nrej = int(nrej_t.item())
            ridx = rej[:nrej]
            codes = verdict.index_select(0, ridx).cpu().numpy()
            if mine is not None:   # pass-depth hashes: ranks merge their rejects in bucket order
                out["reject_hashes"] = [int(x) for x in hl.index_select(0, ridx).cpu().numpy().view(np.uint64)]
            ridx = (ridx if mine is None else mine.index_select(0, ridx)).cpu().numpy()
            out["rejects"] = [(int(i), PRUNE_REASONS[int(c) - 1]) for i, c in zip(ridx, codes)]
        return out

    def run_host(self, host_u8, flagged=None, temperature=0.0):
        """Public batch entry with host buffers: H2D records, one cut, D2H of
        every candidate's total + verdict (with their batch indices) and the
        beam.  Raises GsError on any device-side capacity/schedule error."""
        if host_u8.shape[0] != self.n:
            raise ValueError(f"batch of {host_u8.shape[0]} candidates, plan sized for {self.n}")
        dec = host_u8.to(self.sc.device, non_blocking=True)
        out = self.run(dec, flagged, temperature)
        return self._host_result(out, host_u8.numel())

    def run_beam_host(self, parents_u8, steps_i32, total=None, flagged=None, temperature=0.0):
        """Public beam-step entry with host buffers, as the search drives it:
        H2D of the beam (parent decision records + step-root indices), the
        candidates generated on the device (every phase-2 tiling of each
        parent's step root, gs_expand_step, search.py:223-235), one cut, D2H
        of every candidate's total + verdict (with their indices) and the
        beam.  `total` (the known candidate count) skips the sizing pass; it
        is checked against the device count before any record is written."""
        par = parents_u8.to(self.sc.device, non_blocking=True)
        st = steps_i32.to(self.sc.device, non_blocking=True)
        dec, _, _ = self.sc.expand_step(par, st, total=total)
        out = self.run(dec, flagged, temperature)
        return self._host_result(out, parents_u8.numel() + 4 * steps_i32.numel())

    @staticmethod
    def _to_host(t):
        """Stream-ordered D2H into pinned memory (torch's caching host
        allocator recycles the blocks across steps); a pageable .cpu() of
        the 8 MB totals ran at a fraction of PCIe speed."""
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        return h

    def _host_result(self, out, h2d):
        tot = self._to_host(out["total"])
        ver = self._to_host(out["verdict"])
        idx = self._to_host(out["local"]) if out["local"] is not None else None
        torch.cuda.current_stream(self.sc.device).synchronize()
        self.sc.check()
        d2h = tot.numel() * 8 + ver.numel() + 8 * len(out["beam"]) + (0 if idx is None else 8 * idx.numel())
        return {"h2d_bytes": h2d, "d2h_bytes": d2h, "beam": out["beam"], "beam_costs": out["beam_costs"],
                "total": tot, "verdict": ver, "index": idx}


def merge_rep_records(parts):
    """Rank-major concatenation of [n_r, 4] int64 records, stably sorted by
    the unsigned 64-bit hash in column 0."""
    allr = torch.cat(parts, dim=0)
    order = torch.sort(allr[:, 0] ^ SIGN, stable=True).indices
    return allr.index_select(0, order)
