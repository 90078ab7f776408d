"""One beam step over a candidate batch, on one GPU or bucket-sharded over
several (one process per GPU, NCCL over NVLink for the exchange).

Sharding: every rank holds the batch's decision records and
hashes all of them at the pass depth (cheap).  A structural-hash bucket is
owned by rank `hash % world`, so buckets never straddle ranks; each rank
featurizes, prunes and costs only its buckets' candidates (the expensive
part) and draws their representatives with the same per-bucket PCG64
streams the reference uses.  Representative records (hash, cost, candidate
index, local order) are exchanged with one all-gather; every rank merges
them into the global (hash ascending, permutation position) order and cuts
the identical beam.  The only collective on the data path is that
all-gather of a few KB per rank.
"""

from __future__ import annotations

import numpy as np
import torch

SIGN = -0x8000000000000000  # flips int64 order into uint64 order


class StepPlan:
    def __init__(self, scorer, n, world, rank, pass_index, phase_seed, beam, penalty, num_passes,
                 tie_band):
        self.sc, self.n, self.world, self.rank = scorer, n, world, rank
        self.pass_index, self.phase_seed, self.beam = pass_index, phase_seed, beam
        self.penalty, self.num_passes, self.tie_band = penalty, num_passes, tie_band
        self.fbuf = None
        self.rcbuf = None
        self.local_count = n

    def _features(self, d):
        # the step consumes features only through K2 with row_src, so K1
        # writes just the computed rows (reuse mode 2)
        prev = self.sc.reuse_mode
        if prev:
            self.sc.set_reuse(2)
        try:
            return self._features_into(d)
        finally:
            if prev:
                self.sc.set_reuse(prev)

    def _features_into(self, d):
        m = d.shape[0]
        if self.fbuf is None or self.fbuf["feats"].shape[0] != m:
            self.fbuf = self.rcbuf = None
            torch.cuda.empty_cache()
            self.fbuf = self.sc.featurize(d)
            self.rcbuf = torch.empty((m, self.sc.R), dtype=torch.float64, device=self.sc.device)
        else:
            self.sc.featurize(d, out=self.fbuf)
        return self.fbuf

    def run(self, dec, times=None):
        """One beam step.  `times` (optional dict) accumulates the device
        milliseconds of each phase: hash, featurize (K1), cost (K2), select
        (K4 + exchange), cut (K5), memo (K3 at depths 1..num_passes)."""
        sc = self.sc
        ev = []

        def mark():
            if times is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev.append(e)

        mark()
        h = sc.struct_hash(dec, self.pass_index)
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
        total, _, _ = sc.cost(f, scratch=self.rcbuf)
        mark()
        rep, _, cnt = sc.select(hl, f["verdict"], self.phase_seed, rejects=False)
        nrep = int(cnt[0].item())
        rep = rep[:nrep]
        costs = total.index_select(0, rep)
        ph = hl.index_select(0, rep)
        cand = rep if mine is None else mine.index_select(0, rep)
        if self.world > 1:
            costs, ph, cand = self._exchange(costs, ph, cand, nrep)
        mark()
        pos, kcnt, bot = sc.beam_topk(costs, ph, None, self.penalty, 0.0, self.phase_seed,
                                      min(self.beam, costs.shape[0]), tie_band=self.tie_band)
        beam = cand.index_select(0, pos[:int(kcnt.item())])
        mark()
        # bad-hash memo: hashes of the bottom half at every pass depth.  All
        # representatives are hashed and the bottom half is picked after the
        # step's one closing sync, so the host never waits mid-step here.
        # at pass depth >= 3 the representatives' bucket hashes ARE their
        # depth-3 hashes (the key caps at 3)
        memo = sc.memo_hashes(dec.index_select(0, cand), self.num_passes,
                              h3=ph if self.pass_index >= 3 else None) if costs.shape[0] > 1 else []
        mark()
        if times is not None:
            torch.cuda.synchronize()
            for name, a, b in zip(("hash", "featurize", "cost", "select", "cut", "memo"), ev[:-1], ev[1:]):
                times[name] = times.get(name, 0.0) + a.elapsed_time(b)
        beam_host = beam.cpu().tolist()
        if memo:
            keep = torch.nonzero(bot).flatten()
            memo = [m.index_select(0, keep) for m in memo]
        return {"beam": beam_host, "total": total, "verdict": f["verdict"], "memo": memo,
                "n_reps": int(costs.shape[0])}

    def _exchange(self, costs, ph, cand, nrep):
        return exchange_reps(costs, ph, cand, self.world)

    def run_host(self, host_u8):
        """Public batch entry with host buffers: H2D records, one step, D2H of
        every candidate's total + verdict and the beam."""
        dec = host_u8.to(self.sc.device, non_blocking=True)
        out = self.run(dec)
        tot = out["total"].cpu()
        ver = out["verdict"].cpu()
        return {"h2d_bytes": host_u8.numel(), "d2h_bytes": tot.numel() * 8 + ver.numel() + 8 * len(out["beam"]),
                "beam": out["beam"]}

    def run_beam_host(self, parents_u8, steps_i32, total=None):
        """Public beam-step entry with host buffers, as the search drives it:
        H2D of the beam (parent decision records + step-root indices), the
        candidates generated on the device (every phase-2 tiling of each
        parent's step root, gs_expand_step), one step, D2H of every
        candidate's total + verdict and the beam."""
        par = parents_u8.to(self.sc.device, non_blocking=True)
        st = steps_i32.to(self.sc.device, non_blocking=True)
        dec, _, _ = self.sc.expand_step(par, st, total=total)
        out = self.run(dec)
        tot = out["total"].cpu()
        ver = out["verdict"].cpu()
        return {"h2d_bytes": parents_u8.numel() + 4 * steps_i32.numel(),
                "d2h_bytes": tot.numel() * 8 + ver.numel() + 8 * len(out["beam"]), "beam": out["beam"]}


def exchange_reps(costs, ph, cand, world, group=None):
    """All-gather every rank's representative records and merge them into
    the global representative order of the reference (search.py:151-164:
    hash ascending, then permutation position inside the bucket).

    Each record is 4 x int64: (hash at pass depth, fp64 cost bits, candidate
    index, local rep order).  Buckets never straddle ranks (owner = hash %
    world), so a stable sort by unsigned hash over the rank-major
    concatenation reproduces the single-GPU order exactly.  Works with any
    torch.distributed backend (NCCL on the GPU path, gloo in the CPU tests).
    Returns (costs f64, pass hashes i64, candidate indices i64)."""
    import torch.distributed as dist
    if dist.get_backend(group) == "gloo" and costs.is_cuda:   # gloo gathers host tensors
        c, p, i = exchange_reps(costs.cpu(), ph.cpu(), cand.cpu(), world, group)
        return c.to(costs.device), p.to(costs.device), i.to(costs.device)
    nrep = int(costs.shape[0])
    dev = costs.device
    rec = torch.stack([ph, costs.view(torch.int64), cand,
                       torch.arange(nrep, device=dev, dtype=torch.int64)], dim=1)
    counts = torch.tensor([nrep], device=dev, dtype=torch.int64)
    allc = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(allc, counts, group=group)
    allc = torch.cat(allc).cpu().tolist()
    mx = max(1, max(allc))
    pad = torch.zeros((mx, 4), device=dev, dtype=torch.int64)
    pad[:nrep] = rec
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    allr = merge_rep_records([p[:c] for p, c in zip(parts, allc)])
    return allr[:, 1].view(torch.float64).contiguous(), allr[:, 0].contiguous(), allr[:, 2].contiguous()


def merge_rep_records(parts):
    """Rank-major concatenation of [n_r, 4] int64 records, stably sorted by
    the unsigned 64-bit hash in column 0."""
    allr = torch.cat(parts, dim=0)
    order = torch.sort(allr[:, 0] ^ SIGN, stable=True).indices
    return allr.index_select(0, order)
