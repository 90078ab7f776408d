"""One beam-search phase on the GPU: the batched replacement of the
reference `_cut` (pkg/src/gpusched/search.py:168-201) and
`_select_representatives` (search.py:127-165).

All candidates of the phase are featurized + prune-checked in one K1
launch, costed (K2), hashed at the pass depth (K3), bucketed and sampled
(K4) and cut (K5) by `shard.StepPlan.run`.  The host only uploads the
decision records and downloads the beam indices, costs, prune rejects and
the memo hashes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .engine import TIE_BAND, as_u64


@dataclass
class CutResult:
    beam: list                     # candidate indices, beam order
    costs: list                    # unpenalized predicted cost per beam entry
    rejects: list                  # (candidate index, prune reason) in draw order
    memo_new: set = field(default_factory=set)   # (depth, hash) to flag
    reps: list = field(default_factory=list)     # representative candidate indices


def beam_cut(scorer, dec: torch.Tensor, pass_index: int, phase_seed: int, flagged,
             beam_size: int, penalty: float, temperature: float, num_passes: int,
             sampling: bool = True, world: int = 1, rank: int = 0, group=None) -> CutResult:
    """One phase cut through `shard.StepPlan` (the single cut
    implementation), with the results in host form.  world > 1: every rank
    calls this with the whole phase; buckets are sharded across the ranks of
    `group` and every rank returns the same result (the memo
    and the rejects are gathered; the rejects in the reference's bucket
    order)."""
    from .shard import StepPlan
    plan = StepPlan(scorer, dec.shape[0], world, rank, pass_index, phase_seed, beam_size, penalty, num_passes,
                    TIE_BAND, sampling=sampling, group=group)
    out = plan.run(dec, flagged=flagged, temperature=temperature, rejects=True)
    scorer.check()
    memo_new = {(depth, int(x)) for depth, hs in enumerate(out["memo"], start=1) for x in as_u64(hs)}
    rejects = out.get("rejects", [])
    if world > 1:
        import torch.distributed as dist
        parts = [None] * world
        dist.all_gather_object(parts, (sorted(memo_new), list(zip(out.get("reject_hashes", []), rejects))),
                               group=group)
        memo_new = {tuple(m) for p in parts for m in p[0]}
        # a bucket lives on one rank: a stable sort by hash restores the
        # reference's draw order (buckets ascending, draws in order)
        merged = [r for p in parts for r in p[1]]
        rejects = [tuple(r[1]) for r in sorted(merged, key=lambda r: r[0])]
    reps = out["reps"].cpu().tolist() if out["reps"] is not None else []
    return CutResult(beam=out["beam"], costs=out["beam_costs"], rejects=rejects,
                     memo_new=memo_new, reps=reps)


def score_batch(scorer, dec: torch.Tensor):
    """Featurize + prune + cost every candidate: (totals, verdicts) on device."""
    f = scorer.featurize(dec)
    total, _, _ = scorer.cost(f)
    return total, f["verdict"], f


def np_u64(values) -> np.ndarray:
    return np.array([int(v) & 0xFFFFFFFFFFFFFFFF for v in values], dtype=np.uint64)
