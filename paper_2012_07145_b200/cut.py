"""One beam-search phase on the GPU: the batched replacement of the
reference `_cut` (pkg/src/gpusched/search.py:168-201) and
`_select_representatives` (search.py:127-165).

All candidates of the phase are featurized + prune-checked in one K1
launch, hashed at the pass depth (K3), bucketed and sampled (K4), the
representatives costed (K2) and cut (K5).  The host only uploads the
decision records and downloads the beam indices, costs, prune rejects and
the memo hashes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .descriptor import PRUNE_REASONS
from .engine import as_u64, u64_sorted_tensor


@dataclass
class CutResult:
    beam: list                     # candidate indices, beam order
    costs: list                    # unpenalized predicted cost per beam entry
    rejects: list                  # (candidate index, prune reason) in draw order
    memo_new: set = field(default_factory=set)   # (depth, hash) to flag
    reps: list = field(default_factory=list)     # representative candidate indices


def beam_cut(scorer, dec: torch.Tensor, pass_index: int, phase_seed: int, flagged,
             beam_size: int, penalty: float, temperature: float, num_passes: int,
             sampling: bool = True) -> CutResult:
    n = dec.shape[0]
    f = scorer.featurize(dec)
    h = scorer.struct_hash(dec, pass_index)
    verdict = f["verdict"]
    if sampling:
        rep, rej, cnt = scorer.select(h, verdict, phase_seed)
        nrep, nrej = (int(x) for x in cnt.tolist())
        rep = rep[:nrep]
        rej = rej[:nrej]
    else:   # test hook: every valid candidate, in order (search.py:142-150)
        valid = verdict == 0
        rep = torch.nonzero(valid).flatten()
        rej = torch.nonzero(~valid).flatten()
        nrep = rep.numel()
    scorer.check()
    vcpu = verdict.cpu().numpy()
    rej_idx = rej.cpu().numpy().tolist()
    rejects = [(i, PRUNE_REASONS[int(vcpu[i]) - 1]) for i in rej_idx]
    if nrep == 0:
        return CutResult([], [], rejects)
    sub = {k: f[k].index_select(0, rep) for k in ("feats", "row_key", "n_rows")}
    total, _, _ = scorer.cost(sub)
    ph = h.index_select(0, rep)
    fl = u64_sorted_tensor(flagged, scorer.device) if flagged else None
    pos, cnt, bot = scorer.beam_topk(total, ph, fl, penalty, temperature, phase_seed,
                                     min(beam_size, nrep))
    k = int(cnt.item())
    pos = pos[:k]
    rep_cpu = rep.cpu().numpy()
    tot_cpu = total.cpu().numpy()
    pos_cpu = pos.cpu().numpy()
    memo_new = set()
    if nrep > 1:
        bsel = torch.nonzero(bot[:nrep]).flatten()
        bdec = dec.index_select(0, rep.index_select(0, bsel))
        for depth, hs in enumerate(scorer.memo_hashes(bdec, num_passes), start=1):
            memo_new |= {(depth, int(x)) for x in as_u64(hs)}
    return CutResult(beam=[int(rep_cpu[p]) for p in pos_cpu],
                     costs=[float(tot_cpu[p]) for p in pos_cpu],
                     rejects=rejects, memo_new=memo_new,
                     reps=[int(x) for x in rep_cpu])


def score_batch(scorer, dec: torch.Tensor):
    """Featurize + prune + cost every candidate: (totals, verdicts) on device."""
    f = scorer.featurize(dec)
    total, _, _ = scorer.cost(f)
    return total, f["verdict"], f


def np_u64(values) -> np.ndarray:
    return np.array([int(v) & 0xFFFFFFFFFFFFFFFF for v in values], dtype=np.uint64)
