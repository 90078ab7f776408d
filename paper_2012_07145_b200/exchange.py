"""The cut of a bucket-sharded phase: every rank holds the
representatives of its own buckets; the ranks agree on the reference cut
(search.py:168-201) by exchanging only what can reach it.

Order.  The reference sorts the representatives stably by key, i.e. by
(key, global representative position), and the global position order is
(bucket hash ascending, permutation position) (search.py:151-164).  A
bucket lives on one rank (owner = hash % world), so the pair (hash as
uint64, local position) orders any two representatives exactly as their
global positions do — no rank needs another rank's positions.  With the
tie band (engine.TIE_BAND) keys are grouped as in K5 (select.cu
`cut_kernel`): a band group is a maximal value-ordered run whose adjacent
gaps are within the band, and the order is (group, hash, local position).

Beam (top-k).  Each rank sorts its keys and sends its local window: the
first keys up to the end of the band group holding its k-th key (at most
`TOP_CAP` records), plus the smallest key it did not send.  Every rank
merges the world's windows identically and takes the first k.  The global
k-th key is at most any rank's local k-th key, so every key that can reach
the beam or share a group with it was sent — checked exactly at run time:
the merged group holding the k-th key must end a band gap below every
rank's smallest unsent key.  One fixed-size all-gather of
world x TOP_CAP x 48 B.

Memo threshold (bottom half by unpenalized cost, search.py:196-200).  The
key of global rank floor(n/2) comes from a distributed radix select: eight
all-reduces of a 256-bin histogram of one byte of the sortable cost bits.
The ranks then exchange only the keys within a margin of it (at most
`MEMO_CAP` each), plus counts and the nearest keys outside the margin, and
order that window exactly like K5.  Everything below the window is in the
top half, everything above it in the bottom half.

If a check fails (a tie group wider than a window, or explore_temperature
> 0, whose Gumbel draws follow global positions), the phase falls back to
gathering every representative's (key, hash, position) record — exact, and
rare.  `LAST_BYTES` holds the bytes the last call exchanged per rank.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

SIGN = -0x8000000000000000
TOP_CAP = 128
MEMO_CAP = 512
MEMO_MARGIN = 64.0       # window half-width in tie bands
LAST_BYTES = 0
LAST_FALLBACK = False

_INF = float("inf")


def _comm(t, group):
    """Tensors go through the collective on the backend's device."""
    if dist.get_backend(group) == "gloo" and t.is_cuda:
        return t.cpu()
    return t


def _all_gather(t, world, group):
    global LAST_BYTES
    src = _comm(t.contiguous(), group)
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src, group=group)
    LAST_BYTES += src.numel() * src.element_size()
    return torch.stack(parts).to(t.device)


def _all_reduce(t, op, group):
    global LAST_BYTES
    src = _comm(t.contiguous(), group)
    dist.all_reduce(src, op=op, group=group)
    LAST_BYTES += src.numel() * src.element_size()
    return src.to(t.device)


def band_breaks(v, band):
    """brk[j] = a band gap between sorted values v[j-1] and v[j] (brk[0] = 0)."""
    brk = torch.zeros(v.shape, dtype=torch.bool, device=v.device)
    if v.numel() > 1:
        a, b = v[:-1], v[1:]
        brk[1:] = (torch.isinf(b) & ~torch.isinf(a)) | ((b - a) > band * torch.maximum(a.abs(), b.abs()))
    return brk


def band_order(v, h, pos, band):
    """Permutation ordering (value, hash, pos) records by (band group of the
    value, hash as uint64, pos).  Returns (order, group id per sorted value,
    value-sort permutation)."""
    vs, vperm = torch.sort(v, stable=True)
    gid = torch.cumsum(band_breaks(vs, band).to(torch.int64), 0)
    g = torch.empty_like(gid)
    g[vperm] = gid
    order = torch.argsort(pos, stable=True)
    order = order[torch.argsort((h ^ SIGN)[order], stable=True)]
    order = order[torch.argsort(g[order], stable=True)]
    return order, g


def penalized_keys(costs, ph, flagged, penalty):
    """apply_pass_penalty (search.py:76-87) on the representatives."""
    if flagged is None or flagged.numel() == 0:
        return costs.clone()
    fu = flagged ^ SIGN                        # uint64 order as int64 order
    hu = ph ^ SIGN
    i = torch.searchsorted(fu, hu).clamp(max=fu.numel() - 1)
    hit = fu[i] == hu
    return torch.where(hit, costs * penalty, costs)


def sharded_cut(sc, costs, ph, cand, flagged, penalty, temperature, phase_seed, k, band, world, group=None):
    """The cut of one phase over bucket-sharded representatives.

    costs / ph / cand: this rank's representatives (unpenalized cost, hash
    at the pass depth, batch candidate index) in local representative
    order.  Returns (beam candidate indices [<= k], their unpenalized costs,
    this rank's bottom-half flags (bool [n_local]), global rep count) — the
    same on every rank."""
    global LAST_BYTES, LAST_FALLBACK
    LAST_BYTES = 0
    LAST_FALLBACK = False
    dev = costs.device
    n_l = costs.numel()
    lpos = torch.arange(n_l, device=dev, dtype=torch.int64)
    keys = penalized_keys(costs, ph, flagged, penalty)
    n_tot = int(_all_reduce(torch.tensor([n_l], device=dev, dtype=torch.int64), dist.ReduceOp.SUM,
                            group).item())
    if n_tot == 0:
        return cand[:0], costs[:0], torch.zeros(n_l, dtype=torch.bool, device=dev), 0
    if temperature > 0:
        return _gather_all_cut(sc, costs, ph, cand, lpos, flagged, penalty, temperature, phase_seed, k, band,
                               world, group)
    kk = min(k, n_tot)
    beam, bcost, ok_top = _top_exchange(keys, costs, ph, cand, lpos, kk, band, world, group)
    if n_tot > 1:
        bottom, ok_bot = _memo_exchange(costs, ph, lpos, n_tot, band, world, group)
        ok_top = ok_top & ok_bot
    else:
        bottom = torch.zeros(n_l, dtype=torch.bool, device=dev)
    if not bool(ok_top.item()):
        return _gather_all_cut(sc, costs, ph, cand, lpos, flagged, penalty, 0.0, phase_seed, k, band, world,
                               group)
    return beam, bcost, bottom, n_tot


def _gap(a, b, band):
    """A band gap between values a <= b (infinite ends always break)."""
    return torch.isinf(a) | torch.isinf(b) | ((b - a) > band * torch.maximum(a.abs(), b.abs()))


def _top_exchange(keys, costs, ph, cand, lpos, kk, band, world, group):
    dev = keys.device
    n_l = keys.numel()
    f64 = torch.float64
    inf = torch.tensor([_INF], dtype=f64, device=dev)
    vs, perm = torch.sort(keys, stable=True)
    j = torch.arange(n_l, device=dev)
    # end of the band group holding local rank kk-1: the first break at j >= kk
    end = torch.where(band_breaks(vs, band) & (j >= kk), j, torch.full_like(j, n_l)).min() if n_l \
        else torch.zeros((), dtype=torch.int64, device=dev)
    C = TOP_CAP
    take = perm[:C]
    m = take.numel()
    rec = torch.zeros((C + 1, 6), dtype=torch.int64, device=dev)
    rec[:C, 0] = inf.view(torch.int64)
    valid = torch.arange(m, device=dev) < end
    rec[:m, 0] = torch.where(valid, keys[take], inf.expand(m)).view(torch.int64)
    rec[:m, 1] = ph[take]
    rec[:m, 2] = lpos[take]
    rec[:m, 3] = cand[take]
    rec[:m, 4] = costs[take].view(torch.int64)
    rec[:m, 5] = valid.to(torch.int64)
    unsent = torch.cat([vs, inf])[end]                    # smallest key not sent
    rec[C, 0] = unsent.view(torch.int64).reshape(())
    rec[C, 1] = (end > C).to(torch.int64)
    allr = _all_gather(rec, world, group)                 # [world, C+1, 6]
    body = allr[:, :C].reshape(-1, 6)
    hdr = allr[:, C]
    v = body[:, 0].view(f64)
    order, g = band_order(v, body[:, 1], body[:, 2], band)
    first = order[:kk]                                    # unsent keys sort last (+inf)
    beam = body[first, 3]
    bcost = body[first, 4].view(f64)
    # exactness: the group of the last beam key ends a band gap below every
    # rank's smallest unsent key, and no window overflowed
    gmax = torch.where(g == g[first[-1]], v, -inf).max()
    ok = _gap(gmax, hdr[:, 0].view(f64).min(), band) & (hdr[:, 1].sum() == 0)
    return beam, bcost, ok


def _memo_exchange(costs, ph, lpos, n_tot, band, world, group):
    """Bottom-half flags of this rank's representatives (see module doc)."""
    dev = costs.device
    n_l = costs.numel()
    bits = costs.view(torch.int64)
    # sortable uint64 key, held as int64 bits
    skey = torch.where(bits < 0, ~bits, bits ^ SIGN)
    target = n_tot // 2
    prefix = torch.zeros((), dtype=torch.int64, device=dev)
    rank = torch.tensor(target, dtype=torch.int64, device=dev)
    for p in range(8):
        shift = 56 - 8 * p
        if p == 0:
            match = torch.ones(n_l, dtype=torch.bool, device=dev)
        else:
            mask_hi = -(1 << (64 - 8 * p)) if 64 - 8 * p < 63 else SIGN
            match = ((skey ^ prefix) & mask_hi) == 0
        dig = (skey >> shift) & 255
        hist = torch.bincount(dig[match], minlength=256)[:256].to(torch.int64)
        hist = _all_reduce(hist, dist.ReduceOp.SUM, group)
        cum = torch.cumsum(hist, 0)
        d = torch.searchsorted(cum, rank.reshape(1), right=True).reshape(()).clamp(max=255)
        before = torch.where(d > 0, cum[(d - 1).clamp(min=0)], torch.zeros_like(rank))
        rank = rank - before
        prefix = prefix | (d << shift)
    vstar_bits = torch.where(prefix < 0, prefix ^ SIGN, ~prefix)
    vstar = vstar_bits.view(torch.float64)
    half = MEMO_MARGIN * band * vstar.abs()
    lo, hi = vstar - half, vstar + half
    below = costs < lo
    above = costs > hi
    inwin = ~below & ~above
    C = MEMO_CAP
    widx = torch.nonzero(inwin).flatten()[:C]
    m = widx.numel()
    rec = torch.zeros((C + 1, 4), dtype=torch.int64, device=dev)
    inf_bits = torch.tensor([_INF], dtype=torch.float64, device=dev).view(torch.int64)
    rec[:C, 0] = inf_bits
    rec[:m, 0] = costs[widx].view(torch.int64)
    rec[:m, 1] = ph[widx]
    rec[:m, 2] = lpos[widx]
    rec[:m, 3] = 1
    ninf = torch.tensor(-_INF, device=dev, dtype=torch.float64)
    pinf = torch.tensor(_INF, device=dev, dtype=torch.float64)
    maxb = torch.where(below, costs, ninf).max() if n_l else ninf
    mina = torch.where(above, costs, pinf).min() if n_l else pinf
    rec[C, 0] = below.sum()
    rec[C, 1] = maxb.view(torch.int64).reshape(())
    rec[C, 2] = mina.view(torch.int64).reshape(())
    rec[C, 3] = (inwin.sum() > C).to(torch.int64)
    allr = _all_gather(rec, world, group)
    body = allr[:, :C]
    hdr = allr[:, C]
    rank_of = torch.arange(world, device=dev).reshape(-1, 1).expand(world, C).reshape(-1)
    body = body.reshape(-1, 4)
    v = body[:, 0].view(torch.float64)
    valid = body[:, 3] == 1
    order, _ = band_order(v, body[:, 1], body[:, 2], band)
    c_lo = hdr[:, 0].sum()
    g_maxb = hdr[:, 1].view(torch.float64).max()
    g_mina = hdr[:, 2].view(torch.float64).min()
    wv = v[valid]
    wmin = wv.min() if wv.numel() else pinf
    wmax = wv.max() if wv.numel() else ninf
    ok = _gap(g_maxb, wmin, band) & _gap(wmax, g_mina, band) & (hdr[:, 3].sum() == 0)
    bottom = above.clone()
    me = dist.get_rank(group)
    ranks_in_order = torch.empty_like(order)
    ranks_in_order[order] = torch.arange(order.numel(), device=dev)
    sel = valid & (rank_of == me)
    gl_rank = c_lo + ranks_in_order[sel]
    bottom[body[sel, 2]] = gl_rank >= target
    return bottom, ok


def _gather_all_cut(sc, costs, ph, cand, lpos, flagged, penalty, temperature, phase_seed, k, band, world,
                    group):
    """Exact fallback: gather every representative's record, rebuild the
    global representative order and cut it with K5 on every rank."""
    global LAST_FALLBACK
    LAST_FALLBACK = True
    dev = costs.device
    n_l = costs.numel()
    cnt = _all_gather(torch.tensor([n_l], device=dev, dtype=torch.int64), world, group).reshape(-1)
    counts = cnt.cpu().tolist()
    mx = max(1, max(counts))
    rec = torch.zeros((mx, 4), dtype=torch.int64, device=dev)
    rec[:n_l, 0] = ph
    rec[:n_l, 1] = costs.view(torch.int64)
    rec[:n_l, 2] = cand
    rec[:n_l, 3] = lpos
    allr = _all_gather(rec, world, group)
    me = dist.get_rank(group)
    parts, owner = [], []
    for r, c in enumerate(counts):
        parts.append(allr[r, :c])
        owner.append(torch.full((c,), r, dtype=torch.int64, device=dev))
    allr = torch.cat(parts)
    own = torch.cat(owner)
    order = torch.sort(allr[:, 0] ^ SIGN, stable=True).indices    # global rep order
    allr, own = allr[order], own[order]
    gcost = allr[:, 1].view(torch.float64).contiguous()
    n_all = gcost.numel()
    if n_all == 0:
        return cand[:0], costs[:0], torch.zeros(n_l, dtype=torch.bool, device=dev), 0
    pos, kcnt, bot = sc.beam_topk(gcost, allr[:, 0].contiguous(), flagged, penalty, temperature, phase_seed,
                                  min(k, n_all), tie_band=band)
    kk = int(kcnt.item())
    if kk < 0:
        from ._lib import GsError
        raise GsError("beam_topk: a tie group exceeds the cut window")
    beam = allr[pos[:kk], 2]
    bottom = torch.zeros(n_l, dtype=torch.bool, device=dev)
    mine = own == me
    bottom[allr[mine, 3]] = bot[mine].bool()
    return beam, gcost[pos[:kk]], bottom, n_all
