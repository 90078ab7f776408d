"""Decision log -> padded-tile geometry (restates reference `resolve.py`).

Output of `resolve_geometry`:
  geos    — dict func -> Geo, insertion order = the reference `cs.funcs`
            order: non-inline funcs in decision order, then externals /
            unscheduled producers in graph order, then inline funcs in
            decision order (resolve.py:233-365).
  kernels — dict owner -> Kernel (blocks, members, threads, shared bytes).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .boxes import bbox, box_through

UNROLL_LIMIT = 16  # resolve.py:24
TIER_OF_KIND = {"compute_root": "global", "fuse_at_block": "shared",
                "fuse_at_thread": "register", "inline": "none"}


@dataclass
class Read:
    owner: str        # func whose body issues the load
    producer: str
    tier: str
    chain: tuple      # links; each link = per-dim (stride, lo, hi)
    elem_bytes: int

    @property
    def total_stride(self):
        nd = len(self.chain[0])
        return [math.prod(link[d][0] for link in self.chain) for d in range(nd)]


@dataclass
class Geo:
    name: str
    kind: str
    tier: str
    kernel: str | None
    consumer: str | None
    serial: tuple | None
    thread: tuple | None
    blocks: tuple | None
    region: list
    total: list
    realizations: int
    n_threads: int
    ctx: tuple            # context thread extents
    base: tuple           # lane base
    coeff: tuple          # lane coeff
    ext: tuple            # lane extent
    unrolled: bool
    reads: list = field(default_factory=list)   # per stage
    primary: str | None = None
    calls: int = 0

    @property
    def pts_thread(self):
        return math.prod(self.ext)

    @property
    def pts_block(self):
        return self.pts_thread * self.n_threads

    def block_box(self):
        """resolve.py:112-122."""
        if self.blocks is not None:
            return [(0, t * s - 1) for t, s in zip(self.thread, self.serial)]
        if self.kind == "fuse_at_block":
            return list(self.region)
        return [(b, b + (ct - 1) * c + e - 1)
                for b, c, e, ct in zip(self.base, self.coeff, self.ext, self.ctx)]

    def lane_box(self):
        return [(b, b + e - 1) for b, e in zip(self.base, self.ext)]

    @property
    def alloc(self):
        if self.tier == "none":
            return 0
        return math.prod(hi - lo + 1 for lo, hi in self.region)


@dataclass
class Kernel:
    owner: str
    blocks: tuple
    members: list
    threads: int = 0
    shared_bytes: int = 0

    @property
    def n_blocks(self):
        return math.prod(self.blocks)


def default_tiling(extents):
    """resolve.py:159-164."""
    inner = next((i for i, e in enumerate(extents) if e >= 16), 0)
    return (tuple(1 for _ in extents),
            tuple(min(32, e) if i == inner else 1 for i, e in enumerate(extents)))


def expand_stage(graph, dmap, func, si, prefix=()):
    """Reads of one stage with inlined producers substituted
    (resolve.py:167-200).  Returns (reads, {inline func: calls per point})."""
    reads, calls = [], {}
    for acc in graph.func(func).stages[si].accesses:
        chain = prefix + (tuple(acc.dims),)
        pnode = graph.func(acc.producer)
        pd = dmap.get(acc.producer)
        if pd is not None and pd.kind == "inline":
            vol = 1
            for link in chain:
                for _s, lo, hi in link:
                    vol *= hi - lo + 1
            calls[acc.producer] = calls.get(acc.producer, 0) + vol
            sub, subcalls = expand_stage(graph, dmap, acc.producer, 0, chain)
            reads += sub
            for k, v in subcalls.items():
                calls[k] = calls.get(k, 0) + v
            continue
        if pd is None or pd.kind == "compute_root" or pnode.is_external_input:
            tier = "global"
        else:
            tier = TIER_OF_KIND[pd.kind]
        reads.append(Read(func, acc.producer, tier, chain, pnode.elem_bytes))
    return reads, calls


def resolve_geometry(graph, decisions, provisional=True):
    dmap = dict(decisions)
    geos: dict[str, Geo] = {}
    kernels: dict[str, Kernel] = {}
    expanded = {}

    def stage_reads(f, si):
        key = (f, si)
        if key not in expanded:
            expanded[key] = expand_stage(graph, dmap, f, si)
        return expanded[key]

    def sources(func):
        # resolve.py:379-393: (consumer geo, chain) pairs, consumer order =
        # geos insertion order at the time of the call.
        out = []
        for cname, cg in geos.items():
            if cg.kind in ("external", "inline"):
                continue
            for si in range(len(graph.func(cname).stages)):
                for r in stage_reads(cname, si)[0]:
                    if r.producer == func:
                        out.append((cg, r.chain))
        return out

    # Pass 1 (resolve.py:232-333): non-inline decisions in order.
    for func, d in decisions:
        node = graph.func(func)
        if d.kind == "inline":
            continue
        if d.kind == "compute_root":
            serial, thread = d.serial, d.thread
            if serial is None or thread is None:
                if not provisional:
                    raise ValueError(f"{func} untiled")
                serial, thread = default_tiling(node.extents)
            blocks = tuple(max(1, -(-e // (s * t)))
                           for e, s, t in zip(node.extents, serial, thread))
            region = [(0, b * t * s - 1) for b, t, s in zip(blocks, thread, serial)]
            geos[func] = Geo(func, d.kind, "global", func, None, serial, thread, blocks,
                             region, list(region), 1, math.prod(thread), thread,
                             tuple(0 for _ in serial), serial, serial,
                             math.prod(serial) < UNROLL_LIMIT)
            kernels[func] = Kernel(func, blocks, [func])
            continue
        src = sources(func)
        if not src:
            raise ValueError(f"{func} is fused but has no resolved consumers")
        if d.kind == "fuse_at_block":
            serial = d.serial if d.serial is not None else tuple(1 for _ in node.extents)
            raw = bbox([box_through(cg.block_box(), ch) for cg, ch in src])
            thread = tuple(max(1, -(-(hi - lo + 1) // s)) for (lo, hi), s in zip(raw, serial))
            region = [(lo, lo + t * s - 1) for (lo, _), t, s in zip(raw, thread, serial)]
            traw = bbox([box_through(cg.total, ch) for cg, ch in src])
            total = [(lo, max(hi, lo + t * s - 1)) for (lo, hi), t, s in zip(traw, thread, serial)]
            kern = kernels[src[0][0].kernel]
            geos[func] = Geo(func, d.kind, "shared", kern.owner, d.consumer, serial, thread,
                             None, region, total, kern.n_blocks, math.prod(thread), thread,
                             tuple(lo for lo, _ in region), serial, serial,
                             math.prod(serial) < UNROLL_LIMIT)
            kern.members.append(func)
        else:
            cg0, ch0 = src[0]
            lane = cg0.lane_box()
            region = bbox([box_through(lane, ch) for _, ch in src])
            coeff = tuple(c * math.prod(link[dd][0] for link in ch0)
                          for dd, c in enumerate(cg0.coeff))
            kern = kernels[cg0.kernel]
            ext = tuple(hi - lo + 1 for lo, hi in region)
            geos[func] = Geo(func, d.kind, "register", kern.owner, d.consumer, None, None,
                             None, region, bbox([box_through(cg0.total, ch) for _, ch in src]),
                             kern.n_blocks * cg0.n_threads, cg0.n_threads, cg0.ctx,
                             tuple(lo for lo, _ in region), coeff, ext,
                             math.prod(ext) < UNROLL_LIMIT)
            kern.members.append(func)

    # External inputs and unscheduled producers (resolve.py:396-425).
    for fnode in graph.funcs:
        if fnode.name in geos or (fnode.name in dmap and not fnode.is_external_input):
            continue
        boxes = []
        for cname, cg in list(geos.items()):
            if cg.kind in ("external", "inline"):
                continue
            for si in range(len(graph.func(cname).stages)):
                for r in stage_reads(cname, si)[0]:
                    if r.producer == fnode.name:
                        boxes.append(box_through(cg.total, r.chain))
        box = bbox(boxes) if boxes else [(0, e - 1) for e in fnode.extents]
        nd = fnode.ndim
        geos[fnode.name] = Geo(fnode.name, "external", "global", None, None, None, None,
                               None, box, list(box), 0, 1, (1,) * nd, (0,) * nd,
                               (0,) * nd, (1,) * nd, False)

    # Pass 2 (resolve.py:337-349): read lists and inline call accounting.
    inl_total, inl_best = {}, {}
    for func, g in geos.items():
        if g.kind == "external":
            continue
        for si in range(len(graph.func(func).stages)):
            reads, calls = stage_reads(func, si)
            g.reads.append(reads)
            for iname, vol in calls.items():
                c = vol * g.pts_block * kernels[g.kernel].n_blocks
                inl_total[iname] = inl_total.get(iname, 0) + c
                if iname not in inl_best or c > inl_best[iname][0]:
                    inl_best[iname] = (c, func)

    # Inline rows in the primary consumer's context (resolve.py:351-375).
    for func, d in decisions:
        if d.kind != "inline":
            continue
        primary = inl_best.get(func, (0, None))[1]
        host = geos.get(primary) if primary else None
        nd = graph.func(func).ndim
        own = [r for g in geos.values() if g.kind != "external"
               for rs in g.reads for r in rs if r.owner == func]
        geos[func] = Geo(func, "inline", "none", host.kernel if host else None, primary,
                         None, None, None, [(0, -1)] * nd, [(0, -1)] * nd, 0,
                         host.n_threads if host else 1,
                         host.ctx if host else (1,) * nd, (0,) * nd, (0,) * nd, (1,) * nd,
                         host.unrolled if host else True, [own], primary,
                         inl_total.get(func, 0))

    # Kernel aggregates (resolve.py:368-373).
    for k in kernels.values():
        k.threads = max((geos[m].n_threads for m in k.members), default=1)
        k.shared_bytes = sum(geos[m].alloc * graph.func(m).elem_bytes
                             for m in k.members if geos[m].tier == "shared")
    return geos, kernels
