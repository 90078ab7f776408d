"""Exact integer interval arithmetic (restates reference `boxes.py`).

Intervals are inclusive (lo, hi) pairs.  A "product" is one sorted disjoint
interval list per dimension and denotes their cross product.
"""

from __future__ import annotations

import itertools


def merge(ivs):
    """Sort + merge overlapping or touching intervals (boxes.py:21-31)."""
    out = []
    for lo, hi in sorted(ivs):
        if out and lo <= out[-1][1] + 1:
            if hi > out[-1][1]:
                out[-1] = (out[-1][0], hi)
        else:
            out.append((lo, hi))
    return out


def window_union(a, b, s, lo, hi):
    """Union over x in [a, b] of [x*s+lo, x*s+hi] (boxes.py:53-63)."""
    if s <= hi - lo + 1:
        return [(a * s + lo, b * s + hi)]
    return [(x * s + lo, x * s + hi) for x in range(a, b + 1)]


def through_links(ivs, links):
    """Exact footprint of an interval union through per-dim chain links
    (resolve.py:36-44)."""
    cur = list(ivs)
    for s, lo, hi in links:
        nxt = []
        for a, b in cur:
            nxt += window_union(a, b, s, lo, hi)
        cur = merge(nxt)
    return cur


def box_through(box, chain):
    """Bounding box of a chain applied to a box (resolve.py:29-33, 47-53)."""
    out = []
    for d, (a, b) in enumerate(box):
        for link in chain:
            s, lo, hi = link[d]
            a, b = a * s + lo, b * s + hi
        out.append((a, b))
    return out


def bbox(boxes):
    return [(min(b[d][0] for b in boxes), max(b[d][1] for b in boxes))
            for d in range(len(boxes[0]))]


def _pieces(lists):
    """Elementary segments of the union of several interval lists
    (boxes.py:69-84): split at every endpoint, keep covered pieces."""
    cuts = sorted({x for ivs in lists for lo, hi in ivs for x in (lo, hi + 1)})
    covered = merge([iv for ivs in lists for iv in ivs])
    out, j = [], 0
    for a, b in zip(cuts, cuts[1:]):
        while j < len(covered) and covered[j][1] < a:
            j += 1
        if j < len(covered) and covered[j][0] <= a:
            out.append((a, b - 1))
    return out


def _inside(ivs, seg):
    return any(lo <= seg[0] and seg[1] <= hi for lo, hi in ivs)


def union_count(products, lines: bool) -> int:
    """Points (lines=False) or maximal dim-0 runs (lines=True) in the union
    of products (boxes.py:92-138)."""
    products = [p for p in products if all(p)]
    if not products:
        return 0
    nd = len(products[0])
    if nd == 0:
        return 0 if lines else 1
    outer = [_pieces([p[d] for p in products]) for d in range(1, nd)]
    total = 0
    for cell in itertools.product(*outer):
        live = [p for p in products
                if all(_inside(p[d + 1], cell[d]) for d in range(nd - 1))]
        if not live:
            continue
        row = merge([iv for p in live for iv in p[0]])
        w = 1
        for lo, hi in cell:
            w *= hi - lo + 1
        total += w * (len(row) if lines else sum(hi - lo + 1 for lo, hi in row))
    return total
