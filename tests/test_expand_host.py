"""The host beam-step enumeration (gen.root_tilings / expand_step), which the
device expansion is checked against, equals the reference's own menus:
`gpusched.options.enumerate_serial_tilings` / `enumerate_thread_tilings`
(options.py:144-183) in `_phase2_candidates` order (search.py:223-235),
called from the unmodified reference (importable in the build container;
skipped where it is absent)."""

import math
import os
import sys

import pytest

from paper_2012_07145_b200 import gen

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
for _p in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
    if os.path.isdir(os.path.join(_p, "gpusched")) and _p not in sys.path:
        sys.path.append(_p)
options = pytest.importorskip("gpusched.options")


def _reference_phase2_order(extents):
    cfg = options.DEFAULT_TILING
    out = []
    for serial in options.enumerate_serial_tilings(extents, config=cfg):
        post = tuple(math.ceil(e / s) for e, s in zip(extents, serial))
        for thread in options.enumerate_thread_tilings(post, config=cfg):
            out.append((tuple(serial), tuple(thread)))
    return out


@pytest.mark.parametrize("extents", [(1024, 1024), (1536, 2560, 3), (56, 56, 256), (7, 3), (96, 1), (1280, 960),
                                     (1024,), (33, 17, 5), (2, 2, 2, 2)])
def test_root_tilings_follow_reference_order(extents):
    assert [(tuple(s), tuple(t)) for s, t in gen.root_tilings(extents)] == _reference_phase2_order(extents)


def test_menus_match_reference_config():
    cfg = options.DEFAULT_TILING
    for name in ("serial_powers", "odd_serial", "innermost_thread", "outer_thread", "unroll_budget", "warp_size"):
        mine, ref = getattr(gen.Menus, name), getattr(cfg, name)
        if isinstance(ref, (tuple, list)):
            mine, ref = tuple(mine), tuple(ref)
        assert mine == ref, name
