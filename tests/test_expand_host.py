"""The host beam-step enumeration (gen.root_tilings / expand_step), which the
device expansion is checked against, equals the reference menus
(options.py:144-183 enumerate_serial_tilings / enumerate_thread_tilings in
`_phase2_candidates` order, search.py:223-235), restated here from the
reference source as plain loops."""

import itertools
import math

import pytest

from paper_2012_07145_b200 import gen


def _ref_serial(extents, m=gen.Menus):
    per = []
    for e in extents:
        opts = sorted({s for s in m.serial_powers if s <= e})
        for o in m.odd_serial:
            if o <= e and e % o == 0 and (e // o) % m.warp_size == 0:
                opts.append(o)
        per.append(sorted(set(opts)) or [1])
    return [v for v in itertools.product(*per) if math.prod(v) <= m.unroll_budget]


def _ref_thread(extents, m=gen.Menus):
    inner = next((i for i, e in enumerate(extents) if e >= 16), 0)
    per = [sorted({min(t, e) for t in (m.innermost_thread if i == inner else m.outer_thread)})
           for i, e in enumerate(extents)]
    return list(itertools.product(*per))


@pytest.mark.parametrize("extents", [(1024, 1024), (1536, 2560, 3), (56, 56, 256), (7, 3), (96, 1), (1280, 960)])
def test_root_tilings_follow_reference_order(extents):
    want = []
    for s in _ref_serial(extents):
        post = tuple(math.ceil(e / x) for e, x in zip(extents, s))
        for t in _ref_thread(post):
            want.append((s, t))
    assert gen.root_tilings(extents) == want
