"""The scheduling order the device walks (descriptor.placement_info: the
schedulable funcs in reverse topological order, loopnest.py:106-109) equals
the reference's, read from the order of the reference's own phase-1 walk in
tests/golden/phase1.json.gz (CPU; the menus themselves are checked on the
GPU in tests/test_gpu_phase1.py)."""

import gzip
import json
import os

import pytest

from golden_io import PARAMS  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def gold():
    with gzip.open(os.path.join(GOLD, "phase1.json.gz"), "rt") as fh:
        return json.load(fh)


def test_schedule_order_equals_reference(gold):
    from paper_2012_07145_b200.descriptor import PackedPipeline
    from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS
    from paper_2012_07145_b200.pipeline import parse_pipeline
    for name, g in gold.items():
        graph = parse_pipeline(g["pipeline"], name)
        pp = PackedPipeline(graph, PARAMS, DEFAULT_THRESHOLDS)
        order = [pp.names[i] for i in pp.placement_info()[3]]
        funcs = [ph["func"] for ph in g["phases"]]
        half = len(funcs) // 2   # two walks: unrestricted, then restricted
        assert funcs[:half] == order == funcs[half:], name
