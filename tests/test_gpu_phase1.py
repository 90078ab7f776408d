"""GPU phase-1 expansion (gs_expand_phase1) against the
unmodified reference's `_phase1_candidates` (tests/golden/phase1.json.gz,
tests/golden/make_phase1_golden.py): 12 pipelines, random walks through
every placement phase, unrestricted and with the freeze pre-pass's
restrict_placements — every candidate's decision records bit for bit, in
the reference's order, with the right parent."""

import gzip
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import PARAMS  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def gold():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with gzip.open(os.path.join(GOLD, "phase1.json.gz"), "rt") as fh:
        return json.load(fh)


NAMES = ("diamond", "tiny_fork", "chain3", "stencil_chain", "chain20", "unsharp", "harris", "camera_pipe",
         "local_laplacian", "resnet_small", "blur", "conv")


@pytest.mark.parametrize("name", NAMES)
def test_phase1_matches_reference(gold, name):
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.pipeline import parse_pipeline
    from paper_2012_07145_b200.schedule import parse_dump
    g = gold[name]
    graph = parse_pipeline(g["pipeline"], name)
    sc = Scorer(graph, PARAMS)
    S = sc.S
    for k, ph in enumerate(g["phases"]):
        parents = [parse_dump(t) for t in ph["parents"]]
        want = sc.packed.pack([parse_dump(t) for t in ph["candidates"]], S)
        pd = torch.from_numpy(sc.packed.pack(parents, S).view(np.uint8).reshape(len(parents), -1)).cuda()
        out, owner, offs = sc.expand_phase1(pd, ph["func"], restrict=ph["restrict"])
        sc.check()
        assert np.diff(offs.cpu().numpy()).tolist() == ph["counts"], (name, k, ph["func"])
        got = out.cpu().numpy().view(want.dtype).reshape(want.shape)
        assert np.array_equal(got, want), (name, k, ph["func"])
        assert owner.cpu().tolist() == [i for i, c in enumerate(ph["counts"]) for _ in range(c)]


def test_phase1_errors(gold):
    from paper_2012_07145_b200._lib import GsError
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.pipeline import parse_pipeline
    from paper_2012_07145_b200.schedule import parse_dump
    g = gold["diamond"]
    graph = parse_pipeline(g["pipeline"], "diamond")
    sc = Scorer(graph, PARAMS)
    ph = g["phases"][1]
    # expanding a func every parent already schedules is illegal
    done = g["phases"][0]["func"]
    parents = [parse_dump(t) for t in ph["parents"]]
    pd = torch.from_numpy(sc.packed.pack(parents, sc.S).view(np.uint8).reshape(len(parents), -1)).cuda()
    sc.expand_phase1(pd, done)
    with pytest.raises(GsError):
        sc.check()
    with pytest.raises((GsError, KeyError)):
        sc.expand_phase1(pd, "no_such_func")


@pytest.mark.parametrize("name", NAMES)
def test_random_schedules_match_reference(gold, name):
    """gs_random_schedules(seed, i) == the reference `_random_schedule(graph,
    default_rng((seed, i)))`, record for record."""
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.pipeline import parse_pipeline
    from paper_2012_07145_b200.schedule import parse_dump
    g = gold[name]
    graph = parse_pipeline(g["pipeline"], name)
    sc = Scorer(graph, PARAMS)
    want = sc.packed.pack([parse_dump(t) for t in g["random"]], sc.S)
    out = sc.random_schedules(len(g["random"]), g["random_seed"])
    sc.check()
    got = out.cpu().numpy().view(want.dtype).reshape(want.shape)
    assert np.array_equal(got, want), name
    # a later window of the same stream
    tail = sc.random_schedules(8, g["random_seed"], first=40)
    assert np.array_equal(tail.cpu().numpy().view(want.dtype).reshape(8, -1), want[40:48])
