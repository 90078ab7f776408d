"""Golden phase-1 expansions written by the UNMODIFIED reference:

    python tests/golden/make_phase1_golden.py

For each pipeline, a random walk through the placement phases: at every
func in scheduling order, the reference `_phase1_candidates` (search.py:204-220
over options.py:103-162 and loopnest.py:178-241) of up to 6 beam states,
then a random subset of the candidates becomes the next beam.  Two
configurations: unrestricted, and the freeze pre-pass's
restrict_placements=("compute_root", "inline") (search.py:329).  Plus the
reference test suite's `_random_schedule(graph, default_rng((1234, i)))`
(tests/test_acceptance.py:136-160) for i < 48 — what gs_random_schedules
must reproduce.
Output: phase1.json.gz — per pipeline: text + phases (func, restrict,
parents and candidates as schedule_dump lines) + random schedules."""

from __future__ import annotations

import gzip
import json
import os
import sys
from dataclasses import replace

import numpy as np

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src"), os.path.join(REF, "tests")]
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from gpusched.loopnest import initial_state, schedule_dump  # noqa: E402
from gpusched.pipeline import parse_pipeline  # noqa: E402
from gpusched.search import SearchConfig, _phase1_candidates  # noqa: E402
from test_acceptance import _random_schedule  # noqa: E402

NAMES = ("diamond", "tiny_fork", "chain3", "stencil_chain", "chain20", "unsharp", "harris", "camera_pipe",
         "local_laplacian", "resnet_small", "blur", "conv")


def walk(graph, config, rng, beam_size=6):
    beam = [initial_state(graph)]
    phases = []
    for func in beam[0].schedulable_funcs():
        cands_per = [_phase1_candidates(s, func, graph, config) for s in beam]
        phases.append({"func": func, "restrict": list(config.restrict_placements) if config.restrict_placements else None,
                       "parents": [schedule_dump(s) for s in beam],
                       "counts": [len(c) for c in cands_per],
                       "candidates": [schedule_dump(c) for cs in cands_per for c in cs]})
        allc = [c for cs in cands_per for c in cs]
        pick = rng.choice(len(allc), size=min(beam_size, len(allc)), replace=False)
        beam = [allc[i] for i in sorted(pick)]
    return phases


def main():
    out = {}
    for name in NAMES:
        with gzip.open(os.path.join(HERE, f"{name}.json.gz"), "rt") as fh:
            text = json.load(fh)["pipeline"]
        graph = parse_pipeline(text, name)
        rng = np.random.default_rng(11)
        base = SearchConfig(seed=0)
        phases = walk(graph, base, rng) + walk(graph, replace(base, restrict_placements=("compute_root", "inline")),
                                               rng)
        rand = [schedule_dump(_random_schedule(graph, np.random.default_rng((1234, i)))) for i in range(48)]
        out[name] = {"pipeline": text, "phases": phases, "random_seed": 1234, "random": rand}
        print(name, len(phases), "phases,", sum(len(p["candidates"]) for p in phases), "candidates")
    with gzip.open(os.path.join(HERE, "phase1.json.gz"), "wt") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
