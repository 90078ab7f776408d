"""The oracle's restatement of the reference machine oracle
(machine.py:108-167) reproduces the unmodified reference on every golden
candidate, bit for bit, including the errors it raises (goldens:
tests/golden/make_simulate.py)."""

import gzip
import json
import os

import pytest

from golden_io import GOLDEN, candidate_set

from oracle.machine import simulate_runtime
from paper_2012_07145_b200.params import MachineParams


def golden():
    with gzip.open(os.path.join(GOLDEN, "simulate.json.gz"), "rt") as fh:
        return json.load(fh)


@pytest.mark.parametrize("key", sorted(golden()["results"]))
def test_oracle_simulate_matches_reference(key):
    g = golden()
    mname, name = key.split("/")
    kw = g["machines"][mname]
    mp = MachineParams().override(**{k: v for k, v in kw.items() if k != "registers_per_thread_budget"})
    knobs = {"registers_per_thread_budget": kw["registers_per_thread_budget"]} if "registers_per_thread_budget" in kw \
        else None
    cs = candidate_set(name)
    for i, want in enumerate(g["results"][key]):
        if want[0] == "error":
            with pytest.raises(ValueError) as e:
                simulate_runtime(cs.graph, cs.decisions[i], mp, knobs)
            assert ("fully scheduled" in want[1]) == ("fully scheduled" in str(e.value)), (key, i)
            continue
        rt, spilled, sb = simulate_runtime(cs.graph, cs.decisions[i], mp, knobs)
        assert rt.hex() == want[0] and spilled == want[1] and sb == want[2], (key, i, rt, want)
