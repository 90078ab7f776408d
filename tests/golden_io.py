"""Loaders for the committed golden fixtures (produced by the reference via
tests/golden/make_golden.py).  Pure data: no reference import needed."""

from __future__ import annotations

import gzip
import json
import os
from functools import lru_cache

import numpy as np

from paper_2012_07145_b200.params import MachineParams, Thresholds, load_weights
from paper_2012_07145_b200.pipeline import parse_pipeline
from paper_2012_07145_b200.schedule import parse_dump

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CANDIDATE_SETS = ("chain2", "chain3", "diamond", "self_read", "strided", "tiny_fork",
                  "blur", "conv", "stencil_chain", "chain20", "chain100")
AUTHORED = ("unsharp", "harris", "resnet_small", "camera_pipe", "local_laplacian")
SEARCHES = ("chain2", "diamond", "diamond_T", "stencil_chain", "chain16_freeze")


def available_sets():
    return [n for n in CANDIDATE_SETS + AUTHORED
            if os.path.exists(os.path.join(GOLDEN, f"{n}.npz"))]


class CandidateSet:
    def __init__(self, name):
        with gzip.open(os.path.join(GOLDEN, f"{name}.json.gz"), "rt") as fh:
            m = json.load(fh)
        arr = np.load(os.path.join(GOLDEN, f"{name}.npz"))
        self.name = name
        self.graph = parse_pipeline(m["pipeline"], name)
        self.decisions = [parse_dump(t) for t in m["candidates"]]
        self.rows = [[tuple(k) for k in r] for r in m["rows"]]
        self.prune = m["prune"]
        self.prune_open = m["prune_open"]
        self.full = m["full"]
        self.thresholds = Thresholds(**m["thresholds"])
        self.hashes = [[int(h) for h in hs] for hs in m["hashes"]]
        self.off = arr["offsets"]
        self.feats, self.algo, self.g, self.h = arr["feats"], arr["algo"], arr["g"], arr["h"]
        self.rowcost, self.total = arr["rowcost"], arr["total"]

    def __len__(self):
        return len(self.decisions)

    def cand(self, i):
        a, b = self.off[i], self.off[i + 1]
        return dict(decisions=self.decisions[i], rows=self.rows[i], feats=self.feats[a:b],
                    algo=self.algo[a:b], g=self.g[a:b], h=self.h[a:b],
                    rowcost=self.rowcost[a:b], total=self.total[i], prune=self.prune[i],
                    hashes=self.hashes[i])


@lru_cache(maxsize=None)
def candidate_set(name) -> CandidateSet:
    return CandidateSet(name)


@lru_cache(maxsize=None)
def search_trace(tag):
    with gzip.open(os.path.join(GOLDEN, f"search_{tag}.json.gz"), "rt") as fh:
        m = json.load(fh)
    m["graph"] = parse_pipeline(m["pipeline"], tag)
    for c in m["calls"]:
        c["candidates"] = [parse_dump(t) for t in c["candidates"]]
        c["beam"] = [parse_dump(t) for t in c["beam"]]
        c["memo_before"] = {(int(d), int(h)) for d, h in c["memo_before"]}
        c["memo_after"] = {(int(d), int(h)) for d, h in c["memo_after"]}
    m["final"] = [parse_dump(t) for t in m["final"]]
    return m


@lru_cache(maxsize=None)
def weights(which="seed0"):
    return load_weights(os.path.join(GOLDEN, f"weights_{which}.txt"))


PARAMS = MachineParams()


def decisions_from_records(info, rec):
    """Packed GsDecision records of one candidate -> reference-style
    ((func, Decision), ...) tuple (for the oracle)."""
    from paper_2012_07145_b200.descriptor import KIND_NAME
    from paper_2012_07145_b200.schedule import Decision
    out = []
    for r in rec:
        if r["func"] == 0xFFFF:
            break
        nd = len(info.extents[int(r["func"])])
        out.append((info.names[int(r["func"])], Decision(
            KIND_NAME[int(r["kind"])],
            None if r["consumer"] == 0xFFFF else info.names[int(r["consumer"])],
            tuple(int(x) for x in r["serial"][:nd]) if r["flags"] & 1 else None,
            tuple(int(x) for x in r["thread"][:nd]) if r["flags"] & 2 else None)))
    return tuple(out)


def search_tags():
    """Traced searches present under tests/golden (SEARCHES + C3 freeze traces)."""
    import glob
    tags = [os.path.basename(p)[len("search_"):-len(".json.gz")]
            for p in glob.glob(os.path.join(GOLDEN, "search_*.json.gz"))]
    # beams-only traces (C3 at full size, make_golden.py --c3-full) carry no
    # candidates: tests/test_gpu_c3.py replays them through the search
    return sorted(t for t in tags if not t.endswith("_b32p5"))
