"""Feature text v1 goldens from the unmodified reference: for the first
candidates of some golden sets, `gpusched.featurize.format_features` of the
reference's own features (replayed from the committed decision dumps).
Run here (the reference is importable in this container only):
  python tests/golden/make_feature_text.py"""
import gzip
import json
import os
import sys

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src")]
HERE = os.path.dirname(os.path.abspath(__file__))

from gpusched.featurize import featurize, format_features  # noqa: E402
from gpusched.loopnest import replay_schedule  # noqa: E402
from gpusched.machine import MachineParams  # noqa: E402
from gpusched.pipeline import parse_pipeline  # noqa: E402

SETS = {"blur": 4, "stencil_chain": 4, "diamond": 6, "chain2": 6, "conv": 1, "strided": 4}


def main():
    out = {}
    for name, k in SETS.items():
        with gzip.open(os.path.join(HERE, f"{name}.json.gz"), "rt") as fh:
            m = json.load(fh)
        graph = parse_pipeline(m["pipeline"], name)
        texts = []
        for dump in m["candidates"][:k]:
            st = replay_schedule(graph, dump)
            texts.append(format_features(featurize(st, graph, MachineParams())))
        out[name] = texts
    with gzip.open(os.path.join(HERE, "feature_text.json.gz"), "wt") as fh:
        json.dump(out, fh)
    print({n: len(t) for n, t in out.items()})


if __name__ == "__main__":
    main()
