"""Small K1 run for compute-sanitizer (racecheck / memcheck)."""
import os
import sys
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from golden_io import PARAMS, candidate_set, weights  # noqa: E402
from paper_2012_07145_b200.engine import Scorer  # noqa: E402
import numpy as np  # noqa: E402
cs = candidate_set(sys.argv[1] if len(sys.argv) > 1 else "chain2")
sc = Scorer(cs.graph, PARAMS, cs.thresholds, weights())
f = sc.featurize(sc.upload(cs.decisions))
sc.check()
feats = f["feats"].cpu().numpy()
bad = 0
for i in range(len(cs)):
    c = cs.cand(i)
    R = len(c["rows"])
    bad += int((feats[i, :R] != c["feats"]).any())
print("candidates with wrong features:", bad, "of", len(cs))
sc.set_reuse(False)
f = sc.featurize(sc.upload(cs.decisions))
sc.check()
feats = f["feats"].cpu().numpy()
bad = [i for i in range(len(cs)) if (feats[i, :len(cs.cand(i)["rows"])] != cs.cand(i)["feats"]).any()]
print("reuse off: wrong", bad)
sc.set_reuse(True)
f = sc.featurize(sc.upload(cs.decisions))
feats = f["feats"].cpu().numpy()
bad = [i for i in range(len(cs)) if (feats[i, :len(cs.cand(i)["rows"])] != cs.cand(i)["feats"]).any()]
print("reuse on: wrong", bad)
from paper_2012_07145_b200.schedule import schedule_dump
for i in bad[:3]:
    print(i, schedule_dump(cs.decisions[i])[:300])
    print(i - 1, schedule_dump(cs.decisions[i - 1])[:300])
