"""How much row work a run-level memo could save over K1's previous-candidate diff.

    python tools/row_memo_study.py [n_parents]

Featurizes the first n_parents runs (x 240 tilings) of the C5 step with reuse
off (every row computed), then per run and row position counts
  dirty_prev : rows whose features differ from the previous sibling's
               (the floor of K1's previous-candidate reuse),
  distinct   : distinct feature vectors at that row position in the run
               (what a perfect run-level memo would compute),
and prints K1's actual computed-row count in reuse mode 2 beside them.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2012_07145_b200.engine import Scorer  # noqa: E402
from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights  # noqa: E402

n_par = int(sys.argv[1]) if len(sys.argv) > 1 else 100
graph, recs, _ = bench._workload(n_par)
sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
dec = sc.to_device(recs)
sc.set_reuse(0)
f = sc.featurize(dec)
sc.check()
feats = f["feats"].cpu().numpy()
nrows = f["n_rows"].cpu().numpy()
keys = f["row_key"].cpu().numpy()
sc.set_reuse(2)
sc.stats()
sc.featurize(dec)
st = sc.stats()
n = feats.shape[0]
run = 240
tot_prev = tot_dist = tot_rows = 0
per_pos_prev = {}
dist_hist = []
for r0 in range(0, n - run + 1, run):
    F = feats[r0:r0 + run]
    nr = nrows[r0:r0 + run]
    assert (nr == nr[0]).all()
    R = int(nr[0])
    tot_rows += R * run
    for r in range(R):
        col = F[:, r, :]
        chg = 1 + int(np.any(col[1:] != col[:-1], axis=1).sum())
        u = len({c.tobytes() for c in col})
        tot_prev += chg
        tot_dist += u
        if chg > 1:
            k = int(keys[r0, r])
            per_pos_prev.setdefault(k >> 8, []).append((chg, u))
            dist_hist.append(u)
cand = n
print(f"candidates {cand}: rows/cand {tot_rows / cand:.2f}")
print(f"K1 computed rows/cand (reuse 2): {st['rows_computed'] / max(1, st['candidates']):.3f}  "
      f"geometries/cand {st['geometries'] / max(1, st['candidates']):.3f}")
print(f"floor of prev-diff reuse: {tot_prev / cand:.3f} rows/cand")
print(f"perfect run memo:          {tot_dist / cand:.3f} rows/cand")
print("distinct-per-run histogram of changing rows:",
      np.unique(np.array(dist_hist), return_counts=True))
