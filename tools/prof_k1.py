"""Small K1 workload for ncu: N parents x 240 tilings of the C5 step, in the
beam step's K1 reuse mode (GS_REUSE, default 2: computed rows only)."""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2012_07145_b200.engine import Scorer  # noqa: E402
from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights  # noqa: E402

n_par = int(sys.argv[1]) if len(sys.argv) > 1 else 50
graph, recs, _ = bench._workload(n_par)
sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
sc.set_reuse(int(os.environ.get("GS_REUSE", "2")))
dec = sc.to_device(recs)
for _ in range(2):
    f = sc.featurize(dec)
    sc.cost(f)
sc.check()
print("ok", recs.shape)
