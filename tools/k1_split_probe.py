"""Probe: K1 time with feature rows (the beam step's mode) vs prune only
(resolve + prune, no rows), on the same C5 candidates."""
import os, sys, torch
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import bench
from paper_2012_07145_b200.engine import Scorer
from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights
graph, recs, _ = bench._workload(int(sys.argv[1]) if len(sys.argv) > 1 else 1000)
sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
sc.set_reuse(2)
dec = sc.to_device(recs)
f = sc.featurize(dec)
for name, fn in (("full", lambda: sc.featurize(dec, out=f)), ("prune-only", lambda: sc.prune(dec))):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        fn()
    b.record(); torch.cuda.synchronize()
    print(name, round(a.elapsed_time(b) / 3, 2), "ms")
sc.stats()
sc.prune(dec); print("prune-only stats", sc.stats())
