import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
sys.argv = [sys.argv[0]]
from tools.bench_extras import _pipeline
from paper_2012_07145_b200.engine import Scorer
from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights
g = _pipeline("resnet_block")
sc = Scorer(g, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
dec = sc.random_schedules(262144, 0)
h = sc.struct_hash(dec, 3).cpu().numpy().view(np.uint64)
u, c = np.unique(h, return_counts=True)
c = np.sort(c)[::-1]
print("buckets", len(u), "largest", c[:10], "sum top10", c[:10].sum())
