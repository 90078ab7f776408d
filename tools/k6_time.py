"""K6 machine-oracle throughput on C5 beam-step batches:
python tools/k6_time.py [n_parents ...]"""
import os
import sys

import torch

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2012_07145_b200.engine import Scorer  # noqa: E402
from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights  # noqa: E402

for n_par in [int(a) for a in sys.argv[1:]] or [1000, 4167]:
    graph, recs, _ = bench._workload(n_par)
    sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
    dec = sc.to_device(recs)
    sc.simulate(dec)
    sc.check()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(3):
        rt, sp, st = sc.simulate(dec)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    ok = int((st == 0).sum())
    print(f"simulate: {recs.shape[0]} candidates in {ms:.2f} ms = {recs.shape[0] / ms * 1e3:,.0f} cand/s "
          f"({ok} valid, {int((sp > 0).sum())} spilled)")
