"""Exercise every kernel of the path once, small enough for compute-sanitizer:

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_step.py

K3 (pass depth + memo), K1 in both schedules (a 9,600-candidate C5 subset:
two-phase run heads + sibling slices; a 720-candidate one: run-aligned
units), K2 (row reuse and the dense basis path), K4, K5 (T = 0 and the
Gumbel path), the device expansion and K6 (machine oracle)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2012_07145_b200 import shard  # noqa: E402
from paper_2012_07145_b200.engine import TIE_BAND, Scorer  # noqa: E402
from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights  # noqa: E402

graph, recs, _ = bench._workload(40)
sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [len(recs), 720]
for n in sizes:
    dec = sc.to_device(recs[:n])
    plan = shard.StepPlan(sc, n, 1, 0, bench.PASS_INDEX, bench.PHASE_SEED, 8, 2.0, bench.NUM_PASSES, TIE_BAND)
    out = plan.run(dec, rejects=True)
    fl = [int(x) for x in out["memo"][bench.PASS_INDEX - 1].cpu().numpy().view(np.uint64)[:5]]
    out2 = plan.run(dec, flagged=fl, temperature=0.5, rejects=True)
    sc.check()
    print(n, "beam", out["beam"][:4], out2["beam"][:4])
# dense K2 with the basis, K1 reuse 1
dec = sc.to_device(recs[:300])
f = sc.featurize(dec)
sc.cost(f, rows=True, basis=True)
# K6 machine oracle
sc.simulate(dec[:64])
# device expansion
z = np.load(bench.PARENTS_FILE)
par = torch.as_tensor(np.ascontiguousarray(z["parents"][:6]), device="cuda")
st = torch.as_tensor(z["steps"][:6].astype(np.int32), device="cuda")
sc.expand_step(par, st)
sc.check()
torch.cuda.synchronize()
print("sanitize_step ok")
