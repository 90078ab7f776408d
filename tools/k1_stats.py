"""K1 work counters + CUDA-event time on a C5 subset: python tools/k1_stats.py [n_parents]."""
import os
import sys

import torch

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2012_07145_b200.engine import Scorer  # noqa: E402
from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights  # noqa: E402

n_par = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
graph, recs, _ = bench._workload(n_par)
sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
sc.set_reuse(int(os.environ.get("GS_REUSE", "2")))   # the beam step's mode
dec = sc.to_device(recs)
f = sc.featurize(dec)
sc.cost(f)
sc.check()
sc.stats()
for name, fn in (("K1", lambda: sc.featurize(dec, out=f)), ("K2", lambda: sc.cost(f)),
                 ("K3", lambda: sc.struct_hash(dec, 3))):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(3):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) / 3:.2f} ms for {recs.shape[0]} candidates")
st = sc.stats()
print({k: (v / 3 if k.startswith(("cand", "incr", "rows", "geo")) else v) for k, v in st.items()})
print("rows computed per candidate:", st["rows_computed"] / max(1, st["candidates"]),
      "geometries per candidate:", st["geometries"] / max(1, st["candidates"]))
ph = __import__("numpy").zeros(16, dtype="int64")
sc.lib.gs_debug_phases(__import__("ctypes").c_void_p(ph.ctypes.data))
if ph.sum():
    names = ["diff", "resolve", "prune", "row flags", "copy", "rows", "writes"]
    tot = ph[:7].sum()
    print("phases:", {n: f"{100 * v / tot:.1f}%" for n, v in zip(names, ph[:7])})
    sub = {"setup": ph[8], "unions": ph[9], "loads": ph[13], "store": ph[10], "ws": ph[11], "assembly": ph[12]}
    st = sum(sub.values())
    if st:
        print("row phases:", {n: f"{100 * v / st:.1f}%" for n, v in sub.items()})
    print("resolve cycles: sibling pre-geometry", ph[7], "sibling geometry", ph[15], "full (structure+geometry)", ph[14],
          "of resolve total", ph[1])
