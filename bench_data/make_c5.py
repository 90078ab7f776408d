"""Generate the C5 beam-step parents (needs a GPU for the batched prune).

    python bench_data/make_c5.py OUT.npz [n_parents] [seed]

Parents are drawn by paper_2012_07145_b200.gen.valid_step_parents with the
GPU prune verdicts (K1, verdict-only mode) on the 100-stage chain at
1024x1024; the committed file bench_data/c5_parents_seed0.npz is what both
bench arms load, so the reference arm needs no GPU to get the same inputs.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

from paper_2012_07145_b200.engine import Scorer  # noqa: E402
from paper_2012_07145_b200.gen import valid_step_parents  # noqa: E402
from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams  # noqa: E402
from paper_2012_07145_b200.pipeline import chain_source, parse_pipeline  # noqa: E402


def main():
    out = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 4167
    seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    graph = parse_pipeline(chain_source(100, 1024), "chain100")
    sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS)

    def prune(arr):
        v = sc.prune(sc.to_device(arr))
        sc.check()
        return v.cpu().numpy()

    t = time.time()
    parents, steps = valid_step_parents(graph, prune, n, seed=seed)
    print(f"{len(parents)} valid parents in {time.time() - t:.1f}s")
    np.savez_compressed(out, parents=parents.view(np.uint8).reshape(len(parents), -1),
                        steps=steps, seed=seed, pipeline="chain100@1024")


if __name__ == "__main__":
    main()
