"""K2's two row-cost kernels agree bit for bit: the FP64 tensor-core kernel
(cost_rows_mma_kernel, DMMA GEMMs over 32 rows per warp) and the scalar
one-row-per-lane kernel (cost_rows_kernel, selected with GS_K2_SCALAR=1) on
the same 20-parent C5 beam step.  The switch is read once per process, so
each path runs in its own interpreter."""

import hashlib
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, sys.argv[1])
import bench, torch
from paper_2012_07145_b200.engine import Scorer
from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights
graph, recs, _ = bench._workload(20)
sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
dec = sc.to_device(recs)
sc.set_reuse(2)
f = sc.featurize(dec)
total, rows, _ = sc.cost(f, rows=True)
sc.check()
h = hashlib.sha256(total.cpu().numpy().tobytes() + rows.cpu().numpy().tobytes()).hexdigest()
print("K2", total.numel(), h)
"""


def _run(scalar):
    env = dict(os.environ)
    env.pop("GS_K2_SCALAR", None)
    if scalar:
        env["GS_K2_SCALAR"] = "1"
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], capture_output=True, text=True, env=env,
                       cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("K2 ")][-1]
    return line.split()[1:]


def test_dmma_and_scalar_row_kernels_bit_identical():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n_mma, h_mma = _run(False)
    n_sc, h_sc = _run(True)
    assert int(n_mma) == int(n_sc) == 20 * 240
    assert h_mma == h_sc, "DMMA and scalar K2 row kernels differ"
