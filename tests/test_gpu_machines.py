"""Non-default machine parameters (reference machine.py:14-33 are all
inputs): the compile-time-specialised transaction counters only cover the
default 32-byte segments / 32 x 4-byte banks, so these cases run the generic
K1 paths (warp-pattern classes, shared-memory residue histograms, and the
out-of-line division paths for non-power-of-two periods).  Features must
equal the CPU oracle (brute-force lane-address emulation) exactly."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import candidate_set, weights  # noqa: E402

pytestmark = pytest.mark.gpu

MACHINES = {
    "seg64": dict(global_transaction_bytes=64),
    "banks16x8": dict(shared_banks=16, bank_width_bytes=8),
    "seg24": dict(global_transaction_bytes=24),
    "banks24": dict(shared_banks=24),
    "sms132": dict(num_sms=132, shared_mem_per_sm=228 * 1024, shared_mem_per_block_limit=227 * 1024),
}


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


@pytest.mark.parametrize("machine", sorted(MACHINES))
@pytest.mark.parametrize("name,limit", [("chain2", 40), ("diamond", 40), ("stencil_chain", 16), ("blur", 24),
                                        ("conv", 4), ("strided", 30)])
def test_generic_machine_matches_oracle(machine, name, limit, dev):
    from oracle import costing, features
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.params import MachineParams
    mp = MachineParams().override(**MACHINES[machine])
    cs = candidate_set(name)
    decs = cs.decisions[:limit]
    sc = Scorer(cs.graph, mp, cs.thresholds, weights())
    f = sc.featurize(sc.upload(decs))
    total, _, _ = sc.cost(f)
    sc.check()
    feats = f["feats"].cpu().numpy()
    ver = f["verdict"].cpu().numpy()
    tot = total.cpu().numpy()
    codes = {None: 0, "excessive_recompute": 1, "idle_sms": 2, "poor_warp_utilization": 3,
             "serial_too_large": 4, "thread_alloc_dynamic_or_large": 5, "hardware_limit": 6}
    for i, d in enumerate(decs):
        rows = features.featurize_rows(cs.graph, d, mp)
        want = np.array([fv for _, fv, _ in rows])
        bad = np.argwhere(feats[i, :len(rows)] != want)
        assert bad.size == 0, (machine, name, i, [(rows[r][0], features.FEATURES[k], feats[i, r, k], want[r, k])
                                                  for r, k in bad[:4]])
        want_total, _, _ = costing.score(cs.graph, d, mp, weights().tensors)
        assert tot[i] == pytest.approx(want_total, rel=1e-9)
        assert ver[i] == codes[costing.prune_reason(cs.graph, d, mp, cs.thresholds)]
