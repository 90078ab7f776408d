"""Beam-step expansion on the device (gs_expand_step) reproduces the host
enumeration of every phase-2 tiling (gen.expand_step, which mirrors the
reference's `_phase2_candidates`, search.py:223-235 and options.py:144-183)
record for record, for 2-D and 3-D pipelines; the host enumeration itself
is checked against the reference menus on CPU (tests/test_expand_host.py)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import PARAMS, weights  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


@pytest.mark.parametrize("name", ["c5", "unsharp", "harris", "camera_pipe"])
def test_device_expansion_matches_host(name, dev):
    from paper_2012_07145_b200 import gen
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.pipeline import builtin_pipeline
    if name == "c5":
        import bench
        from paper_2012_07145_b200.descriptor import DECISION_DTYPE
        z = np.load(bench.PARENTS_FILE)
        par = np.ascontiguousarray(z["parents"]).view(DECISION_DTYPE).reshape(len(z["parents"]), -1)[:300]
        steps = z["steps"][:300]
        graph, _, _ = bench._workload(1)
    else:
        graph = builtin_pipeline(name)
        info = gen.GraphInfo(graph)
        rng = np.random.default_rng(5)
        ps, steps = [], []
        for _ in range(40):
            d, st = info.random_step_parent(rng)
            ps.append(d)
            steps.append(st)
        par = info.pack_rows(ps, len(info.order))
        steps = np.array(steps)
    want, owner = gen.expand_step(par, steps, graph)
    sc = Scorer(graph, PARAMS, None, weights())
    pd = sc.to_device(par)
    st = torch.from_numpy(np.asarray(steps, dtype=np.int32)).to(dev)
    got, gown, offs = sc.expand_step(pd, st)
    sc.check()
    assert got.shape[0] == len(want)
    assert np.array_equal(got.cpu().numpy(), want.view(np.uint8).reshape(len(want), -1))
    assert np.array_equal(gown.cpu().numpy(), owner)
    # sizing pass skipped when the total is known
    got2, _, _ = sc.expand_step(pd, st, total=len(want))
    assert torch.equal(got, got2)
