"""K6 machine oracle (gs_simulate) equals the unmodified reference's
simulate_runtime (machine.py:108-167) bit for bit on every golden candidate,
including spills (a 16-register budget) and the two error cases the
reference raises for (goldens: tests/golden/make_simulate.py)."""

import gzip
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import GOLDEN, candidate_set, weights  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def golden():
    with gzip.open(os.path.join(GOLDEN, "simulate.json.gz"), "rt") as fh:
        return json.load(fh)


@pytest.mark.parametrize("key", sorted(golden()["results"]))
def test_gpu_simulate_matches_reference(key, dev):
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.params import MachineParams
    g = golden()
    mname, name = key.split("/")
    mp = MachineParams().override(**g["machines"][mname])
    cs = candidate_set(name)
    sc = Scorer(cs.graph, mp, cs.thresholds, weights())
    rt, sp, st = sc.simulate(sc.upload(cs.decisions))
    sc.check()
    rt, sp, st = rt.cpu().numpy(), sp.cpu().numpy(), st.cpu().numpy()
    for i, want in enumerate(g["results"][key]):
        if want[0] == "error":
            code = 2 if "fully scheduled" in want[1] else 1
            assert st[i] == code and np.isnan(rt[i]), (key, i, st[i], want)
            continue
        assert st[i] == 0, (key, i, st[i])
        assert float(rt[i]).hex() == want[0], (key, i, float(rt[i]), float.fromhex(want[0]))
        assert bool(sp[i] > 0) == want[1] and int(sp[i]) == want[2], (key, i, sp[i], want)


def test_gpu_simulate_sibling_batch(dev):
    """A beam-step batch (siblings, two-phase K1 with reuse) gives the same
    runtimes as scoring each candidate alone."""
    import bench
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams
    graph, recs, _ = bench._workload(40)
    sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, weights())
    d = sc.to_device(recs)
    rt, sp, st = sc.simulate(d)
    sc.set_reuse(0)
    rt0, sp0, st0 = sc.simulate(d)
    sc.set_reuse(1)
    sc.check()
    assert torch.equal(st, st0) and torch.equal(sp, sp0)
    ok = st == 0
    assert torch.equal(rt[ok], rt0[ok]) and int(ok.sum()) > 0


def test_simulate_runtime_drop_in(dev):
    """`evaluator.simulate_runtime` takes the reference's own states and
    params and returns what the reference's simulate_runtime returns."""
    from test_gpu_search import _reference_on_path
    if not _reference_on_path():
        pytest.skip("reference package not installed (baseline/_ref)")
    import importlib
    from gpusched.loopnest import replay_schedule
    from gpusched.machine import MachineParams, simulate_runtime as ref_sim
    from gpusched.pipeline import parse_pipeline
    ev_mod = importlib.import_module("paper_2012_07145_b200.evaluator")
    if not ev_mod.HAVE_REFERENCE:
        ev_mod = importlib.reload(ev_mod)
    for name in ("stencil_chain", "conv"):
        with gzip.open(os.path.join(GOLDEN, f"{name}.json.gz"), "rt") as fh:
            m = json.load(fh)
        graph = parse_pipeline(m["pipeline"], name)
        params = MachineParams(registers_per_thread_budget=16)
        for dump in m["candidates"][:12]:
            st = replay_schedule(graph, dump)
            try:
                want = ref_sim(st, graph, params)
            except ValueError:
                with pytest.raises(ValueError):
                    ev_mod.simulate_runtime(st, graph, params)
                continue
            got = ev_mod.simulate_runtime(st, graph, params)
            assert type(got) is type(want)
            assert (got.runtime, got.spilled_registers, got.spill_bytes) == \
                (want.runtime, want.spilled_registers, want.spill_bytes)
