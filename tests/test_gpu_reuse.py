"""Sibling reuse in K1 is exact: on beam-step batches (parents x all tilings
of a step root, consecutive siblings) the features with reuse on are
bit-identical to reuse off, and a subsample matches the CPU oracle."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import PARAMS, weights  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _decisions(info, rec):
    from paper_2012_07145_b200.descriptor import KIND_NAME
    from paper_2012_07145_b200.schedule import Decision
    out = []
    for r in rec:
        if r["func"] == 0xFFFF:
            break
        nd = len(info.extents[int(r["func"])])
        out.append((info.names[int(r["func"])], Decision(
            KIND_NAME[int(r["kind"])],
            None if r["consumer"] == 0xFFFF else info.names[int(r["consumer"])],
            tuple(int(x) for x in r["serial"][:nd]) if r["flags"] & 1 else None,
            tuple(int(x) for x in r["thread"][:nd]) if r["flags"] & 2 else None)))
    return tuple(out)


def _run(sc, recs, reuse):
    sc.set_reuse(reuse)
    dec = sc.to_device(recs)
    f = sc.featurize(dec)
    total, _, _ = sc.cost(f)
    full, _, _ = sc.cost(f, reuse=False)
    sc.check()
    assert torch.equal(total, full), "row-reuse K2 differs from the full network pass"
    return {k: v.cpu().numpy() for k, v in f.items() if torch.is_tensor(v)}, total.cpu().numpy()


@pytest.mark.parametrize("src", ["chain100", "stencil_chain", "diamond", "conv"])
def test_reuse_is_bit_exact(src, dev):
    from paper_2012_07145_b200 import gen
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.params import OPEN_THRESHOLDS
    from golden_io import candidate_set
    if src == "chain100":
        import bench
        graph, recs, _ = bench._workload(3)
        th = None
    else:
        graph = candidate_set(src).graph
        par, _, _ = gen.random_schedules(graph, 6, seed=11)
        info = gen.GraphInfo(graph)
        steps = np.array([[i for i in range(par.shape[1]) if par[p, i]["kind"] == 0][0]
                          for p in range(len(par))])
        recs, _ = gen.expand_step(par, steps, graph)
        th = OPEN_THRESHOLDS
    sc = Scorer(graph, PARAMS, th, weights())
    on, t_on = _run(sc, recs, True)
    off, t_off = _run(sc, recs, False)
    assert np.array_equal(on["n_rows"], off["n_rows"])
    assert np.array_equal(on["verdict"], off["verdict"])
    for i in range(len(recs)):
        r = on["n_rows"][i]
        assert np.array_equal(on["feats"][i, :r], off["feats"][i, :r]), (src, i)
        assert np.array_equal(on["row_key"][i, :r], off["row_key"][i, :r])
    assert np.array_equal(t_on, t_off)
    # K3 run-head reuse: every sibling hashes like a per-candidate hash
    sc.set_reuse(True)
    d = sc.to_device(recs)
    from oracle import structure
    info0 = gen.GraphInfo(graph)
    for depth in (0, 1, 2, 3):
        hs = sc.struct_hash(d, depth).cpu().numpy().view(np.uint64)
        for i in range(0, len(recs), max(1, len(recs) // 7)):
            assert int(hs[i]) == structure.structural_hash(_decisions(info0, recs[i]), depth), (src, depth, i)
        one = np.array([sc.struct_hash(d[i:i + 1], depth).cpu().numpy().view(np.uint64)[0]
                        for i in range(0, len(recs), max(1, len(recs) // 7))])
        assert np.array_equal(one, hs[::max(1, len(recs) // 7)])
    # oracle on a strided subsample (siblings of different parents)
    from oracle import features
    info = gen.GraphInfo(graph)
    for i in range(0, len(recs), max(1, len(recs) // 5)):
        rows = features.featurize_rows(graph, _decisions(info, recs[i]), PARAMS)
        want = np.array([f for _, f, _ in rows])
        assert np.array_equal(on["feats"][i, :len(rows)], want), (src, i)


@pytest.mark.parametrize("src,parents", [("chain100", 40), ("diamond", 6)])
def test_rows_only_mode(src, parents, dev):
    """Reuse mode 2 (the beam step's mode): K1 writes only the computed rows;
    those rows, row_src, verdicts and the K2 totals equal mode 1's."""
    from paper_2012_07145_b200 import gen
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.params import OPEN_THRESHOLDS
    from golden_io import candidate_set
    if src == "chain100":
        import bench
        graph, recs, _ = bench._workload(parents)   # >= 8192 candidates: two-phase K1
        th = None
    else:
        graph = candidate_set(src).graph
        par, _, _ = gen.random_schedules(graph, parents, seed=11)
        steps = np.array([[i for i in range(par.shape[1]) if par[p, i]["kind"] == 0][0]
                          for p in range(len(par))])
        recs, _ = gen.expand_step(par, steps, graph)
        th = OPEN_THRESHOLDS
    sc = Scorer(graph, PARAMS, th, weights())
    d = sc.to_device(recs)
    sc.set_reuse(True)
    f1 = sc.featurize(d)
    t1, _, _ = sc.cost(f1)
    a = {k: v.cpu().numpy() for k, v in f1.items() if torch.is_tensor(v)}
    sc.set_reuse(2)
    f2 = sc.featurize(d)
    f2["feats"].fill_(float("nan"))   # unwritten rows must never be read
    f2 = sc.featurize(d, out=f2)
    t2, _, _ = sc.cost(f2)
    sc.check()
    b = {k: v.cpu().numpy() for k, v in f2.items() if torch.is_tensor(v)}
    for k in ("n_rows", "verdict", "row_key", "row_src"):
        assert np.array_equal(a[k], b[k]), k
    own = b["row_src"] == np.arange(len(recs))[:, None]
    own &= np.arange(sc.R)[None, :] < b["n_rows"][:, None]
    assert np.array_equal(a["feats"][own], b["feats"][own])
    assert torch.equal(t1, t2)
    with pytest.raises(ValueError):
        sc.cost(f2, reuse=False)
    # against reuse off (every row of every candidate computed from its own
    # records, no run slots, no pooled rows): the computed rows are equal,
    # every shared row's source row is equal to the row it stands for, and
    # the totals are bit-equal
    sc.set_reuse(0)
    f0 = sc.featurize(d)
    t0, _, _ = sc.cost(f0)
    sc.check()
    z = f0["feats"].cpu().numpy()
    assert np.array_equal(z[own], b["feats"][own])
    valid = np.arange(sc.R)[None, :] < b["n_rows"][:, None]
    ci, ri = np.nonzero(valid)
    assert np.array_equal(z[ci, ri], z[b["row_src"][ci, ri], ri])
    assert torch.equal(t0, t2)
    sc.set_reuse(True)


def test_prune_only_reuses_geometry_and_matches_featurize():
    """Prune-only K1 (feats == NULL, `Scorer.prune`) resolves siblings
    incrementally too, and its verdicts and row counts equal the featurizing
    pass's on a C5 sample and on every golden candidate set."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench
    from golden_io import PARAMS, available_sets, candidate_set, weights
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights
    graph, recs, _ = bench._workload(60)
    sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
    dec = sc.to_device(recs)
    want = sc.featurize(dec)["verdict"]
    sc.stats()
    got = sc.prune(dec)
    st = sc.stats()
    sc.check()
    assert torch.equal(got, want)
    # small batches split runs into ~10-candidate units: one full resolve per unit
    assert st["incremental"] >= 0.85 * len(recs)
    for name in available_sets():
        cs = candidate_set(name)
        s2 = Scorer(cs.graph, PARAMS, cs.thresholds, weights())
        d2 = s2.upload(cs.decisions)
        assert torch.equal(s2.prune(d2), s2.featurize(d2)["verdict"]), name
