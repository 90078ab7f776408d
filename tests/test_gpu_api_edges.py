"""C-ABI edge cases on the device: empty batches, argument errors reported
(never a crash), structurally illegal decision logs raised at gs_check like
the reference's ScheduleError, and a candidate batch that reuses the
pipeline after an error."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import PARAMS, candidate_set, weights  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _scorer(name="stencil_chain"):
    from paper_2012_07145_b200.engine import Scorer
    cs = candidate_set(name)
    return cs, Scorer(cs.graph, PARAMS, cs.thresholds, weights())


def test_empty_batches(dev):
    cs, sc = _scorer()
    dec = sc.upload(cs.decisions[:1])[:0]
    f = sc.featurize(dec)
    total, _, _ = sc.cost(f)
    assert total.numel() == 0
    assert sc.struct_hash(dec, 3).numel() == 0
    rt, sp, st = sc.simulate(dec)
    assert rt.numel() == sp.numel() == st.numel() == 0
    sc.check()


def test_argument_errors_are_reported(dev):
    from paper_2012_07145_b200 import _lib
    cs, sc = _scorer()
    with pytest.raises(_lib.GsError):
        sc.set_reuse(3)
    with pytest.raises(_lib.GsError):   # negative hash depth
        _lib.check(sc.lib.gs_struct_hash(sc.handle, None, 1, 1, -1, None, None))
    # reuse mode 2 needs row_src
    sc.set_reuse(2)
    dec = sc.upload(cs.decisions[:2])
    buf = torch.empty((2, sc.R, 56), dtype=torch.float64, device=dev)
    ints = torch.empty((2, sc.R), dtype=torch.int32, device=dev)
    nr = torch.empty((2,), dtype=torch.int32, device=dev)
    ver = torch.empty((2,), dtype=torch.uint8, device=dev)
    rc = sc.lib.gs_featurize(sc.handle, C.c_void_p(dec.data_ptr()), 2, dec.shape[1] // 16,
                             C.c_void_p(buf.data_ptr()), C.c_void_p(ints.data_ptr()), C.c_void_p(nr.data_ptr()),
                             C.c_void_p(ver.data_ptr()), None, None)
    assert rc != 0 and b"row_src" in sc.lib.gs_last_error()
    sc.set_reuse(1)
    # the pipeline still works afterwards
    f = sc.featurize(dec)
    sc.cost(f)
    sc.check()


def test_illegal_decision_log_raises(dev):
    from paper_2012_07145_b200 import _lib
    from paper_2012_07145_b200.descriptor import DECISION_DTYPE
    cs, sc = _scorer()
    arr = sc.packed.pack(cs.decisions[:2], sc.S)
    bad = arr.copy()
    bad[0, 1] = bad[0, 0]            # the same func decided twice
    sc.featurize(sc.to_device(bad))
    with pytest.raises(_lib.GsError, match="illegal decision log"):
        sc.check()
    # a clean batch afterwards is unaffected
    f = sc.featurize(sc.to_device(arr))
    total, _, _ = sc.cost(f)
    sc.check()
    assert np.isfinite(total.cpu().numpy()).all()
    assert arr.dtype == DECISION_DTYPE
