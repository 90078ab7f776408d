"""Seam-3 drop-ins of the reference cost model, computed on the B200.

Same names, arguments, return types and errors as the reference's public
functions (re-exported by `gpusched/__init__.py:16-27`; SURVEY §8(b) seam 3):

* `featurize(state, graph, params)`            featurize.py:275-303  (K1)
* `predict_coefficients(algo, sched, weights)` costmodel.py:316-324  (K7 gs_predict)
* `stage_cost(f, c)` / `CostBreakdown`         costmodel.py:34-115   (K7, bit-exact for given c)
* `pipeline_cost(feats, weights)`              costmodel.py:327-337  (K7, one launch per call)
* `train(dataset, hyper, init)`                costmodel.py:391-432  (K7 gs_train: every epoch in one launch)

These are what the reference CLI `predict` / `featurize` commands and the
autotune retrain loop call (cli.py:102-128, driver.py:209-220).  When the
reference package is importable, its own dataclasses (`ScheduleFeatures`,
`AlgorithmFeatures`, `CostBreakdown`, `TrainResult`, `CostModelWeights`)
are returned, so callers see the types they expect; otherwise local mirrors
with the same fields are used.  There is no CPU fallback: every number comes
from libgs_sched.so.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .featurefmt import FEATURE_ORDER
from .params import ALGO_DIM, NUM_COEFFICIENTS, SCHED_DIM, TENSOR_NAMES

try:  # the reference's own types, when the user has it installed
    from gpusched.costmodel import CostBreakdown as _RefBreakdown  # type: ignore
    from gpusched.costmodel import TrainConfig as _RefTrainConfig  # type: ignore
    from gpusched.costmodel import TrainResult as _RefTrainResult  # type: ignore
    from gpusched.featurize import AlgorithmFeatures as _RefAlgo  # type: ignore
    from gpusched.featurize import ScheduleFeatures as _RefSched  # type: ignore
    HAVE_REFERENCE = True
except Exception:  # pragma: no cover - standalone use
    HAVE_REFERENCE = False


@dataclass(frozen=True)
class _CostBreakdown:   # mirror of costmodel.py:34-46
    compute: float
    load: float
    store: float
    malloc: float
    parallelism: float
    working_set: float

    @property
    def total(self) -> float:
        return (self.compute + self.store + self.load + self.malloc + self.parallelism + self.working_set)


@dataclass
class _TrainConfig:     # mirror of costmodel.py:369-374
    learning_rate: float = 1e-3
    momentum: float = 0.9
    epochs: int = 100
    seed: int = 0


@dataclass
class _TrainResult:     # mirror of costmodel.py:377-381
    weights: object
    final_loss: float
    loss_history: list = field(default_factory=list)


@dataclass(frozen=True)
class _AlgorithmFeatures:   # mirror of featurize.py:42-58
    op_counts: tuple
    num_accesses: float
    mean_window_volume: float
    elem_bytes: float

    def to_vector(self):
        return np.array(self.op_counts + (self.num_accesses, self.mean_window_volume, self.elem_bytes),
                        dtype=np.float64)


class _ScheduleFeatures:    # mirror of featurize.py:78-150 (named fields in FEATURE_ORDER)
    def __init__(self, **kw):
        for name in FEATURE_ORDER:
            setattr(self, name, float(kw.get(name, 0.0)))
        self.algorithm = kw.get("algorithm")

    def to_vector(self):
        return np.array([getattr(self, n) for n in FEATURE_ORDER], dtype=np.float64)


if HAVE_REFERENCE:
    CostBreakdown, TrainConfig, TrainResult = _RefBreakdown, _RefTrainConfig, _RefTrainResult
    AlgorithmFeatures, ScheduleFeatures = _RefAlgo, _RefSched
else:
    CostBreakdown, TrainConfig, TrainResult = _CostBreakdown, _TrainConfig, _TrainResult
    AlgorithmFeatures, ScheduleFeatures = _AlgorithmFeatures, _ScheduleFeatures


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _device():
    if not torch.cuda.is_available():
        raise _lib.GsError("no CUDA device: the cost model runs only on the GPU")
    return torch.device("cuda")


def _st():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def pack_weights(weights) -> np.ndarray:
    """The eight tensors, raveled and concatenated in the reference order
    (the packed layout of gs_predict / gs_train)."""
    return np.concatenate([np.asarray(weights.tensors[n], dtype=np.float64).ravel() for n in TENSOR_NAMES])


def unpack_weights(flat: np.ndarray, like):
    """Inverse of pack_weights, as an object of `like`'s class."""
    t, o = {}, 0
    for n in TENSOR_NAMES:
        shp = like.tensors[n].shape
        k = int(np.prod(shp))
        t[n] = flat[o:o + k].reshape(shp).copy()
        o += k
    return type(like)(t, version=getattr(like, "version", 1))


def _dims(weights):
    return int(weights.tensors["algo_b"].shape[0]), int(weights.tensors["head_b"].shape[0])


def _predict(algo, sched, weights=None, coeffs=None, breakdown=True):
    """gs_predict over row arrays: (coeffs [n, 30] or None, breakdown [n, 7] or None)."""
    dev = _device()
    lib = _lib.load()
    n = sched.shape[0]
    E, H = _dims(weights) if weights is not None else (1, 1)
    w = torch.from_numpy(pack_weights(weights)).to(dev) if weights is not None else None
    a = torch.from_numpy(np.ascontiguousarray(algo, dtype=np.float64)).to(dev) if algo is not None else None
    s = torch.from_numpy(np.ascontiguousarray(sched, dtype=np.float64)).to(dev)
    cin = torch.from_numpy(np.ascontiguousarray(coeffs, dtype=np.float64)).to(dev) if coeffs is not None else None
    cout = torch.empty((max(1, n), NUM_COEFFICIENTS), dtype=torch.float64, device=dev) if coeffs is None else None
    bd = torch.empty((max(1, n), 7), dtype=torch.float64, device=dev) if breakdown else None
    _lib.check(lib.gs_predict(_p(w), E, H, _p(a), _p(s), _p(cin), n, _p(cout), _p(bd), _st()))
    return (cout[:n].cpu().numpy() if cout is not None else None), (bd[:n].cpu().numpy() if bd is not None else None)


def predict_coefficients(algo_features, schedule_features, weights) -> np.ndarray:
    """Positive coefficient vector for one stage (costmodel.py:316-324)."""
    if hasattr(algo_features, "to_vector"):
        algo_features = algo_features.to_vector()
    if hasattr(schedule_features, "to_vector"):
        schedule_features = schedule_features.to_vector()
    xa = np.asarray(algo_features, dtype=np.float64)
    xs = np.asarray(schedule_features, dtype=np.float64)
    if xa.shape != (ALGO_DIM,) or xs.shape != (SCHED_DIM,):   # _forward's check (costmodel.py:279-282)
        raise ValueError(f"feature dims {xa.shape}/{xs.shape} do not match weights version "
                         f"{getattr(weights, 'version', 1)} ({ALGO_DIM}/{SCHED_DIM})")
    c, _ = _predict(xa[None], xs[None], weights, breakdown=False)
    return c[0]


def _breakdown(row) -> object:
    return CostBreakdown(compute=float(row[0]), load=float(row[1]), store=float(row[2]), malloc=float(row[3]),
                         parallelism=float(row[4]), working_set=float(row[5]))


def stage_cost(f, c):
    """Closed-form per-stage cost for one coefficient vector (costmodel.py:50-115)."""
    c = np.asarray(c, dtype=np.float64)
    if c.shape != (NUM_COEFFICIENTS,):
        raise ValueError(f"expected {NUM_COEFFICIENTS} coefficients, got {c.shape}")
    if np.any(c <= 0):
        raise ValueError("coefficients must be strictly positive")
    _, bd = _predict(None, f.to_vector()[None], coeffs=c[None])
    return _breakdown(bd[0])


def pipeline_cost(feats: dict, weights):
    """Total predicted cost plus per-stage breakdowns (costmodel.py:327-337):
    every stage's coefficients and breakdown in one launch; the total adds
    the breakdown totals in the dict's order, as the reference does."""
    keys = list(feats)
    if not keys:
        return 0.0, {}
    algo = np.stack([feats[k].algorithm.to_vector() for k in keys])
    sched = np.stack([feats[k].to_vector() for k in keys])
    if algo.shape[1] != ALGO_DIM or sched.shape[1] != SCHED_DIM:
        raise ValueError(f"feature dims {algo.shape[1:]}/{sched.shape[1:]} do not match weights version "
                         f"{getattr(weights, 'version', 1)} ({ALGO_DIM}/{SCHED_DIM})")
    _, bd = _predict(algo, sched, weights)
    breakdown = {}
    total = 0.0
    for k, row in zip(keys, bd):
        b = _breakdown(row)
        breakdown[k] = b
        total += b.total
    return total, breakdown


def featurize(state, graph, params, _concrete=None, thresholds=None) -> dict:
    """Per-(func, stage) ScheduleFeatures of one state (featurize.py:275-303),
    from K1: rows in the reference's insertion order, `algorithm` set to the
    stage's AlgorithmFeatures (`_concrete` is accepted and ignored)."""
    from .evaluator import scorer_for
    from .params import DEFAULT_THRESHOLDS
    sc = scorer_for(graph, params, thresholds or DEFAULT_THRESHOLDS, None)
    dec = sc.upload([state])
    f = sc.featurize(dec)
    sc.check()
    n = int(f["n_rows"][0].item())
    keys = sc.packed.row_keys(f["row_key"][0, :n].cpu().numpy())
    rows = f["feats"][0, :n].cpu().numpy()
    out = {}
    for k, v in zip(keys, rows):
        a = sc.packed.algo[sc.packed.stage_index[k]]
        algo = AlgorithmFeatures(op_counts=tuple(float(x) for x in a[:ALGO_DIM - 3]), num_accesses=float(a[-3]),
                                 mean_window_volume=float(a[-2]), elem_bytes=float(a[-1]))
        fs = ScheduleFeatures(**{name: float(x) for name, x in zip(FEATURE_ORDER, v)})
        fs.algorithm = algo
        out[tuple(k)] = fs
    return out


def train(dataset: list, hyper=None, init=None):
    """SGD with momentum on squared log-cost error (costmodel.py:391-432),
    all epochs in one persistent-CTA launch (gs_train).  The per-epoch
    sample order is the reference's `default_rng(seed).permutation` stream;
    gradients are summed over stages in the reference's order."""
    from .params import init_weights
    if len(dataset) < 2 or len({s.runtime for s in dataset}) < 2:
        raise ValueError("training needs >= 2 samples with >= 2 distinct runtimes")
    hyper = hyper or TrainConfig()
    w0 = init if init is not None else init_weights(hyper.seed)
    E, H = _dims(w0)
    rng = np.random.default_rng(hyper.seed)
    order = np.stack([rng.permutation(len(dataset)) for _ in range(hyper.epochs)]).astype(np.int32) \
        if hyper.epochs > 0 else np.zeros((0, len(dataset)), dtype=np.int32)
    for s in dataset:   # a sample without stages predicts 0: the reference raises on it
        if not s.stages:
            raise ValueError(f"non-finite or non-positive predicted cost for sample "
                             f"{getattr(s, 'pipeline_id', '')}/{getattr(s, 'schedule_id', '')}")
    rows = [st for s in dataset for st in s.stages]
    off = np.zeros(len(dataset) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(s.stages) for s in dataset])
    max_rows = int(max(len(s.stages) for s in dataset))
    if max_rows > 1024:
        raise ValueError("at most 1024 stages per training sample")
    dev = _device()
    lib = _lib.load()
    t = lambda a, dt=np.float64: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)  # noqa: E731
    algo = t(np.stack([np.asarray(r[0], dtype=np.float64) for r in rows]))
    sched = t(np.stack([np.asarray(r[1], dtype=np.float64) for r in rows]))
    g = t(np.stack([np.asarray(r[2], dtype=np.float64) for r in rows]))
    h = t(np.array([float(r[3]) for r in rows]))
    rt = t(np.array([float(s.runtime) for s in dataset]))
    ro = t(off, np.int64)
    od = t(order.reshape(-1) if order.size else np.zeros(1, dtype=np.int32), np.int32)
    w = t(pack_weights(w0))
    wsb = lib.gs_train_workspace_bytes(E, H, max_rows)
    ws = torch.empty((max(1, wsb),), dtype=torch.uint8, device=dev)
    hist = torch.zeros((max(1, hyper.epochs),), dtype=torch.float64, device=dev)
    status = torch.zeros((1,), dtype=torch.int32, device=dev)
    _lib.check(lib.gs_train(_p(w), E, H, _p(algo), _p(sched), _p(g), _p(h), _p(ro), _p(rt), _p(od), len(dataset),
                            int(hyper.epochs), float(hyper.learning_rate), float(hyper.momentum), max_rows, _p(ws),
                            wsb, _p(hist), _p(status), _st()))
    bad = int(status.item())
    if bad:
        s = dataset[bad - 1]
        raise ValueError(f"non-finite or non-positive predicted cost for sample "
                         f"{getattr(s, 'pipeline_id', '')}/{getattr(s, 'schedule_id', '')}")
    history = hist[:hyper.epochs].cpu().tolist()
    weights = unpack_weights(w.cpu().numpy(), w0)
    return TrainResult(weights=weights, final_loss=history[-1], loss_history=history)
