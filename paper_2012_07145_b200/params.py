"""Machine model, prune thresholds and cost-model weights on the host.

Same field names, defaults and file formats as the reference
(`MachineParams` machine.py:14-68, `Thresholds` options.py:60-87,
`CostModelWeights` / weights text format v1 costmodel.py:183-268), so either
the reference objects or these can be handed to the packers.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

ALGO_DIM = 10
SCHED_DIM = 56
NUM_COEFFICIENTS = 30
TENSOR_NAMES = ("algo_w", "algo_b", "sched_w", "sched_b", "head_w", "head_b", "out_w", "out_b")


@dataclass(frozen=True)
class MachineParams:
    warp_size: int = 32
    num_sms: int = 80
    max_threads_per_block: int = 1024
    max_active_warps_per_sm: int = 64
    max_active_blocks_per_sm: int = 32
    shared_mem_per_block_limit: int = 48 * 1024
    shared_mem_per_sm: int = 96 * 1024
    registers_per_thread_budget: int = 255
    global_transaction_bytes: int = 32
    shared_banks: int = 32
    bank_width_bytes: int = 4
    # machine-oracle throughput knobs (machine.py:26-31), not hardware limits
    compute_throughput: float = 2.5e12
    global_bandwidth: float = 900e9
    shared_bandwidth: float = 9e12
    kernel_launch_overhead: float = 5e-6

    @property
    def register_bytes_per_thread(self) -> int:
        return self.registers_per_thread_budget * 4

    def override(self, **kw):
        return replace(self, **{k: v for k, v in kw.items() if v is not None})


@dataclass(frozen=True)
class Thresholds:
    recompute_factor: float = 8.0
    min_blocks_per_sm_factor: float = 2.0
    warp_utilization_floor: float = 0.25
    unroll_budget: int = 64
    thread_alloc_bytes: int = 256


DEFAULT_THRESHOLDS = Thresholds()
OPEN_THRESHOLDS = Thresholds(recompute_factor=1e9, min_blocks_per_sm_factor=0.0,
                             warp_utilization_floor=0.0, unroll_budget=64,
                             thread_alloc_bytes=10 ** 9)


def _shapes(embed, hidden):
    return {"algo_w": (ALGO_DIM, embed), "algo_b": (embed,),
            "sched_w": (SCHED_DIM, embed), "sched_b": (embed,),
            "head_w": (2 * embed, hidden), "head_b": (hidden,),
            "out_w": (hidden, NUM_COEFFICIENTS), "out_b": (NUM_COEFFICIENTS,)}


class CostModelWeights:
    """Eight fp64 tensors of the two-tower coefficient network."""

    def __init__(self, tensors: dict, version: int = 1):
        try:
            embed, hidden = tensors["algo_b"].shape[0], tensors["head_b"].shape[0]
        except KeyError as e:
            raise ValueError(f"missing weight tensor {e}") from None
        for n, shp in _shapes(embed, hidden).items():
            t = tensors.get(n)
            if t is None or tuple(t.shape) != shp:
                raise ValueError(f"weight tensor {n} must have shape {shp}")
            if not np.all(np.isfinite(t)):
                raise ValueError(f"weight tensor {n} contains non-finite values")
        self.tensors = {n: np.asarray(tensors[n], dtype=np.float64) for n in TENSOR_NAMES}
        self.version = version

    @property
    def embed_dim(self):
        return self.tensors["algo_b"].shape[0]

    @property
    def hidden_dim(self):
        return self.tensors["head_b"].shape[0]


def init_weights(seed: int = 0, embed_dim: int = 32, hidden_dim: int = 64) -> CostModelWeights:
    """He-normal init, zero biases, out_b = -2 (same draws as costmodel.py:223-235)."""
    rng = np.random.default_rng(seed)
    t = {}
    for n, shp in _shapes(embed_dim, hidden_dim).items():
        t[n] = np.zeros(shp) if n.endswith("_b") else rng.normal(0.0, math.sqrt(2.0 / shp[0]), size=shp)
    t["out_b"] += -2.0
    return CostModelWeights(t)


def load_weights(path) -> CostModelWeights:
    """Weights text format v1 (costmodel.py:238-268)."""
    with open(path, encoding="utf-8") as fh:
        lines = [ln.strip() for ln in fh if ln.strip()]
    head = lines[0].split()
    if head[:1] != ["gpusched-cost-model"]:
        raise ValueError(f"{path}: not a cost model weights file")
    if int(head[1]) != 1:
        raise ValueError(f"{path}: weights version {head[1]}, expected 1")
    t = {}
    for i in range(1, len(lines), 2):
        parts = lines[i].split()
        if parts[0] != "tensor":
            raise ValueError(f"{path}: expected tensor header")
        t[parts[1]] = np.array([float(x) for x in lines[i + 1].split()]).reshape(
            tuple(int(d) for d in parts[2:]))
    return CostModelWeights(t)


def save_weights(w, path):
    out = [f"gpusched-cost-model {getattr(w, 'version', 1)}"]
    for n in TENSOR_NAMES:
        a = w.tensors[n]
        out.append(f"tensor {n} {' '.join(str(d) for d in a.shape)}")
        out.append(" ".join(f"{v:.17g}" for v in a.ravel()))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(out) + "\n")
