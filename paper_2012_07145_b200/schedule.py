"""Candidate schedules on the host: decision records and their wire formats.

A candidate is an ordered decision log `((func, Decision), ...)` exactly as
the reference `LoopNestState.decisions` holds it (`pkg/src/gpusched/loopnest.py:34-48`,
`63-127`).  The scoring path never needs more than that log, so this module
keeps only:

* `Decision` / `State` — duck-type compatible with the reference types
  (`.kind/.consumer/.serial/.thread`, `.decisions`);
* `schedule_dump` / `parse_dump` — the JSON-lines wire format of
  `loopnest.py:275-299`;
* `apply_decision` — the legality rules of `loopnest.py:178-241`, used by the
  synthetic candidate generators (tests and bench), not by the scoring path.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, replace

PLACEMENT_KINDS = ("compute_root", "fuse_at_block", "fuse_at_thread", "inline")
KIND_CODE = {k: i for i, k in enumerate(PLACEMENT_KINDS)}


class ScheduleError(Exception):
    """Structurally illegal decision (mirrors the reference exception)."""


@dataclass(frozen=True)
class Decision:
    kind: str
    consumer: str | None = None
    serial: tuple | None = None
    thread: tuple | None = None

    def __post_init__(self):
        if self.kind not in KIND_CODE:
            raise ScheduleError(f"unknown decision kind {self.kind!r}")
        if self.kind in ("fuse_at_block", "fuse_at_thread") and not self.consumer:
            raise ScheduleError(f"{self.kind} needs a consumer")
        for ext in (self.serial, self.thread):
            if ext is not None and any(e < 1 for e in ext):
                raise ScheduleError("tile extents must be >= 1")


@dataclass(frozen=True)
class State:
    """Immutable decision log over a graph (subset of `LoopNestState`)."""

    graph: object
    decisions: tuple = ()

    def decision(self, func):
        for f, d in self.decisions:
            if f == func:
                return d
        return None

    def kernel_of(self, func):
        d = self.decision(func)
        while d is not None and d.kind in ("fuse_at_block", "fuse_at_thread"):
            func = d.consumer
            d = self.decision(func)
        if d is None or d.kind == "inline":
            return None
        return func

    def effective_consumers(self, func) -> set:
        out = set()
        for c in self.graph.consumers_of(func):
            d = self.decision(c)
            if d is not None and d.kind == "inline":
                out |= self.effective_consumers(c)
            else:
                out.add(c)
        return out

    def schedulable_funcs(self) -> list:
        return [f for f in reversed(self.graph.topo_order)
                if not self.graph.func(f).is_external_input]


def apply_decision(state: State, func: str, d: Decision) -> State:
    """Append (or phase-2 re-tile) one decision, enforcing the reference's
    legality rules (`loopnest.py:178-241`)."""
    g = state.graph
    node = g.func(func)
    if node.is_external_input:
        raise ScheduleError(f"{func} is an external input")
    old = state.decision(func)
    if old is not None:
        if (old.kind == d.kind == "compute_root" and old.serial is None
                and d.serial is not None):
            _check_root_tiling(node, d)
            return replace(state, decisions=tuple(
                (f, d if f == func else x) for f, x in state.decisions))
        if d == old:
            return state
        raise ScheduleError(f"{func} is already scheduled")
    if d.kind == "inline":
        if func in g.outputs or len(node.stages) > 1 or any(
                a.producer == func for st in node.stages for a in st.accesses):
            raise ScheduleError(f"cannot inline {func}")
    elif d.kind in ("fuse_at_block", "fuse_at_thread"):
        c = d.consumer
        if func in g.outputs or c == func or c not in g:
            raise ScheduleError(f"bad fusion of {func} into {c}")
        cd = state.decision(c)
        if cd is None or cd.kind == "inline":
            raise ScheduleError(f"fusion target {c} must be scheduled and not inlined")
        eff = state.effective_consumers(func)
        if c not in eff:
            raise ScheduleError(f"{c} is not a consumer of {func}")
        if d.kind == "fuse_at_thread":
            if eff != {c}:
                raise ScheduleError(f"{func} has consumers besides {c}")
        else:
            k = state.kernel_of(c)
            if any(state.kernel_of(o) != k for o in eff):
                raise ScheduleError(f"{func} consumers span kernels")
            if d.serial is not None and len(d.serial) != node.ndim:
                raise ScheduleError("serial tiling rank mismatch")
        if d.thread is not None:
            raise ScheduleError("fused funcs never carry thread tilings")
    elif d.serial is not None:
        _check_root_tiling(node, d)
    return replace(state, decisions=state.decisions + ((func, d),))


def _check_root_tiling(node, d):
    if d.serial is None or d.thread is None:
        raise ScheduleError(f"root tiling of {node.name} needs serial and thread")
    if len(d.serial) != node.ndim or len(d.thread) != node.ndim:
        raise ScheduleError(f"tiling rank mismatch for {node.name}")
    if any(s > e for s, e in zip(d.serial, node.extents)):
        raise ScheduleError(f"serial extent exceeds domain of {node.name}")


def schedule_dump(decisions) -> str:
    """JSON-lines dump of a decision log (reference `loopnest.py:275-284`)."""
    rows = []
    for f, d in decisions:
        rows.append(json.dumps({
            "func": f, "kind": d.kind, "consumer": d.consumer,
            "serial": list(d.serial) if d.serial else None,
            "thread": list(d.thread) if d.thread else None}))
    return "\n".join(rows) + "\n"


def parse_dump(text: str) -> tuple:
    """Decision log from a JSON-lines dump (no legality replay)."""
    out = []
    for line in text.splitlines():
        if not line.strip():
            continue
        r = json.loads(line)
        out.append((r["func"], Decision(
            r["kind"], r.get("consumer"),
            tuple(r["serial"]) if r.get("serial") else None,
            tuple(r["thread"]) if r.get("thread") else None)))
    return tuple(out)
