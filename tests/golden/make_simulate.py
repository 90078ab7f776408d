"""Machine-oracle goldens from the unmodified reference: `simulate_runtime`
(machine.py:108-167) of the committed golden candidates, or the error it
raises.  Run here (the reference is importable in this container only):
  python tests/golden/make_simulate.py"""
import gzip
import json
import os
import sys

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src")]
HERE = os.path.dirname(os.path.abspath(__file__))

from gpusched.loopnest import replay_schedule  # noqa: E402
from gpusched.machine import MachineParams, simulate_runtime  # noqa: E402
from gpusched.pipeline import parse_pipeline  # noqa: E402

SETS = ("chain2", "chain3", "diamond", "self_read", "strided", "tiny_fork", "blur", "conv", "stencil_chain",
        "chain20", "unsharp", "harris")
MACHINES = {"default": {}, "small_regs": {"registers_per_thread_budget": 16, "num_sms": 20}}


def main():
    out = {}
    for mname, kw in MACHINES.items():
        params = MachineParams().override(**kw)
        for name in SETS:
            path = os.path.join(HERE, f"{name}.json.gz")
            if not os.path.exists(path):
                continue
            with gzip.open(path, "rt") as fh:
                m = json.load(fh)
            graph = parse_pipeline(m["pipeline"], name)
            res = []
            for dump in m["candidates"]:
                st = replay_schedule(graph, dump)
                try:
                    r = simulate_runtime(st, graph, params)
                    res.append([r.runtime.hex(), r.spilled_registers, r.spill_bytes])
                except ValueError as e:
                    res.append(["error", str(e)])
            out[f"{mname}/{name}"] = res
    with gzip.open(os.path.join(HERE, "simulate.json.gz"), "wt") as fh:
        json.dump({"machines": MACHINES, "results": out}, fh)
    print({k: (len(v), sum(1 for r in v if r[0] == "error"), sum(1 for r in v if r[0] != "error" and r[1]))
           for k, v in out.items()})


if __name__ == "__main__":
    main()
