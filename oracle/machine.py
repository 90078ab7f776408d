"""CPU restatement of the reference machine oracle `simulate_runtime`
(reference machine.py:108-167) over the oracle's own resolve and features.

TEST INFRASTRUCTURE ONLY: the checker for K6 (`gs_simulate`); the product
path never calls it.  Pinned to the reference by tests/golden/simulate.json.gz
(tests/golden/make_simulate.py runs the unmodified reference)."""

from __future__ import annotations

from .features import FIDX, featurize_rows
from .geometry import resolve_geometry

# machine.py:26-31 (oracle-only throughput knobs) and :24 (register budget)
ORACLE_DEFAULTS = dict(registers_per_thread_budget=255, compute_throughput=2.5e12, global_bandwidth=900e9,
                       shared_bandwidth=9e12, kernel_launch_overhead=5e-6)


def simulate_runtime(graph, decisions, mp, knobs=None):
    """(runtime, spilled_registers, spill_bytes); raises ValueError where the
    reference does (not fully scheduled, hardware limit violation)."""
    k = {**ORACLE_DEFAULTS, **(knobs or {})}
    dmap = dict(decisions)
    for f in graph.funcs:                                                     # loopnest.py:112-124
        if f.is_external_input:
            continue
        d = dmap.get(f.name)
        if (d is None or (d.kind == "compute_root" and (d.serial is None or d.thread is None))
                or (d.kind == "fuse_at_block" and d.serial is None)):
            raise ValueError("oracle requires a fully scheduled state")      # machine.py:121-122
    geos, kernels = resolve_geometry(graph, decisions)
    for kern in kernels.values():                                             # machine.py:91-105
        if kern.threads > mp.max_threads_per_block or kern.shared_bytes > mp.shared_mem_per_block_limit:
            raise ValueError("hardware limit violation")
    rows = featurize_rows(graph, decisions, mp)
    budget = k["registers_per_thread_budget"] * 4
    total, spilled, spill_bytes = 0.0, False, 0
    F = FIDX
    for owner, kern in kernels.items():                                       # machine.py:134-166
        work = gbytes = sbytes = 0.0
        occ = 1.0
        kspill = 0
        for (func, _si), f, algo in rows:
            if geos[func].kernel != owner:
                continue
            ops = float(sum(int(x) for x in algo[:7]))
            work += f[F["num_scalars"]] * (1.0 + ops)
            gbytes += f[F["num_blocks"]] * (f[F["num_global_mem_loads_per_block"]]
                                            + f[F["num_global_mem_stores_per_block"]]) * mp.global_transaction_bytes
            sbytes += f[F["num_blocks"]] * (f[F["num_shared_mem_loads_per_block"]]
                                            + f[F["num_shared_mem_stores_per_block"]]) \
                * mp.shared_banks * mp.bank_width_bytes
            occ = min(occ, f[F["max_warp_occupancy"]])
            ws = int(f[F["working_set_at_thread"]])
            if ws > budget:
                kspill = max(kspill, ws - budget)
        balance = min(1.0, kern.n_blocks / (2.0 * mp.num_sms))
        util = max(1e-3, occ * balance)
        ct = work / (k["compute_throughput"] * util)
        mt = gbytes / k["global_bandwidth"] + sbytes / k["shared_bandwidth"]
        t = max(ct, mt)
        if kspill > 0:
            spilled = True
            spill_bytes += kspill
            t *= 2.0 + kspill / budget
        total += t + k["kernel_launch_overhead"]
    return total, spilled, spill_bytes
