"""What sibling reuse hides, and the BASELINE configs beyond C5 (VERDICT r01
item 3): one JSON line per workload, each the same phase cut the bench times
(StepPlan.run: K3 -> K1 -> K2 -> K4 -> K5 + memo) on device-resident inputs,
with the reference CPU path timed on a strided sample of the SAME candidates
(16 processes and 1 process) and the K1 roofline figures.

    python tools/bench_extras.py [--only NAME ...] [--cpu-seconds S]

Workloads:
  c5_reuse0   the 1,000,080-candidate C5 step with K1 reuse off (every row
              of every candidate computed: no sibling shortcut)
  c5_stress   1,000,000 independent random complete chain100 schedules
              (SURVEY §8(d) stress variant), generated on the device by
              gs_random_schedules = the reference `_random_schedule` per
              candidate seed
  c2_unsharp  64K-candidate unsharp beam step (parents x step-root tilings)
  c2_harris   64K-candidate Harris beam step
  c4_resnet   262,144 random ResNet-50 bottleneck-block schedules (device
              generated), depth-3 buckets
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def _pipeline(name):
    from paper_2012_07145_b200.pipeline import chain_source, parse_pipeline
    if name == "chain100":
        return parse_pipeline(chain_source(100, 1024), "chain100")
    with open(os.path.join(ROOT, "paper_2012_07145_b200", "pipelines", f"{name}.txt")) as fh:
        return parse_pipeline(fh.read(), name)


def _time_step(sc, dec, pass_index, reuse, steps=2, warmup=1):
    import torch
    from paper_2012_07145_b200 import shard
    from paper_2012_07145_b200.engine import TIE_BAND
    n = dec.shape[0]
    plan = shard.StepPlan(sc, n, 1, 0, pass_index, pass_index * 101 + 57, bench.BEAM, 2.0, bench.NUM_PASSES,
                          TIE_BAND, reuse=reuse)
    for _ in range(warmup):
        plan.run(dec)
    sc.check()
    sc.stats()
    times = {}
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(steps):
        plan.run(dec, times=times)
    b.record()
    torch.cuda.synchronize()
    st = sc.stats()
    ms = a.elapsed_time(b) / steps
    return ms, {k: round(v / steps, 3) for k, v in times.items()}, st


def run(name, graph, recs_dev, pass_index, reuse, args, note, host_recs=None):
    import torch
    sc = recs_dev[0]
    dec = recs_dev[1]
    n = int(dec.shape[0])
    ms, br, st = _time_step(sc, dec, pass_index, reuse)
    rows_per = st["rows_computed"] / max(1, st["candidates"])
    geo_per = st["geometries"] / max(1, st["candidates"])
    k1 = br.get("featurize")
    R = sc.R
    peak, peak_kind = bench._peaks()
    bytes_k1 = n * (R * (16 + 448 + 4) + 5)
    line = {"workload": name, "note": note, "candidates": n, "stage_rows_per_candidate": R,
            "device_ms_per_step": ms, "candidates_per_s": n / (ms / 1e3),
            "step_breakdown_ms": br, "k1_reuse_mode": reuse,
            "k1_rows_computed_per_candidate": rows_per, "k1_geometries_per_candidate": geo_per,
            "k1_rows_computed_per_s": rows_per * n / (k1 / 1e3) if k1 else None,
            "roofline": {"bound": "hbm", "achieved": bytes_k1 / (k1 / 1e3) / 1e9 if k1 else None, "peak": peak,
                         "unit": "GB/s", "frac": bytes_k1 / (k1 / 1e3) / 1e9 / peak if k1 else None,
                         "peak_source": peak_kind, "algorithmic_bytes_per_launch": bytes_k1,
                         "k1_ms_per_launch": k1}}
    if name in args.cpu_skip:
        line["cpu_baseline"] = {"value": None, "why": args.cpu_skip[name]}
    elif not args.no_cpu:
        from paper_2012_07145_b200.descriptor import DECISION_DTYPE
        recs = host_recs if host_recs is not None else dec.cpu().numpy().view(DECISION_DTYPE).reshape(n, -1)
        per_sec = args.cpu_rate.get(name, 9.0)
        v16, c16, kind, desc = bench.cpu_reference(graph, recs, seconds=args.cpu_seconds, per_sec=per_sec)
        v1, c1, _, desc1 = bench.cpu_reference(graph, recs, seconds=args.cpu_seconds, cores=1, per_sec=per_sec)
        line["cpu_baseline"] = {"value": v16, "unit": "candidates/s", "cores": c16, "kind": kind, "sample": desc,
                                "one_core": {"value": v1, "cores": c1, "sample": desc1}, "cpu_model": _cpu_model()}
        line["gpu_over_cpu"] = line["candidates_per_s"] / v16
    print(json.dumps(line), flush=True)
    del sc
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--stress-n", type=int, default=1_000_000)
    run_all(ap.parse_args())


def run_all(args):
    args.cpu_rate = {"c2_unsharp": 300.0, "c2_harris": 150.0}
    args.cpu_skip = {"c4_resnet": "the reference featurizer materialises per-lane address tensors for the "
                                  "256-channel stride-0 windows (featurize.py:508-571) and exhausts host memory "
                                  "on the full-size block; tests check it via resnet_small"}
    import torch
    from paper_2012_07145_b200 import gen
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights
    want = set(args.only or ["c5_reuse0", "c5_stress", "c2_unsharp", "c2_harris", "c4_resnet"])
    w = init_weights(0)
    if "c5_reuse0" in want:
        graph, recs, _ = bench._workload(bench.PARENTS)
        sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, w)
        run("c5_reuse0", graph, (sc, sc.to_device(recs)), bench.PASS_INDEX, 0, args,
            "C5 bench step, K1 sibling reuse off: all 100 rows of every candidate computed", host_recs=recs)
    if "c5_stress" in want:
        graph = _pipeline("chain100")
        sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, w)
        dec = sc.random_schedules(args.stress_n, 0)
        run("c5_stress", graph, (sc, dec), bench.PASS_INDEX, 2, args,
            "independent random complete chain100 schedules (reference _random_schedule per seed (0, i)), "
            "device-generated")
    for name, pipe in (("c2_unsharp", "unsharp"), ("c2_harris", "harris")):
        if name not in want:
            continue
        graph = _pipeline(pipe)
        recs, _, _ = gen.beam_step(graph, 64, seed=3)
        per = len(recs) / 64
        recs, _, _ = gen.beam_step(graph, int(np.ceil(65536 / per)), seed=3)
        recs = recs[:65536]
        sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, w)
        run(name, graph, (sc, sc.to_device(recs)), 3, 2, args,
            f"{pipe} beam step: parents x all step-root tilings, 65,536 candidates", host_recs=recs)
    if "c4_resnet" in want:
        graph = _pipeline("resnet_block")
        sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, w)
        dec = sc.random_schedules(262144, 0)
        run("c4_resnet", graph, (sc, dec), 3, 2, args,
            "ResNet-50 bottleneck block 56x56x256, 262,144 random complete schedules (device-generated), "
            "depth-3 buckets")


if __name__ == "__main__":
    main()
