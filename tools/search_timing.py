"""C3 wall time: the unmodified reference search (`schedule_with_freezing`,
search.py:347-356) on an authored ~100-func pipeline, run (a) on the CPU
reference and (b) through the drop-in seam (GpuCostEvaluator + gpu_cut
installed into gpusched.search), with the same config; prints one JSON line
with both wall times, the candidate count and whether the final beams are
identical.

    python tools/search_timing.py [--pipeline local_laplacian] [--beam 8] [--passes 2] [--no-cpu]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "gpusched")) and p not in sys.path:
        sys.path.append(p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pipeline", default="local_laplacian")
    ap.add_argument("--beam", type=int, default=8)
    ap.add_argument("--passes", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-gpu", action="store_true")
    args = ap.parse_args()
    import gpusched.search as gs
    from gpusched.costmodel import init_weights
    from gpusched.loopnest import schedule_dump
    from gpusched.machine import MachineParams
    from gpusched.pipeline import parse_pipeline
    with open(os.path.join(ROOT, "paper_2012_07145_b200", "pipelines", f"{args.pipeline}.txt")) as fh:
        graph = parse_pipeline(fh.read(), args.pipeline)
    cfg = gs.SearchConfig(beam_size=args.beam, num_passes=args.passes, seed=0, freeze_enabled=True)
    params = MachineParams()
    w = init_weights(0)
    count = {"candidates": 0, "cuts": 0}
    orig_cut = gs._cut

    def counting(cut):
        def f(candidates, *a, **k):
            count["candidates"] += len(candidates)
            count["cuts"] += 1
            return cut(candidates, *a, **k)
        return f

    out = {"pipeline": args.pipeline, "funcs": len(graph.funcs), "beam_size": args.beam, "num_passes": args.passes,
           "freeze": True}
    finals = {}
    if not args.no_gpu:
        import torch
        from paper_2012_07145_b200 import evaluator as ev_mod
        ev = ev_mod.GpuCostEvaluator(w, params, cfg.thresholds)
        prev = ev_mod.install(gs, expand=True)
        gs._cut = counting(ev_mod.gpu_cut)
        try:
            gs.schedule_with_freezing(graph, params, cfg, ev)   # warm-up: CUDA context, pipeline upload
            count.update(candidates=0, cuts=0)
            torch.cuda.synchronize()
            t = time.perf_counter()
            final = gs.schedule_with_freezing(graph, params, cfg, ev)
            torch.cuda.synchronize()
            out["gpu_seam_s"] = time.perf_counter() - t
        finally:
            gs._cut, gs._phase1_candidates, gs._phase2_candidates = prev
        out["cut_calls"] = count["cuts"]
        finals["gpu"] = [(schedule_dump(s), s.cost) for s in final]
    if not args.no_cpu:
        count.update(candidates=0, cuts=0)
        gs._cut = counting(orig_cut)
        try:
            t = time.perf_counter()
            final = gs.schedule_with_freezing(graph, params, cfg, gs.CostEvaluator(w, params))
            out["cpu_reference_s"] = time.perf_counter() - t
        finally:
            gs._cut = orig_cut
        out["candidates"] = count["candidates"]
        finals["cpu"] = [(schedule_dump(s), s.cost) for s in final]
        out["cpu_cores"] = 1
    if len(finals) == 2:
        a, b = finals["gpu"], finals["cpu"]
        out["final_beams_identical"] = [x for x, _ in a] == [x for x, _ in b]
        out["final_cost_max_rel_err"] = max(abs(x - y) / abs(y) for (_, x), (_, y) in zip(a, b)) if a else 0.0
        out["speedup"] = out["cpu_reference_s"] / out["gpu_seam_s"]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
