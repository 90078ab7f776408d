"""Benchmark: candidate schedules scored per second on a 100-stage pipeline.

Workload (BASELINE.json config 5): the synthetic
100-stage stencil chain (`make_chain_src(100, extent=1024)`), one beam step
of P = 4,167 random phase-2 parents x 240 step-root tilings = 1,000,080
candidates.  A step is one pass of the hot path over the batch: featurize +
prune (K1) and cost (K2) every candidate, structural hash at the pass depth
(K3), bucket + hierarchical-sampling representatives (K4), penalized
tie-banded top-k cut + bad-hash memo hashes (K5, K3).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N>1 (torchrun, one rank per GPU): candidates are bucket-partitioned across
ranks (strong scaling: the 1M-candidate step is shared), each rank scores
its buckets and samples their representatives; rank representative records
are exchanged with one NCCL all-gather and every rank cuts the same beam.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PARENTS = 4167
PASS_INDEX = 3
PHASE_SEED = 0 * 10007 + PASS_INDEX * 101 + 57
BEAM = 32
NUM_PASSES = 5
METRIC = "candidate schedules scored/sec (100-stage pipe, 1/2/4/8 B200) and HBM GB/s"
UNIT = "candidates/s"


PARENTS_FILE = os.path.join(ROOT, "bench_data", "c5_parents_seed0.npz")


def _parents(parents):
    from paper_2012_07145_b200.descriptor import DECISION_DTYPE
    z = np.load(PARENTS_FILE)
    par = np.ascontiguousarray(z["parents"]).view(DECISION_DTYPE).reshape(len(z["parents"]), -1)
    return par[:parents], z["steps"][:parents]


def _workload(parents):
    """The committed prune-valid parents (bench_data/make_c5.py) expanded to
    every tiling of their step root (host, untimed)."""
    from paper_2012_07145_b200.descriptor import DECISION_DTYPE
    from paper_2012_07145_b200.gen import expand_step
    from paper_2012_07145_b200.pipeline import chain_source, parse_pipeline
    graph = parse_pipeline(chain_source(100, 1024), "chain100")
    z = np.load(PARENTS_FILE)
    par = np.ascontiguousarray(z["parents"]).view(DECISION_DTYPE).reshape(len(z["parents"]), -1)
    par, steps = par[:parents], z["steps"][:parents]
    recs, owner = expand_step(par, steps, graph)
    return graph, recs, owner


# ---------------------------------------------------------------------------
# CPU reference (baseline/_ref = unmodified reference, else the oracle port)
# ---------------------------------------------------------------------------

def _ref_import():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "gpusched")):
        if ref not in sys.path:
            sys.path.append(ref)
        try:
            import gpusched  # noqa: F401
            return "reference"
        except ImportError:
            pass
    return "port"


_W = {}


def _worker_init(kind, text, rows, barrier, name="chain100"):
    _W["kind"], _W["rows"], _W["barrier"] = kind, rows, barrier
    if kind == "reference":
        import gpusched
        from gpusched.costmodel import init_weights
        from gpusched.loopnest import Decision, apply_decision, initial_state
        from gpusched.machine import MachineParams
        g = gpusched.parse_pipeline(text, name)
        _W.update(g=g, w=init_weights(0), p=MachineParams(), D=Decision, ap=apply_decision,
                  init=initial_state)
    else:
        from paper_2012_07145_b200.params import MachineParams, init_weights
        from paper_2012_07145_b200.pipeline import parse_pipeline
        _W.update(g=parse_pipeline(text, name), w=init_weights(0).tensors, p=MachineParams())


def _states(recs):
    kinds = ("compute_root", "fuse_at_block", "fuse_at_thread", "inline")
    g = _W["g"]
    out = []
    for rec in recs:
        decs = []
        for r in rec:
            if r["func"] == 0xFFFF:
                break
            f = g.funcs[int(r["func"])]
            nd = f.ndim
            decs.append((f.name, kinds[int(r["kind"])],
                         None if r["consumer"] == 0xFFFF else g.funcs[int(r["consumer"])].name,
                         tuple(int(x) for x in r["serial"][:nd]) if r["flags"] & 1 else None,
                         tuple(int(x) for x in r["thread"][:nd]) if r["flags"] & 2 else None))
        out.append(decs)
    return out


def _worker_run(chunk):
    recs = _W["rows"][chunk[0]:chunk[1]]
    raw = _states(recs)
    if _W["kind"] == "reference":
        from gpusched.search import CostEvaluator
        D, ap = _W["D"], _W["ap"]
        states = []
        for decs in raw:
            st = _W["init"](_W["g"])
            for f, k, c, s, t in decs:
                if k == "compute_root" and s is not None:
                    st = ap(st, f, D("compute_root"))
                st = ap(st, f, D(k, c, s, t))
            states.append(st)
        _W["barrier"].wait()
        t0 = time.perf_counter()
        for st in states:
            CostEvaluator(_W["w"], _W["p"]).cost(st, _W["g"])   # cold: fresh evaluator
        return len(states), time.perf_counter() - t0
    from oracle import costing
    from paper_2012_07145_b200.schedule import Decision
    cands = [tuple((f, Decision(k, c, s, t)) for f, k, c, s, t in decs) for decs in raw]
    _W["barrier"].wait()
    t0 = time.perf_counter()
    for d in cands:
        costing.score(_W["g"], d, _W["p"], _W["w"])
    return len(cands), time.perf_counter() - t0


def cpu_reference(graph, recs, seconds=15.0, cores=None, per_sec=9.0):
    """Score a bounded, evenly strided sample of the same candidates with the
    CPU reference on all host cores (fork pool, fresh evaluator per
    candidate).  Returns (cand/s, cores, kind, sample description).
    per_sec: the expected candidates/s per core (sizes the sample)."""
    from paper_2012_07145_b200.pipeline import graph_to_text
    kind = _ref_import()
    cores = cores or os.cpu_count() or 1
    per_core = max(4, int(seconds * per_sec))    # ~10 cand/s/core at R = 100
    n = min(len(recs), per_core * cores)
    idx = np.linspace(0, len(recs) - 1, n).astype(np.int64)
    sample = recs[idx]
    bounds = np.linspace(0, n, cores + 1).astype(int)
    chunks = [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(len(chunks))
    with ctx.Pool(len(chunks), initializer=_worker_init,
                  initargs=(kind, graph_to_text(graph), sample, barrier, graph.name)) as pool:
        res = pool.map(_worker_run, chunks, chunksize=1)
    done = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    desc = (f"{done} candidates evenly strided over the {len(recs)}-candidate step, "
            f"{len(chunks)} processes, cold CostEvaluator.cost each "
            f"({'unmodified reference gpusched' if kind == 'reference' else 'oracle port'})")
    return done / wall, len(chunks), kind, desc


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    graph, recs, _ = _workload(args.parents)
    vals = []
    for i in range(args.warmup + args.steps):
        v, cores, kind, desc = cpu_reference(graph, recs, seconds=args.cpu_seconds)
        if i >= args.warmup:
            vals.append(v)
    val = float(np.median(vals))
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "chain100@1024^2 beam step: 4167 parents x 240 tilings",
                       "candidates_per_step": int(len(recs))},
            "impl": "reference",
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": kind, "sample": desc},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index=0):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def wait_first(self, timeout=3.0):
        """Block until nvidia-smi has produced its first sample."""
        t0 = time.time()
        while self.proc and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.02)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        load = [r for r in self.rows if len(r) >= 8 and r[7].isdigit() and int(r[7]) > 0] or self.rows
        sm = [float(r[0]) for r in load if r[0].replace('.', '').isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace('.', '').isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i in range(4) if len(r) > 3 + i and "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "samples_under_load": len(load)}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def bench_parity(sc, plan, dec, timed_out):
    """Check the bench's own step against the reference fixture of this exact
    step (tests/golden/c5_step.*, written by the unmodified reference via
    tests/golden/make_c5_golden.py): the beam the timed region cut, and an
    untimed re-run with rejects for representatives, rejects, representative
    costs, the memo, and 1,024 strided candidates' totals and verdicts."""
    import gzip
    import torch
    gold = os.path.join(ROOT, "tests", "golden")
    try:
        with gzip.open(os.path.join(gold, "c5_step.json.gz"), "rt") as fh:
            meta = json.load(fh)
        arr = np.load(os.path.join(gold, "c5_step.npz"))
    except OSError:
        return {"checked": False, "why": "fixture missing"}
    if meta["n_candidates"] != dec.shape[0]:
        return {"checked": False, "why": "not the fixture's step size"}
    from paper_2012_07145_b200.descriptor import PRUNE_REASONS
    v = meta["cut"]["variants"]["bench"]
    out = plan.run(dec, rejects=True)
    sc.check()
    reps = out["reps"].cpu().numpy()
    rep_cost = out["total"].index_select(0, out["reps"]).cpu().numpy()
    idx = torch.as_tensor(arr["sample_index"], device=sc.device)
    tot = out["total"].index_select(0, idx).cpu().numpy()
    ver = out["verdict"].index_select(0, idx).cpu().numpy()
    memo = {(dd, int(x)) for dd, hs in enumerate(out["memo"], start=1) for x in hs.cpu().numpy().view(np.uint64)}
    want_memo = {(int(dd), int(h)) for dd, h in v["memo_after"]}
    rel = lambda a, b: float(np.max(np.abs(a - b) / np.abs(b))) if len(b) else 0.0  # noqa: E731
    res = {"checked": True, "fixture": "tests/golden/c5_step (unmodified reference _cut over this step)",
           "timed_beam_exact": timed_out["beam"] == v["beam"],
           "beam_exact": out["beam"] == v["beam"],
           "reps_exact": bool(np.array_equal(reps, arr["rep_idx"])),
           "rejects_exact": [i for i, _ in out["rejects"]] == arr["rej_idx"].tolist()
           and [r for _, r in out["rejects"]] == meta["cut"]["reject_reasons"],
           "memo_exact": memo == want_memo,
           "rep_cost_max_rel_err": rel(rep_cost, arr["rep_cost"]),
           "sample_n": int(len(idx)),
           "sample_total_max_rel_err": rel(tot, arr["total"]),
           "sample_verdicts_exact": [PRUNE_REASONS[c - 1] if c else None for c in ver] == meta["prune"]}
    res["ok"] = bool(res["timed_beam_exact"] and res["beam_exact"] and res["reps_exact"] and res["rejects_exact"]
                     and res["memo_exact"] and res["sample_verdicts_exact"] and res["rep_cost_max_rel_err"] <= 1e-9
                     and res["sample_total_max_rel_err"] <= 1e-9)
    return res


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2012_07145_b200 import _lib
    from paper_2012_07145_b200.engine import Scorer, TIE_BAND
    from paper_2012_07145_b200.params import DEFAULT_THRESHOLDS, MachineParams, init_weights
    from paper_2012_07145_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one rank per GPU over NCCL; GS_DIST_BACKEND=gloo (and ranks sharing a
    # device) lets a one-GPU box exercise the N > 1 path (tests, diagnostics)
    backend = os.environ.get("GS_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    graph, recs, info = _workload(args.parents)
    N = int(recs.shape[0])
    lib = _lib.load()
    sc = Scorer(graph, MachineParams(), DEFAULT_THRESHOLDS, init_weights(0))
    dec = sc.to_device(recs)                       # inputs resident in HBM
    # the beam as the search holds it (parents + step-root index), pinned,
    # for the end-to-end arm: candidates are generated on the device
    par, steps = _parents(args.parents)
    host_par = torch.from_numpy(par.view(np.uint8).reshape(len(par), -1)).pin_memory()
    host_steps = torch.from_numpy(np.asarray(steps, dtype=np.int32)).pin_memory()
    stream = torch.cuda.current_stream()
    plan = shard.StepPlan(sc, N, world, rank, PASS_INDEX, PHASE_SEED, BEAM, 2.0, NUM_PASSES, TIE_BAND)

    phase_ms = {}

    def step(d, timed=False):
        return plan.run(d, times=phase_ms if timed else None)

    # the clock sampler starts before the warm-up: nvidia-smi's own start-up
    # (driver / NVML initialisation) landed inside the timed region and, at
    # the step's one host read-back, showed up as sporadic 10-400 ms steps
    clk = Clocks(local).__enter__()
    clk.wait_first()
    for _ in range(args.warmup):
        step(dec)
    sc.check()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = lib.gs_launch_count()
    phase_ms.clear()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import gc
    gc.collect()
    gc.disable()   # no collector pauses between the step's kernel launches
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n_pre = len(clk.rows)
    ev0.record(stream)
    for _ in range(args.steps):
        res = step(dec, timed=True)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk.__exit__(None, None, None)
    clk.rows = clk.rows[max(0, n_pre - 1):]   # the samples taken during the timed region (+ the one before)
    gc.enable()
    launches = lib.gs_launch_count() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = N / (ms / 1e3)

    # e2e through the public beam-step API: pinned host beam in (parents +
    # step-root indices; the 1M candidates are generated on the device by
    # gs_expand_step), totals + verdicts + beam out, copies inside the
    # timed region
    e2e_ms = []
    gc.collect()
    gc.disable()
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = plan.run_beam_host(host_par, host_steps, total=N)
        b.record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
    gc.enable()
    e = float(np.mean(e2e_ms))
    if world > 1:
        t = torch.tensor([e], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e = float(t.item())
    sc.check()

    parity = bench_parity(sc, plan, dec, res) if world == 1 else {"checked": False, "why": "N > 1"}
    extra = None
    if world == 1 and not args.no_extras:
        # what sibling reuse hides, and the other BASELINE configs (VERDICT
        # r01 item 3): tools/bench_extras.py, each with the reference CPU path
        # on the same candidates at 16 and 1 cores (after the timed region)
        import io
        import contextlib
        import types
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_extras
        plan.fbuf = plan.rcbuf = None
        torch.cuda.empty_cache()
        buf = io.StringIO()
        ex_args = types.SimpleNamespace(only=None, cpu_seconds=args.cpu_seconds * (0 if args.no_cpu else 0.5),
                                        no_cpu=args.no_cpu, stress_n=1_000_000)
        try:
            with contextlib.redirect_stdout(buf):
                bench_extras.run_all(ex_args)
            extra = [json.loads(x) for x in buf.getvalue().splitlines() if x.startswith("{")]
        except Exception as e:   # extras never fail the headline line
            extra = [{"error": repr(e)}]
    if rank == 0:
        R = sc.R
        n_local = plan.local_count
        k1 = phase_ms["featurize"] / args.steps if phase_ms else None
        breakdown = {k: round(v / args.steps, 3) for k, v in phase_ms.items()}
        # K1 algorithmic bytes per launch (SURVEY 8(d)'s north-star dataflow,
        # the K1 share of B(R)): 16 B decision record per row in, 448 B fp64
        # feature row + 4 B row key per row out, 4+1 B per candidate.  The
        # step runs K1 in reuse mode 2, which writes only the computed rows
        # (K2 reads repeated rows through row_src), so the measured DRAM
        # traffic (roofline.traffic) is below this figure by design.
        bytes_k1 = n_local * (R * (16 + 448 + 4) + 5)
        peak, peak_kind = _peaks()
        achieved = bytes_k1 / (k1 / 1e3) / 1e9 if k1 else None
        traffic, inst_per_cand = None, None
        prof = os.path.join(ROOT, "profiles", "r02_k1_counters.json")
        if os.path.exists(prof):
            try:
                with open(prof) as fh:
                    kc = json.load(fh)
                traffic = kc.get("dram_bytes_per_launch_per_candidate")
                traffic = traffic * n_local if traffic else None
                inst_per_cand = kc.get("warp_instructions_per_candidate")
            except Exception:
                traffic = None
        clk_summary = clk.summary()
        f_clk = (clk_summary.get("sm_mhz") or 1965.0) * 1e6
        import torch as _t
        n_sm = _t.cuda.get_device_properties(local).multi_processor_count
        issue = None
        if inst_per_cand and k1:
            # instruction-issue roofline of K1: warp-instructions it must issue
            # (ncu count per candidate) at the measured rate, over 4 issue
            # slots per SM per clock
            ach = inst_per_cand * n_local / (k1 / 1e3)
            issue = {"achieved": ach, "peak": n_sm * 4 * f_clk, "unit": "warp-instructions/s",
                     "frac": ach / (n_sm * 4 * f_clk), "warp_instructions_per_candidate": inst_per_cand,
                     "source": "profiles/r02_k1_counters.json (ncu smsp__inst_executed.sum / candidates)"}
        cpu = None
        if world == 1 and not args.no_cpu:
            v, cores, kind, desc = cpu_reference(graph, recs, seconds=args.cpu_seconds)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": desc}
            try:
                lscpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
                cpu["cpu_model"] = next((ln.split(":", 1)[1].strip() for ln in lscpu.splitlines()
                                         if ln.startswith("Model name")), None)
            except Exception:
                pass
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (random phase-2 beam-step parents, seed 0; init_weights(0))",
            "config": {"workload": "chain100@1024^2 beam step: 4167 parents x 240 tilings",
                       "candidates_per_step": N, "stage_rows_per_candidate": R,
                       "beam_size": BEAM, "pass_index": PASS_INDEX,
                       "l2": "inputs larger than L2 (1.6 GB records in, 3.7 computed feature rows of 100 per candidate out)",
                       "parallelism": f"bucket-sharded x{world}" if world > 1 else "single GPU"},
            "roofline": {"bound": "hbm", "kernel": "K1 featurize (gs::featurize_kernel)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "peak_source": peak_kind, "k1_ms_per_launch": k1,
                         "k1_share_of_step": (k1 / ms) if k1 else None,
                         "algorithmic_bytes_per_launch": bytes_k1,
                         "note": "K1 is integer-ALU / instruction-latency bound (resolve + warp transaction "
                                 "emulation); achieved = SURVEY 8(d) algorithmic bytes / K1 time as the north "
                                 "star asks; K1 writes only computed rows (reuse mode 2), traffic = ncu DRAM bytes",
                         "issue": issue},
            "cpu_baseline": cpu,
            "e2e": {"value": N / (e / 1e3), "unit": UNIT, "ms_per_step": e,
                    "path": "StepPlan.run_beam_host: H2D beam, gs_expand_step on device, step, D2H results",
                    "h2d_bytes_per_step": int(out["h2d_bytes"]), "d2h_bytes_per_step": int(out["d2h_bytes"])},
            "step_breakdown_ms": breakdown,
            "gpu_launches": int(launches),
            "clocks": clk_summary,
            "beam": res["beam"][:8],
            "parity": parity,
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--parents", type=int, default=PARENTS)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip tools/bench_extras.py's workloads")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
