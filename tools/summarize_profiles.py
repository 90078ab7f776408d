"""Summarise the ncu artefacts a gpurun call brought back (gpurun_out/) into
tracked files under profiles/ for one round tag:

  profiles/<tag>_launches.csv   per-kernel totals of the launch list
                                (gpu__time_duration.sum, --clock-control none)
  profiles/<tag>_<k>_raw.txt    key raw metrics of each `ncu --set full` capture
  profiles/<tag>_<k>_lines.txt  top source lines by warp-stall samples

usage: python tools/summarize_profiles.py r01 [k1 k2 ...]
"""

import collections
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
       "launch__registers_per_thread", "launch__occupancy_limit_registers",
       "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
       "smsp__thread_inst_executed_per_inst_executed.ratio"] + [
       f"smsp__average_warps_issue_stalled_{r}_per_issue_active.ratio"
       for r in ("no_instruction", "long_scoreboard", "wait", "short_scoreboard", "barrier", "branch_resolving")]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, cwd=ROOT).stdout


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        a = agg.setdefault(d["Kernel Name"].split("(")[0], [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as fh:
        fh.write("kernel,launches,total_ns,share\n")
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"\"{k}\",{n},{t:.0f},{t / tot:.4f}\n")


def raw(tag, k):
    rep = os.path.join(OUT, f"prof_{k}.ncu-rep")
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    h, u = rows[0], rows[1]
    with open(os.path.join(PROF, f"{tag}_{k}_raw.txt"), "w") as fh:
        for v in rows[2:]:
            fh.write(f"kernel: {v[h.index('Kernel Name')]}\n")
            for i, n in enumerate(h):
                if n in RAW:
                    fh.write(f"  {n} = {v[i]} {u[i]}\n")


def lines(tag, k, top=40):
    rep = os.path.join(OUT, f"prof_{k}.ncu-rep")
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv",
                                           "--print-source=cuda,sass"))))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    data = []
    for r in rows[hi + 1:]:
        if len(r) < 8 or r[2] != "-":
            continue
        try:
            data.append((int(r[0]), r[1].strip()[:100], int(r[4]), int(r[7])))
        except ValueError:
            pass
    ts = sum(d[2] for d in data) or 1
    ti = sum(d[3] for d in data) or 1
    with open(os.path.join(PROF, f"{tag}_{k}_lines.txt"), "w") as fh:
        fh.write("line  stall%  inst%  source\n")
        for d in sorted(data, key=lambda x: -x[2])[:top]:
            fh.write(f"{d[0]:5d} {100 * d[2] / ts:6.1f} {100 * d[3] / ti:6.1f}  {d[1]}\n")


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    if os.path.exists(os.path.join(OUT, "launches.csv")):
        launches(tag)
    for k in sys.argv[2:]:
        raw(tag, k)
        lines(tag, k)
