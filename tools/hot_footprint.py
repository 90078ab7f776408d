"""Hot instruction footprint of a kernel from an ncu report: how many static
SASS instructions carry 50/90/99% of the executed ones, the no-instruction
(I-cache) stall share, and the hot static instructions per source function
with the number of disjoint address ranges they occupy (inlined copies).

usage: python tools/hot_footprint.py REPORT.ncu-rep SOURCE.cu"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, src_path = sys.argv[1], sys.argv[2]


def page(kind):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", kind],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
stall = {h: v for h, v in zip(r[0], r[2]) if "average_warps_issue_stalled" in h and h.endswith("issue_active.ratio")}
tot_stall = sum(float(v) for v in stall.values())
for h, v in sorted(stall.items(), key=lambda x: -float(x[1]))[:5]:
    print("%-40s %.2f (%.0f%%)" % (h.split("stalled_")[1].split("_per")[0], float(v), 100 * float(v) / tot_stall))

src = open(src_path).read().split("\n")
starts = []
for i, l in enumerate(src):
    m = re.match(r"(?:template <[^>]*>\s*)?(?:__device__|__global__|static|inline|__noinline__|__forceinline__)"
                 r"[^;{]*?\b(\w+)\s*\(", l)
    if m:
        starts.append((i + 1, m.group(1)))


def fn_of(line):
    name = "?"
    for s, n in starts:
        if s > line:
            break
        name = n
    return name


rows = page("cuda,sass")
ex = []
cur_file, cur_line = None, None
for row in rows:
    if row and row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if len(row) < 8:
        continue
    if row[0].isdigit():
        cur_line = int(row[0])
        continue
    if row[0] == "" and row[2].startswith("0x"):
        e = int(row[7]) if row[7].isdigit() else 0
        key = fn_of(cur_line) if cur_file == src_path.split("/")[-1] else cur_file
        ex.append((int(row[2], 16), e, key))
tot = sum(e for _, e, _ in ex)
s = sorted(ex, key=lambda x: -x[1])
for q in (0.5, 0.9, 0.99):
    acc = 0
    for n, x in enumerate(s):
        acc += x[1]
        if acc >= q * tot:
            print("%d%% of executed instructions in %d static (%d KB)" % (q * 100, n + 1, (n + 1) * 16 // 1024))
            break
hot, rng, share = collections.Counter(), collections.defaultdict(list), collections.Counter()
for a, e, k in ex:
    share[k] += e
    if e > tot * 1e-6:
        hot[k] += 1
        rng[k].append(a)
print("%-28s %6s %7s %s" % ("function", "hot", "exec%", "ranges"))
for k, v in hot.most_common(25):
    a = sorted(rng[k])
    print("%-28s %6d %6.1f%% %d" % (k, v, 100 * share[k] / tot, 1 + sum(1 for x, y in zip(a, a[1:]) if y - x > 256)))
print("hot static total", sum(hot.values()), "=", sum(hot.values()) * 16 // 1024, "KB")

# stall samples by function (all reasons / no-instruction / long scoreboard)
hdr, cf, cl = None, None, None
al, ni, lsb = collections.Counter(), collections.Counter(), collections.Counter()
for row in rows:
    if row and row[0] == "File Path":
        cf = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        hdr = row
        continue
    if len(row) < 8 or hdr is None:
        continue
    if row[0].isdigit():
        cl = int(row[0])
        continue
    if row[0] == "" and row[2].startswith("0x"):
        k = fn_of(cl) if cf == src_path.split("/")[-1] else cf
        al[k] += int(row[4])
        ni[k] += int(row[hdr.index("stall_no_inst")])
        lsb[k] += int(row[hdr.index("stall_long_sb")])
T, N, L = sum(al.values()) or 1, sum(ni.values()) or 1, sum(lsb.values()) or 1
print("%-28s %7s %7s %7s" % ("function", "samples", "no_inst", "long_sb"))
for k, v in al.most_common(20):
    print("%-28s %6.1f%% %6.1f%% %6.1f%%" % (k, 100 * v / T, 100 * ni[k] / N, 100 * lsb[k] / L))
