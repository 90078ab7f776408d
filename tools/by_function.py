"""Per-function instruction / stall shares of an ncu source export (cuda,sass view)."""
import csv
import re
import sys

path, src_file = sys.argv[1], sys.argv[2]
n_units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
rows = list(csv.reader(open(path)))
cur, data = None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1]
        continue
    if not r or r[0] in ("Line No", "Function Name") or len(r) < 8 or r[2] != "-":
        continue
    try:
        data.append((cur, int(r[0]), int(r[4]), int(r[7])))
    except ValueError:
        pass
src = open(src_file).read().split("\n")
starts = [(i + 1, m.group(2)) for i, l in enumerate(src)
          for m in [re.match(r"^(__device__|__global__).*?(\w+)\s*\(", l)] if m]


def fn(f, line):
    if not f or not f.endswith(src_file.split("/")[-1]):
        return "<headers/intrinsics>"
    name = "?"
    for s, n in starts:
        if s <= line:
            name = n
    return name


agg = {}
ts = sum(d[2] for d in data) or 1
ti = sum(d[3] for d in data) or 1
for f, l, s, i in data:
    a = agg.setdefault(fn(f, l), [0, 0])
    a[0] += s
    a[1] += i
for n, (s, i) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:24s} stall {100 * s / ts:5.1f}%  inst {100 * i / ti:5.1f}%  {i / n_units:9.0f}/unit")
