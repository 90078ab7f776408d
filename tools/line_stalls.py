"""Stall samples / no-instruction stalls / executed instructions per source
line of one file, from an ncu report's interleaved cuda,sass source page.
usage: python tools/line_stalls.py REPORT.ncu-rep SOURCE.cu [N] [LO HI]"""
import collections
import csv
import io
import subprocess
import sys

rep, src_path = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
lo, hi = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (0, 1 << 30)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
base = src_path.split("/")[-1]
src = open(src_path).read().split("\n")
al, ni, ex, st = collections.Counter(), collections.Counter(), collections.Counter(), collections.Counter()
hdr = cf = cl = None
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
    if row[0] == "" and row[2].startswith("0x") and cf == base and lo <= cl <= hi:
        al[cl] += int(row[4])
        ni[cl] += int(row[hdr.index("stall_no_inst")])
        e = int(row[7]) if row[7].isdigit() else 0
        ex[cl] += e
        st[cl] += 1
T = sum(al.values()) or 1
print("line  samples  no_inst   executed static  source")
for l, v in al.most_common(n):
    print("%5d %6.2f%% %8d %10d %5d  %s" % (l, 100 * v / T, ni[l], ex[l], st[l], src[l - 1].strip()[:70]))
