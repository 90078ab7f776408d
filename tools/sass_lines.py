"""Static SASS instruction count per source line of one kernel (and its
non-inlined callees) in a cubin disassembled with nvdisasm --print-line-info."""
import collections
import re
import sys

sass, src_path, key = sys.argv[1], sys.argv[2], sys.argv[3]
lines = open(sass).read().split("\n")
secs = [i for i, l in enumerate(lines) if l.startswith("//---")]
cnt, cur = collections.Counter(), None
for i in secs:
    if key not in lines[i]:
        continue
    j = next((x for x in secs if x > i), len(lines))
    for l in lines[i:j]:
        m = re.search(r'//## File "(.*?)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        if re.search(r"/\*[0-9a-f]{4,}\*/\s+\S", l):
            cnt[cur] += 1
src = open(src_path).read().split("\n")
base = src_path.split("/")[-1]
print("total", sum(cnt.values()))
for k, c in cnt.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 30):
    s = src[k[1] - 1].strip()[:80] if k and k[0] == base else ""
    print(c, k, s)
