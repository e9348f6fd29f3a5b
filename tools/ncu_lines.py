"""Instructions executed per source line of one kernel: ncu's SASS page (execution counts) joined
with nvdisasm's line table of the same cubin (run here, no GPU).
    python tools/ncu_lines.py sass.csv disasm.txt kernel_mangled_name [--top 30]"""
import collections
import csv
import re
import sys

sass_csv, dis, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [(int(r[ix["Address"]], 16), int(r[ix["Instructions Executed"]] or 0))
        for r in rows[2:] if len(r) >= len(hdr)]
base = data[0][0]
lines = open(dis).read().split("\n")
start = [i for i, l in enumerate(lines) if re.match(r"\s*\.text\." + re.escape(fn) + ":", l)][0]
cur, off2line = None, {}
for l in lines[start + 1:]:
    if re.match(r"\s*\.text\.", l) or re.match(r"\s*\.section", l):
        break
    m = re.search(r'//## File "(.*?)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
    m2 = re.search(r"/\*([0-9a-f]{4,6})\*/\s+\S", l)
    if m2:
        off2line[int(m2.group(1), 16)] = cur
by, tot = collections.Counter(), 0
for a, e in data:
    ln = off2line.get(a - base)
    if ln:
        by[ln] += e
        tot += e
for (f, n), c in by.most_common(top):
    print(f"{100 * c / tot:5.1f}% {f}:{n}")
print("total", tot)
