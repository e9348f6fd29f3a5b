"""Join ncu per-instruction execution counts with nvdisasm line info (run here, no GPU).

    python tools/sass_lines.py rep.ncu-rep cubin kernel_mangled_name [--top 40]

Prints instructions executed and stall samples summed per CUDA source line (file:line)."""
import argparse
import collections
import csv
import io
import re
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("cubin")
ap.add_argument("kernel")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("-k", default=None, help="kernel name filter when the report holds several")
args = ap.parse_args()
cmd = ["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "sass"]
if args.k:
    cmd[3:3] = ["-k", args.k]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
prof = []
for r in rows[2:]:
    if r and r[0] in ("Kernel Name", "Address"):
        break  # a second launch of the kernel: keep the first
    if len(r) < len(hdr):
        continue
    prof.append((int(r[ix["Address"]], 16), int(r[ix["Instructions Executed"]] or 0),
                 int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
base = min(a for a, _, _ in prof)
dis = subprocess.run(["nvdisasm", "-g", "-c", args.cubin], capture_output=True, text=True).stdout
sec = dis[dis.index(".text." + args.kernel + ":"):]
nxt = sec.find("//---------------------", 10)
sec = sec[:nxt] if nxt > 0 else sec
line_of = {}
cur = "?"
for ln in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0, 0])
for a, e, s in prof:
    k = line_of.get(a - base, "?")
    agg[k][0] += e
    agg[k][1] += s
tot_e = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total instructions {tot_e}, stall samples {tot_s}")
for k, (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:args.top]:
    print(f"{k:28s} {e:12d} {100 * e / tot_e:5.1f}%  stalls {100 * s / tot_s:5.1f}%")
