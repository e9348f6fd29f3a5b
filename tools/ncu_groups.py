"""Group a kernel's SASS instructions into runs with equal execution counts (run here, no GPU):
the biggest (count x length) runs are the loops and paths that dominate the instruction budget.

    python tools/ncu_groups.py rep.ncu-rep kernel_filter [--top 25]
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("k")
ap.add_argument("--top", type=int, default=25)
args = ap.parse_args()
out = subprocess.run(["ncu", "-i", args.rep, "-k", "regex:" + args.k, "--page", "source", "--csv",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
prof = []
for r in rows[2:]:
    if r and r[0] in ("Kernel Name", "Address"):
        break
    if len(r) < len(hdr):
        continue
    prof.append((int(r[ix["Address"]], 16), int(r[ix["Instructions Executed"]] or 0),
                 int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r[ix["Source"]][:60]))
base = prof[0][0]
groups = []
for a, e, st, src in prof:
    if groups and groups[-1][1] == e:
        groups[-1][2] += 1
        groups[-1][3] += st
    else:
        groups.append([a - base, e, 1, st, src])
tot = sum(p[1] for p in prof)
tst = sum(p[2] for p in prof) or 1
print(f"total {tot}")
for off, e, n, st, src in sorted(groups, key=lambda g: -g[1] * g[2])[:args.top]:
    print(f"{off:6x} count {e:10d} x{n:3d} = {e * n / 1e6:8.1f}M ({100 * e * n / tot:4.1f}%) "
          f"stalls {100 * st / tst:4.1f}%  {src}")
