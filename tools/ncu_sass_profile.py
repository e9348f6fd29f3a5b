"""Per-instruction execution counts and stall samples of one kernel in an ncu report, grouped
into contiguous SASS ranges (run here, no GPU): shows where the instructions go.

    python tools/ncu_sass_profile.py rep.ncu-rep [--min 1e6]
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--min", type=float, default=1e6, help="print instructions executed >= this")
args = ap.parse_args()
out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
tot = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    e = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += e
    if e >= args.min:
        print(f"{r[ix['Address']][-5:]} {e:12d} {s:7d}  {r[ix['Source']].strip()[:90]}")
print("total", tot)
