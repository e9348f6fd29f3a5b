"""One line per captured launch of an ncu report: time, DRAM bytes, occupancy, issue, instructions
(run here, no GPU).   python tools/ncu_kernels.py rep.ncu-rep [--json out.json --workload W]"""
import argparse
import csv
import io
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
SCALE = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "Gbyte": 1e9, "Mbyte": 1e6,
         "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}

ap = argparse.ArgumentParser()
ap.add_argument("rep")
args = ap.parse_args()
out = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
res = []
for r in rows[2:]:
    d = {"kernel": r[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            v = float(r[h.index(k)].replace(",", "") or 0)
            u = units[h.index(k)]
            d[k] = v * SCALE.get(u, 1.0) if u in SCALE else v
    res.append(d)
for d in res:
    t = d["gpu__time_duration.sum"]
    rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
    print(f"{d['kernel'][:48]:48s} {t * 1e3:9.3f} ms  read {rd / 1e9:7.3f} GB  write {wr / 1e9:7.3f} GB"
          f"  -> {(rd + wr) / t / 1e9:7.1f} GB/s  warps {d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):5.1f}%"
          f"  issue {d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):5.1f}%"
          f"  inst {d.get('smsp__inst_executed.sum', 0) / 1e9:6.2f} G")
print(json.dumps(res))
