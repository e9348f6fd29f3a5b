"""Per-kernel mean time and DRAM bytes from an ncu --csv launch list (run here, no GPU):
    python tools/launch_table.py launches.csv [filter]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
ix = {h: i for i, h in enumerate(rows[0])}
agg = {}
for r in rows[1:]:
    k = r[ix["Kernel Name"]][:48]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1, "nsecond": 1e-6,
             "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1, "GB": 1, "MB": 1e-3}.get(unit, 1)
    agg.setdefault(k, {}).setdefault(r[ix["Metric Name"]], []).append(v * scale)
for k, d in agg.items():
    if flt not in k:
        continue
    t = d.get("gpu__time_duration.sum", [0])
    rd = d.get("dram__bytes_read.sum", [0])
    wr = d.get("dram__bytes_write.sum", [0])
    print(f"{k:48s} n={len(t):3d} {sum(t) / len(t):9.3f} ms  rd {sum(rd) / len(rd):7.2f} GB  "
          f"wr {sum(wr) / len(wr):7.2f} GB")
