"""Summarise an ncu --set full report of one kernel (run here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [-k kernel_regex] [--json out.json] [--top 25]

Prints duration, DRAM bytes/throughput, occupancy, issue utilisation, the stall-reason mix and
the hottest SASS instructions (stall samples + execution counts).
"""
import argparse
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--json")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("-k", default=None, help="kernel name regex (reports holding several kernels)")
    args = ap.parse_args()
    filt = ["-k", "regex:" + args.k] if args.k else []
    rows = ncu_csv(args.rep, "raw", filt)
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    summary = {"kernel": d.get("Kernel Name", "?")}
    for k in KEYS:
        if k in d:
            summary[k] = f"{d[k]} {u.get(k, '')}".strip()
    stalls = sorted(((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0))
                     for h, v in d.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                     and not h.endswith("not_issued")), key=lambda x: -x[1])
    tot = sum(v for _, v in stalls) or 1.0
    summary["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in stalls[:10]}
    for k, v in summary.items():
        print(f"{k:70s} {v}")
    src = ncu_csv(args.rep, "source", ["--print-source", "sass", *filt])
    hdr2 = src[1]
    ix = {h: i for i, h in enumerate(hdr2)}
    top, tot_s, tot_e = [], 0, 0
    for r in src[2:]:
        if r and r[0] in ("Kernel Name", "Address"):
            break  # a second kernel's block: keep the first
        if len(r) < len(hdr2):
            continue
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        e = int(r[ix["Instructions Executed"]] or 0)
        tot_s += s
        tot_e += e
        top.append((s, r[ix["Address"]][-5:], r[ix["Source"]].strip()[:72], e))
    print(f"\nstall samples {tot_s}, warp instructions {tot_e}")
    for s, a, srcl, e in sorted(top, reverse=True)[:args.top]:
        print(f"{100 * s / max(tot_s, 1):5.1f}% {a} {srcl:72s} {e}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump(summary, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())
