"""Benchmark of the B200 parametric segment voxelizer (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl ours|reference]

A step is one pass of the hot path over one batch: plan kernel + look-back offset scan
(batch_preprocess) and the emit (batch_voxelize's kernel + assemble phases), inputs resident in
HBM. Workloads (BASELINE.json configs):
  cfg4 (default)  4M segments, N ~ U{1..2048}, voxel-list output        -> "weak" scaling (a shard
                  of 4M segments per rank, no data-path collective)
  cfg1            65,536 segments, N = 128, 512^3 volume, voxel list     -> weak
  cfg3            16M segments, N = 64, 1024^3 bitmap                    -> weak
  cfg5            64M segments, N ~ U{1..2048}, 4096^3 bitmap, z-slab per rank -> strong
  cfg2            one segment of 10^6 voxels (latency)                   -> replicas
value = Gvoxels/s (sum of deduplicated chain lengths == reference BatchResult.total_voxels, or
bitmap samples for bitmap configs) over all ranks / max-over-ranks device time.
`--impl reference` times the reference's own CPU run_batch (oracle/_ref, compiled unmodified from
/root/reference) on the host's cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {
    "cfg1": dict(kind="list", n=65536, len_fixed=128, len_max=0, V=512, seed=0x5EED0101,
                 desc="65,536 random 3D segments of fixed length 128 voxels in a 512^3 volume, "
                      "voxel-coordinate list output", scaling="weak"),
    "cfg2": dict(kind="single", n=1, len_fixed=1_000_000, len_max=0, V=0, seed=0x5EED0102,
                 desc="single 3D segment of 10^6 voxels (latency regime)", scaling="weak"),
    "cfg3": dict(kind="bitmap", n=16 * 1024 * 1024, len_fixed=64, len_max=0, V=1024,
                 seed=0x5EED0103, desc="16M fixed-length segments (64 voxels) in a 1024^3 volume, "
                 "packed occupancy bitmap output", scaling="weak"),
    "cfg4": dict(kind="list", n=4 * 1024 * 1024, len_fixed=0, len_max=2048, V=4096,
                 seed=0x5EED0104, desc="4M arbitrary-length segments (uniform 1-2048 voxels), "
                 "scan-balanced emit to a voxel list", scaling="weak"),
    "cfg5": dict(kind="slab", n=64 * 1024 * 1024, len_fixed=0, len_max=2048, V=4096,
                 seed=0x5EED0105, desc="64M arbitrary-length segments in a 4096^3 bitmap volume, "
                 "z-slab sharded", scaling="strong"),
}
L2_BYTES = 126 * 1024 * 1024


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and throttle reasons sampled every ~5 ms during the timed region: NVML polled
    from a thread in this process (nvidia-ml-py), else `nvidia-smi -lms` line-buffered through
    stdbuf. (A plain nvidia-smi pipe is block-buffered: a short timed region can end before its
    first line arrives.)"""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples: list[tuple[float, float, frozenset]] = []  # (sm MHz, max MHz, reasons)
        self.proc = None
        self.stop = threading.Event()
        self.t = None
        self.error = None
        self.source = None

    def _nvml_loop(self, nv, h):
        bits = [(name, getattr(nv, attr, 0)) for name, attr in self.REASONS]
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((float(sm), float(mx),
                                     frozenset(n for n, b in bits if b and (r & b))))
            except Exception as e:  # (reported once in the summary)
                self.error = self.error or repr(e)
            self.stop.wait(0.005)

    def _smi_loop(self):
        names = [n for n, _ in self.REASONS]
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                self.samples.append((float(parts[1]), float(parts[2]), frozenset(
                    n for n, v in zip(names, parts[3:7]) if v.lower() == "active")))
            except ValueError:
                continue

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.t = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.source = "nvml"
        except Exception as e:
            self.error = repr(e)
            try:
                cmd = ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                       "-i", str(self.gpu), "-lms", "25"]
                if shutil.which("stdbuf"):
                    cmd = ["stdbuf", "-oL"] + cmd
                self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                             stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._smi_loop, daemon=True)
                self.source = "nvidia-smi"
            except Exception as e:
                self.error = (self.error or "") + " / " + repr(e)
                self.t = None
        if self.t:
            self.t.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "source": self.source, "error": self.error}
        reasons = set()
        for _, _, r in self.samples:
            reasons |= r
        return {"sm_mhz": statistics.median(x[0] for x in self.samples),
                "sm_max_mhz": max(x[1] for x in self.samples), "reasons": sorted(reasons),
                "samples": len(self.samples), "source": self.source}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def barrier_max(torch, value: float, world: int) -> float:
    from paper_2009_09500_b200.shard import max_over_ranks
    return max_over_ranks(value) if world > 1 else value


def barrier_sum(torch, value: float, world: int) -> float:
    from paper_2009_09500_b200.shard import sum_over_ranks
    return sum_over_ranks(value) if world > 1 else value


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def load_traffic(workload: str):
    """(dram bytes per launch of the dominant kernel, source) from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f).get(workload)
        return (t["bytes"], t["source"]) if t else (None, None)
    except Exception:
        return None, None


# ============================================================================ reference arm
def cpu_reference(cfg, workload, steps, warmup, sample_segments=None, quiet=False):
    """The reference's own run_batch (oracle/_ref) with all host threads on a bounded sample."""
    from oracle.pyoracle import REF_SO, Oracle, RefOracle
    cores = os.cpu_count() or 1
    orc = Oracle()
    if os.path.exists(REF_SO):
        impl, kind = RefOracle(), "reference"
    else:
        impl, kind = None, "port"
    if cfg["kind"] == "single":
        segs = orc.gen_batch(1, cfg["len_fixed"], 0, cfg["V"], cfg["seed"])
        nsamp = 1
    else:
        nsamp = sample_segments or {"list": 131072, "bitmap": 262144, "slab": 131072}[cfg["kind"]]
        nsamp = min(nsamp, cfg["n"])
        segs = orc.gen_batch(nsamp, cfg["len_fixed"], cfg["len_max"], cfg["V"], cfg["seed"])
    times, total = [], 0
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        if impl is not None:
            _, _, total, _ = impl.run_batch(segs, workers=cores, group_size=64, with_voxels=False)
        else:
            _, _, total = orc.run_batch(segs, nthreads=cores)
        dt = time.perf_counter() - t0
        if it >= warmup:
            times.append(dt)
    med = statistics.median(times)
    gvps = total / med / 1e9
    sample = (f"{nsamp} of {cfg['n']} segments of {workload} ({total} voxels), "
              f"run_batch(workers={cores}, group_size=64), median of {steps} after {warmup} warm-up")
    return {"value": gvps, "unit": "Gvoxels/s", "cores": cores, "kind": kind, "sample": sample,
            "ms_per_step": med * 1e3, "segments_per_s": nsamp / med}


def run_reference_arm(args, cfg):
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return
    r = cpu_reference(cfg, args.workload, args.steps, args.warmup)
    line = {"metric": "Gvoxels/s", "value": r["value"], "unit": "Gvoxels/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SplitMix64 volume generator, same seeds as the GPU arm)",
            "config": {"workload": args.workload, "desc": cfg["desc"]},
            "segments_per_s": r["segments_per_s"],
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": "Gvoxels/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ============================================================================ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--segments", type=int, default=0, help="override the segment count")
    ap.add_argument("--equal-slabs", action="store_true",
                    help="bitmap slabs of equal depth instead of equal sample counts")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: ranks may share one GPU (functional test of the N > 1 path)")
    args = ap.parse_args()
    cfg = dict(WORKLOADS[args.workload])
    if args.segments:
        cfg["n"] = args.segments
    if args.impl == "reference":
        return run_reference_arm(args, cfg)

    import torch
    world, rank, local = dist_setup(args)
    if args.dist_backend == "gloo":  # functional check of the N > 1 path on a one-GPU box
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    import paper_2009_09500_b200 as vx
    ctx = vx.Context(local)
    # one dedicated stream for everything: the library's kernels, torch's allocations and the
    # timing events are all ordered on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    # ---- inputs: generated on the device by the product generator (bit-identical to oracle)
    kind = cfg["kind"]
    n = cfg["n"]
    seed = cfg["seed"] + (rank if cfg["scaling"] == "weak" else 0) * 0x1000193
    d_segs = torch.empty((n, 6), dtype=torch.float64, device="cuda")
    ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, cfg["len_fixed"], cfg["len_max"],
                                       cfg["V"], seed, d_segs.data_ptr(), 1))
    V = cfg["V"]
    slab_cuts = None
    if kind == "slab":  # the z-slab partitioner: rank r owns one slab
        from paper_2009_09500_b200.shard import sample_balanced_slabs, slab_bounds
        if world > 1 and not args.equal_slabs:
            # equal sample counts (the work), from the batch itself: decided once, before timing
            bb = vx.Batch(None, ctx=ctx, device_ptr=d_segs.data_ptr(), n=n)
            slabs = sample_balanced_slabs(bb.slab_samples, V, world)
            bb.close()
            z_lo, z_hi = slabs[rank]
            slab_cuts = "sample-balanced (64 coarse bins)"
        else:
            z_lo, z_hi = slab_bounds(V, world, rank)
            slab_cuts = "equal depth"
    else:
        z_lo, z_hi = 0, V

    out = chain = words = None
    batch = vx.Batch(None, ctx=ctx, device_ptr=d_segs.data_ptr(), n=n)
    capacity = batch.capacity
    if kind in ("list", "single"):
        out = torch.empty((capacity, 3), dtype=torch.int32, device="cuda")
        chain = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    else:
        nwords = (V * V * (z_hi - z_lo) + 63) // 64
        words = torch.zeros(nwords, dtype=torch.int64, device="cuda")
    batch.close()

    # a rank's slab of the bitmap: every step filters the (broadcast) segments down to those
    # that reach the slab on the device, then plans and bins only those
    slab_segs = None
    if kind == "slab" and (z_lo > 0 or z_hi < V):
        from paper_2009_09500_b200.shard import select_slab_segments
        slab_segs = torch.empty_like(d_segs)

    def step():
        src, cnt = d_segs, n
        if slab_segs is not None:
            cnt = select_slab_segments(ctx, d_segs.data_ptr(), n, z_lo, z_hi, slab_segs.data_ptr())
            src = slab_segs
            if cnt == 0:  # (no segment reaches this slab: nothing to do)
                return None, 0, 0, 0
        b = vx.Batch(None, ctx=ctx, device_ptr=src.data_ptr(), n=cnt)
        if kind in ("list", "single"):
            units = b.emit_list_device(out.data_ptr(), capacity, chain.data_ptr())
        else:
            b.emit_bitmap_device(words.data_ptr(), V, z_lo, z_hi, clip=(kind == "slab"))
            units = None
        plan_ns, emit_ns, aux_ns = b.gpu_timing()
        b.close()
        return units, plan_ns, emit_ns, aux_ns

    for _ in range(args.warmup):
        units, _, _, _ = step()
    if kind in ("bitmap", "slab"):
        bb = vx.Batch(None, ctx=ctx, device_ptr=d_segs.data_ptr(), n=n)
        units = bb.slab_samples(z_lo, z_hi) if kind == "slab" else bb.capacity
        bb.close()
    torch.cuda.synchronize()
    barrier(world)

    launches0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    emit_ms, plan_ms, aux_ms = [], [], []
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier(world)
        ev0.record(stream)
        for _ in range(args.steps):
            u, p_ns, e_ns, a_ns = step()
            plan_ms.append(p_ns / 1e6)
            emit_ms.append(e_ns / 1e6)
            aux_ms.append(a_ns / 1e6)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    launches = ctx.launches - launches0
    local_ms = ev0.elapsed_time(ev1)
    ms = barrier_max(torch, local_ms, world) / args.steps
    total_units = barrier_sum(torch, float(units), world)
    total_segments = barrier_sum(torch, float(n), world) if cfg["scaling"] == "weak" else float(n)
    value = total_units / (ms / 1e3) / 1e9

    # ---- roofline of the dominant (emit) kernel: algorithmic bytes / its event-timed duration
    hbm, peak_src = peaks()
    emit_avg = statistics.mean(emit_ms)
    if kind in ("list", "single"):
        alg_bytes = 12 * units + 8 * (n + 1) + 48 * n
        dominant = "list_fused_kernel (count + emit tasks overlapped)" \
            if capacity >= 43_000_000 else "list_emit_kernel"
    else:
        alg_bytes = 8 * ((V * V * (z_hi - z_lo) + 63) // 64) + 48 * n
        dominant = "tiles_fill_kernel"
    achieved = alg_bytes / (emit_avg / 1e3) / 1e9
    # FP64-pipe view: every sample costs 10 FP64 operations (3 DMUL + 3 DADD for S + W*k, 3 DADD
    # for llround, 1 DADD for k); peak = DADD/DMUL issue measured on this pool's B200s
    # (tools/microbench_fp64.cu: 63.4 op/clk/SM, 18.42 TOP/s at 1965 MHz; profiles/)
    samples = float(units) if kind in ("bitmap", "slab") else None
    traffic, traffic_src = load_traffic(args.workload)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": dominant, "kernel_ms": emit_avg, "plan_kernel_ms": statistics.mean(plan_ms),
                "aux_kernels_ms": statistics.mean(aux_ms),
                "algorithmic_bytes": alg_bytes, "peak_source": peak_src,
                "step_share": emit_avg / ms}
    if samples is not None:  # bitmaps: the FP64 evaluation, not HBM, bounds the fill kernel
        fp64 = 10.0 * samples / (emit_avg / 1e3) / 1e12
        roofline["fp64"] = {"achieved": fp64, "peak": 18.42, "unit": "TOP/s", "frac": fp64 / 18.42,
                            "source": "profiles/r1_microbench_fp64.txt (measured DADD/DMUL rate)"}

    # ---- end to end through the public host API (pinned host buffers, copies inside the timer)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(vx, ctx, torch, d_segs, cfg, kind, n, capacity, units, z_lo, z_hi, world,
                      max(1, min(args.steps, 3)))
    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        del out, chain, words
        torch.cuda.empty_cache()
        try:
            r = cpu_reference(cfg, args.workload, steps=3, warmup=1)
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # the checker may be absent on a box without oracle builds
            cpu = {"value": None, "unit": "Gvoxels/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": "Gvoxels/s", "value": value, "unit": "Gvoxels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (SplitMix64 volume generator on device; inputs "
            "larger than L2)" if n * 48 > L2_BYTES else "synthetic (SplitMix64 volume generator)",
            "config": {"workload": args.workload, "desc": cfg["desc"], "segments_per_rank": n,
                       "volume": V, "z_slab": [z_lo, z_hi] if kind == "slab" else None,
                       "slab_cuts": slab_cuts,
                       "l2": "inputs+outputs larger than L2 (no flush needed)"
                       if alg_bytes > 2 * L2_BYTES else "L2-resident working set",
                       "parallelism": f"{cfg['scaling']}-sharded x{world}"},
            "segments_per_s": total_segments / (ms / 1e3),
            "units": "deduplicated voxels (BatchResult.total_voxels)" if kind in ("list", "single")
            else "bitmap samples set", "units_per_step": total_units,
            "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_e2e(vx, ctx, torch, d_segs, cfg, kind, n, capacity, units, z_lo, z_hi, world, steps):
    """Same metric through the public host-buffer API: pinned host segments -> Batch (H2D +
    plan) -> emit to pinned host buffers (kernel + D2H), timed on the host around the call."""
    import psutil
    segs_h = vx.pinned_empty((n, 6), np.float64)
    segs_h[:] = d_segs.cpu().numpy()
    V = cfg["V"]
    if kind in ("list", "single"):
        need = 12 * units + 8 * (n + 1)
        avail = psutil.virtual_memory().available
        if need * world * 1.6 < avail:
            mode = "full"
            out_h = vx.pinned_empty((max(units, 1), 3), np.int32)
            chain_h = vx.pinned_empty((n + 1,), np.int64)
        else:
            mode = "unavailable"
            return {"value": None, "unit": "Gvoxels/s", "h2d_bytes_per_step": 48 * n,
                    "d2h_bytes_per_step": need, "note": f"host RAM {avail} < {need * world}"}
    else:
        mode = "full"
        nwords = (V * V * (z_hi - z_lo) + 63) // 64
        words_h = vx.pinned_empty((nwords,), np.uint64)
        need = 8 * nwords
    torch.cuda.empty_cache()
    times = []
    for it in range(steps + 1):
        barrier(world)
        t0 = time.perf_counter()
        b = vx.Batch(segs_h, ctx=ctx)
        if kind in ("list", "single"):
            _, _, total = b.emit_list(out=out_h, chain_off=chain_h)
            assert total == units
        else:
            b.emit_bitmap(V, z_lo, z_hi, clip=(kind == "slab"), words=words_h, overwrite=True)
        b.close()
        dt = time.perf_counter() - t0
        if it > 0:
            times.append(dt)
    sec = barrier_max(torch, statistics.median(times), world)
    total_units = barrier_sum(torch, float(units), world)
    h2d = 48 * n
    return {"value": total_units / sec / 1e9, "unit": "Gvoxels/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": need, "ms_per_step": sec * 1e3, "mode": mode,
            "api": "paper_2009_09500_b200.Batch(host) + Batch.emit_list/emit_bitmap(host)"}


if __name__ == "__main__":
    main()
