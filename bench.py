"""Benchmark of the B200 parametric segment voxelizer (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg5] [--impl ours|reference]
                    [--verify]

A step is one pass of the hot path over one batch: plan kernel + look-back offset scan
(batch_preprocess) and the emit (batch_voxelize's kernel + assemble phases), inputs resident in
HBM; a bitmap step writes a fresh bitmap of its batch (VXG_BITMAP_OVERWRITE; VXG_BENCH_OR=1
ORs into the buffer instead). Workloads (BASELINE.json configs; the other configs are `--workload` lines):
  cfg5 (default)  64M segments, N ~ U{1..2048}, 4096^3 bitmap  -> z-slab per rank (strong)
  cfg3            16M segments, N = 64, 1024^3 bitmap          -> z-slab per rank (strong)
  cfg4            4M segments, N ~ U{1..2048}, voxel list      -> one batch cut into sample-
                                                                  balanced segment ranges (strong)
  cfg1            65,536 segments, N = 128, 512^3, voxel list   -> as cfg4 (strong)
  cfg2            one segment of 10^6 voxels (latency)          -> replicas
value = Gvoxels/s: voxels = the batch's deduplicated chain voxels (reference
BatchResult.total_voxels, src/batch.cpp:148-150) -- for bitmap configs counted once per batch by
the device count pass -- over the max-over-ranks device time; samples/s and segments/s beside.
`--impl reference` times the reference's own CPU code (oracle/_ref, compiled unmodified from
/root/reference): run_batch on all host cores (+ the bit-setting pass for bitmap configs) over a
bounded sample of the same workload, in the same unit.
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

# kind: list (one batch, sample-balanced segment ranges per rank), slab (bitmap, one z-slab per
# rank), single (one segment: replicas). cpu_sample: segments of the CPU arm's bounded sample.
WORKLOADS = {
    "cfg1": dict(kind="list", n=65536, len_fixed=128, len_max=0, V=512, seed=0x5EED0101,
                 desc="65,536 random 3D segments of fixed length 128 voxels in a 512^3 volume, "
                      "voxel-coordinate list output", scaling="strong", cpu_sample=65536),
    "cfg2": dict(kind="single", n=1, len_fixed=1_000_000, len_max=0, V=0, seed=0x5EED0102,
                 desc="single 3D segment of 10^6 voxels (latency regime)", scaling="weak",
                 cpu_sample=1),
    "cfg3": dict(kind="slab", n=16 * 1024 * 1024, len_fixed=64, len_max=0, V=1024,
                 seed=0x5EED0103, desc="16M fixed-length segments (64 voxels) in a 1024^3 volume, "
                 "packed occupancy bitmap output, z-slab sharded", scaling="strong",
                 cpu_sample=1 << 20),
    "cfg4": dict(kind="list", n=4 * 1024 * 1024, len_fixed=0, len_max=2048, V=4096,
                 seed=0x5EED0104, desc="4M arbitrary-length segments (uniform 1-2048 voxels), "
                 "scan-balanced emit to a voxel list", scaling="strong", cpu_sample=262144),
    "cfg5": dict(kind="slab", n=64 * 1024 * 1024, len_fixed=0, len_max=2048, V=4096,
                 seed=0x5EED0105, desc="64M arbitrary-length segments in a 4096^3 bitmap volume, "
                 "z-slab sharded", scaling="strong", cpu_sample=262144),
}
DEFAULT_WORKLOAD = "cfg5"
L2_BYTES = 126 * 1024 * 1024
# the bitmap fill's inner loop: warp instructions per 32 in-tile samples (62 per 4-sample unrolled
# iteration of fx_loop_int, read from cuobjdump -sass of tiles_fill_kernel<32, 1, false>, the
# instantiation cfg3 and cfg5 run)
FILL_SLOTS_PER_ROW = 15.5
SM_MAX_MHZ_FALLBACK = 1965.0  # B200 max SM clock (MEASURED_PEAKS.json sm_max_mhz)


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


def time_slab_step(vx, shard, ctx, torch, d_segs, n, V, z_lo, z_hi) -> float:
    """One rank's bitmap step on slab [z_lo, z_hi) (filter, plan, bin, fill), device ms of the
    second of two runs -- the partition's calibration, before the timed region."""
    local = torch.empty_like(d_segs)
    words = torch.zeros(max(V * V * (z_hi - z_lo) // 64, 1), dtype=torch.int64, device="cuda")
    ms = 0.0
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        k = shard.select_slab_segments(ctx, d_segs.data_ptr(), n, z_lo, z_hi, local.data_ptr())
        if k > 0:
            b = vx.Batch(None, ctx=ctx, device_ptr=local.data_ptr(), n=k).set_slab(z_lo, z_hi)
            b.emit_bitmap_device(words.data_ptr(), V, z_lo, z_hi, True,
                                 overwrite=not os.environ.get("VXG_BENCH_OR"))
            b.close()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    del local, words
    torch.cuda.empty_cache()
    return ms


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def barrier_max(value: float, world: int) -> float:
    from paper_2009_09500_b200.shard import max_over_ranks
    return max_over_ranks(value) if world > 1 else value


def barrier_sum(value: float, world: int) -> float:
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
def _median_time(fn, reps: int, warmup: int):
    for _ in range(warmup):
        fn()
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        times.append(time.perf_counter() - t0)
    return statistics.median(times), r


def cpu_reference(cfg, workload, reps, warmup, quiet=False):
    """The reference's own CPU code (oracle/_ref; the C restatement if _ref is absent) on a
    bounded sample of the workload -- its first cpu_sample segments -- timed like its harness
    (src/bench.cpp:188-215: warm-ups, then the median of the repetitions):
      * run_batch(workers = all host cores, group_size 64), the CLI default
        (tools/voxline_cli.cpp:72-74,97), plus for bitmap configs the harness's bit-setting pass
        over the chains (times reported separately);
      * the sequential method: one voxelize_parametric call per segment on one core.
    Both in deduplicated voxels per second (BatchResult.total_voxels), the GPU arm's unit."""
    from oracle.pyoracle import REF_SO, Oracle, RefOracle
    cores = os.cpu_count() or 1
    orc = Oracle()
    ref = RefOracle() if os.path.exists(REF_SO) else None
    kind = "reference" if ref is not None else "port"
    nsamp = min(cfg["cpu_sample"], cfg["n"])
    segs = orc.gen_batch(nsamp, cfg["len_fixed"], cfg["len_max"], cfg["V"], cfg["seed"])
    V = cfg["V"]
    split = None
    if cfg["kind"] == "slab":
        words = np.zeros((V * V * V + 63) // 64, np.uint64)
        words[:] = 0  # (touched once: page faults are not the reference's cost)
        parts = []

        def body():
            if ref is not None:
                _, tot, _, t = ref.run_batch_bitmap(segs, V, 0, V, workers=cores, group_size=64,
                                                    words=words)
                parts.append(t)
                return tot
            t0 = time.perf_counter_ns()
            _, _, tot = orc.run_batch(segs, nthreads=cores)
            t1 = time.perf_counter_ns()
            orc.bitmap(segs, V, nthreads=cores)
            parts.append((t1 - t0, time.perf_counter_ns() - t1))
            return tot
        med, total = _median_time(body, reps, warmup)
        timed = parts[warmup:]
        split = {"run_batch_ms": statistics.median(p[0] for p in timed) / 1e6,
                 "bit_setting_ms": statistics.median(p[1] for p in timed) / 1e6}
        what = (f"run_batch(workers={cores}, group_size=64) + the harness bit-setting pass "
                f"over its chains into the {V}^3 bitmap")
    else:
        def body():
            if ref is not None:
                return ref.run_batch(segs, workers=cores, group_size=64, with_voxels=False)[2]
            return orc.run_batch(segs, nthreads=cores)[2]
        med, total = _median_time(body, reps, warmup)
        what = f"run_batch(workers={cores}, group_size=64)"
    # the sequential method on one core (src/bench.cpp:188-205), on at most 16,384 segments
    nseq = min(nsamp, 16384)
    seq_segs = segs[:nseq]
    if ref is not None:
        seq_med, seq_total = _median_time(lambda: ref.sequential_map(seq_segs), max(reps, 5), 2)
    else:
        seq_med, seq_total = _median_time(lambda: orc.run_batch(seq_segs, nthreads=1)[2],
                                          max(reps, 5), 2)
    sample = (f"first {nsamp} of {cfg['n']} segments of {workload} ({total} voxels): {what}, "
              f"median of {reps} after {warmup} warm-up(s)")
    out = {"value": total / med / 1e9, "unit": "Gvoxels/s", "cores": cores, "kind": kind,
           "sample": sample, "ms_per_step": med * 1e3, "segments_per_s": nsamp / med,
           "voxels_per_step": total,
           "sequential_1core": {"value": seq_total / seq_med / 1e9, "unit": "Gvoxels/s",
                                "cores": 1, "sample": f"first {nseq} segments, "
                                "voxelize_parametric per segment (src/bench.cpp:188-205), "
                                f"median of {max(reps, 5)} after 2 warm-ups",
                                "ms": seq_med * 1e3}}
    if split:
        out["phases_ms"] = split
    return out


def run_reference_arm(args, cfg):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    r = cpu_reference(cfg, args.workload, max(1, args.steps), args.warmup)
    line = {"metric": "Gvoxels/s", "value": r["value"], "unit": "Gvoxels/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SplitMix64 volume generator, same seeds as the GPU arm)",
            "config": {"workload": args.workload, "desc": cfg["desc"]},
            "segments_per_s": r["segments_per_s"],
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "sequential_1core": r["sequential_1core"],
            "e2e": {"value": r["value"], "unit": "Gvoxels/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if "phases_ms" in r:
        line["phases_ms"] = r["phases_ms"]
    print(json.dumps(line), flush=True)


# ============================================================================ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--verify", action="store_true",
                    help="N > 1: compare every rank's output digest with the one-rank result")
    ap.add_argument("--segments", type=int, default=0, help="override the segment count")
    ap.add_argument("--no-rebalance", action="store_true",
                    help="bitmaps, N > 1: keep the sample-balanced slabs (no timed refinement)")
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
    world, rank, local = dist_setup()
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
    from paper_2009_09500_b200 import shard
    ctx = vx.Context(local)
    # one dedicated stream for everything: the library's kernels, torch's allocations and the
    # timing events are all ordered on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    # ---- inputs: the whole batch, generated on the device by the product generator
    # (bit-identical to the oracle's); every rank holds the same batch
    kind, n, V = cfg["kind"], cfg["n"], cfg["V"]
    d_segs = torch.empty((n, 6), dtype=torch.float64, device="cuda")
    ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, cfg["len_fixed"], cfg["len_max"],
                                       V, cfg["seed"], d_segs.data_ptr(), 1))

    # ---- partition, decided once before timing
    part = {}
    batch_voxels = None
    if kind == "list":
        cuts = [0, n]
        if world > 1:
            bb = vx.Batch(None, ctx=ctx, device_ptr=d_segs.data_ptr(), n=n)
            cuts = [int(c) for c in shard.batch_sample_cuts(bb, world)]
            bb.close()
        s0, s1 = cuts[rank], cuts[rank + 1]
        part = {"segments": [s0, s1], "cuts": "sample-balanced segment ranges of one batch"
                if world > 1 else "whole batch"}
        z_lo, z_hi = 0, V
    elif kind == "slab":
        bb = vx.Batch(None, ctx=ctx, device_ptr=d_segs.data_ptr(), n=n)
        if world > 1 and not args.equal_slabs:
            slabs = shard.sample_balanced_slabs(bb.slab_samples, V, world)
            part["cuts"] = "sample-balanced z-slabs (64 coarse bins)"
            if not args.no_rebalance:  # one refinement from every rank's measured step
                t = time_slab_step(vx, shard, ctx, torch, d_segs, n, V, *slabs[rank])
                slabs = shard.time_balanced_slabs(bb.slab_samples, V, slabs,
                                                  shard.gather_floats(t))
                part["cuts"] = ("sample-balanced z-slabs (64 coarse bins), rebalanced once from "
                                "every rank's measured step before timing")
        else:
            slabs = [shard.slab_bounds(V, world, r) for r in range(world)]
            part["cuts"] = "equal-depth z-slabs"
        z_lo, z_hi = slabs[rank]
        part["z_slab"] = [z_lo, z_hi]
        batch_voxels = bb.count_voxels()  # BatchResult.total_voxels of the whole batch
        rank_samples = bb.slab_samples(z_lo, z_hi)
        batch_samples = bb.capacity
        bb.close()
        s0, s1 = 0, n
    else:
        s0, s1 = 0, n
        z_lo, z_hi = 0, V
    my_n = s1 - s0
    my_ptr = d_segs.data_ptr() + 48 * s0

    out = chain = words = None
    if kind in ("list", "single"):
        bb = vx.Batch(None, ctx=ctx, device_ptr=my_ptr, n=my_n)
        capacity = bb.capacity
        bb.close()
        out = torch.empty((max(capacity, 1), 3), dtype=torch.int32, device="cuda")
        chain = torch.empty(my_n + 1, dtype=torch.int64, device="cuda")
    else:
        capacity = None
        nwords = (V * V * (z_hi - z_lo) + 63) // 64
        words = torch.zeros(nwords, dtype=torch.int64, device="cuda")

    # a rank's slab of the bitmap: every step filters the (whole) batch down to the segments
    # that reach the slab on the device, then plans and bins only those
    slab_segs = torch.empty_like(d_segs) if kind == "slab" and (z_lo > 0 or z_hi < V) else None
    sel_n = [my_n]

    # small list batches: the one-launch path (plan + count + prefix + emit in one kernel,
    # vxg_run_batch_device), enqueued back to back; the total is read once after the loop
    small = kind == "list" and my_n <= (1 << 18)
    small_ev = []
    ev_pool = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(max(args.steps, args.warmup))] if small else []

    def step_small():
        e0, e1 = ev_pool[len(small_ev)]
        e0.record(stream)
        vx.run_batch_device(my_ptr, my_n, out.data_ptr(), capacity, chain.data_ptr(), ctx=ctx,
                            sync=False)
        e1.record(stream)
        small_ev.append((e0, e1))
        return None, 0, 0, 0

    seg_host = d_segs[s0].cpu().numpy() if kind == "single" else None  # (48 B: the input)

    def step():
        if small:
            return step_small()
        if kind == "single":  # voxelize_parametric: one launch + one readback of the count
            u = vx.voxelize_parametric_device(seg_host, out.data_ptr(), capacity, ctx=ctx)
            return u, 0, 0, 0  # (its kernel time is read once, after the timed loop)
        src, cnt = my_ptr, my_n
        if slab_segs is not None:
            cnt = shard.select_slab_segments(ctx, d_segs.data_ptr(), n, z_lo, z_hi,
                                             slab_segs.data_ptr())
            src = slab_segs.data_ptr()
            sel_n[0] = cnt
            if cnt == 0:  # (no segment reaches this slab: nothing to do)
                return 0, 0, 0, 0
        b = vx.Batch(None, ctx=ctx, device_ptr=src, n=cnt)
        if slab_segs is not None:
            b.set_slab(z_lo, z_hi)  # (filtered above: the tile path skips its own filter)
        if kind in ("list", "single"):
            units = b.emit_list_device(out.data_ptr(), capacity, chain.data_ptr())
        else:
            # (overwrite: the step's bitmap replaces the buffer -- the fill stores every word,
            # no read of the old ones; VXG_BENCH_OR=1 ORs into the buffer instead)
            b.emit_bitmap_device(words.data_ptr(), V, z_lo, z_hi, clip=True,
                                 overwrite=not os.environ.get("VXG_BENCH_OR"))
            units = batch_voxels
        plan_ns, emit_ns, aux_ns = b.gpu_timing()
        b.close()
        return units, plan_ns, emit_ns, aux_ns

    units = 0
    for _ in range(args.warmup):
        units, _, _, _ = step()
    if small:
        units = vx.run_batch_device_result(ctx)[0]
        small_ev.clear()
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
    if small:  # (every step computed the same batch; its result, errors included, read once)
        assert vx.run_batch_device_result(ctx)[0] == units
        emit_ms = [a.elapsed_time(b) for a, b in small_ev]
        plan_ms = aux_ms = [0.0]
    if kind == "single":  # the last call's long_chain_kernel (CUDA events inside the library)
        emit_ms = [vx.voxelize_parametric_kernel_ns(ctx) / 1e6]
    ms = barrier_max(local_ms, world) / args.steps
    if kind == "slab":
        total_units = float(batch_voxels)
        total_samples = float(batch_samples)
    else:
        total_units = barrier_sum(float(units), world)
        total_samples = barrier_sum(float(capacity), world)
    value = total_units / (ms / 1e3) / 1e9

    # ---- roofline of the dominant kernel: its work / its event-timed duration
    hbm, peak_src = peaks()
    emit_avg = statistics.mean(emit_ms) if emit_ms else 0.0
    traffic, traffic_src = load_traffic(args.workload)
    if kind in ("list", "single"):
        alg_bytes = 12 * units + (8 * (my_n + 1) + 48 * my_n if kind == "list" else 0)
        achieved = alg_bytes / (emit_avg / 1e3) / 1e9
        dominant = ("long_chain_kernel (plan + samples + dedup + look-back + emit in one launch)"
                    if kind == "single"
                    else "list_small_kernel (plan + count + prefix + emit in one launch)" if small
                    else "list_fused_kernel (count + emit tasks overlapped)"
                    if capacity >= 43_000_000 else "list_emit_kernel")
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                    "algorithmic_bytes": alg_bytes, "peak_source": peak_src}
    else:
        # The fill writes an 8 GiB bitmap for 68.8 G samples (cfg5): HBM is not its bound (the
        # hbm object below). It is issue-bound: every in-tile sample costs its lane the fixed-
        # point loop body, FILL_SLOTS_PER_ROW warp instructions per 32 samples (fx_loop_int in
        # csrc/vxg_bitmap.cu, counted in the compiled SASS), against a peak of one warp
        # instruction per cycle per SM sub-partition. frac = the share of the issue slots that do
        # that work (the rest: per-piece setup, lanes idling at piece ends, stalls).
        num_sms = torch.cuda.get_device_properties(local).multi_processor_count
        sm_max_mhz = float(clocks.summary().get("sm_max_mhz") or 0.0) or SM_MAX_MHZ_FALLBACK
        rows = rank_samples / 32.0
        issue = FILL_SLOTS_PER_ROW * rows / (emit_avg / 1e3) / 1e9
        issue_peak = 4 * num_sms * sm_max_mhz * 1e6 / 1e9
        alg_bytes = 8 * ((V * V * (z_hi - z_lo) + 63) // 64) + 48 * sel_n[0]
        achieved = alg_bytes / (emit_avg / 1e3) / 1e9
        dominant = "tiles_fill_kernel"
        roofline = {"bound": "issue", "achieved": issue, "peak": issue_peak,
                    "unit": "G warp-instructions/s", "frac": issue / issue_peak,
                    "traffic": traffic, "traffic_source": traffic_src,
                    "work": f"{FILL_SLOTS_PER_ROW} loop instructions x {rank_samples} samples / 32 "
                            "(32.32 fixed-point steps, the near-boundary test, the shared address "
                            "and the shared-memory OR per sample)",
                    "peak_source": f"4 sub-partitions x {num_sms} SMs x {sm_max_mhz:.0f} MHz "
                                   "(one warp instruction per cycle each)",
                    "hbm": {"achieved": achieved, "peak": hbm, "unit": "GB/s",
                            "frac": achieved / hbm, "algorithmic_bytes": alg_bytes,
                            "peak_source": peak_src}}
    roofline.update({"kernel": dominant, "kernel_ms": emit_avg,
                     "plan_kernel_ms": statistics.mean(plan_ms) if plan_ms else 0.0,
                     "aux_kernels_ms": statistics.mean(aux_ms) if aux_ms else 0.0,
                     "step_share": emit_avg / ms if ms else None})

    # ---- end to end through the public host API (pinned host buffers, copies inside the timer)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(vx, shard, ctx, torch, d_segs, cfg, kind, n, s0, s1, units, capacity, z_lo,
                      z_hi, world, max(1, min(args.steps, 3)), batch_voxels)
    verify = None
    if args.verify:
        verify = run_verify(vx, shard, ctx, torch, d_segs, cfg, kind, n, s0, s1, units, out,
                            chain, words, z_lo, z_hi, world, rank)
    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    seq = None
    if rank == 0 and world == 1 and not args.no_cpu:
        del out, chain, words
        torch.cuda.empty_cache()
        try:
            r = cpu_reference(cfg, args.workload, reps=5, warmup=2)
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
            if "phases_ms" in r:
                cpu["phases_ms"] = r["phases_ms"]
            seq = r["sequential_1core"]
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
            "config": {"workload": args.workload, "desc": cfg["desc"], "segments": n,
                       "volume": V, "partition": part,
                       "l2": "inputs+outputs larger than L2 (no flush needed)"
                       if alg_bytes > 2 * L2_BYTES else "L2-resident working set",
                       "parallelism": f"{cfg['scaling']}-sharded x{world}",
                       **({"bitmap_step": "OR into the buffer" if os.environ.get("VXG_BENCH_OR")
                           else "fresh bitmap per batch (overwrite: every word stored)"}
                          if kind == "slab" else {})},
            "segments_per_s": n * (world if kind == "single" else 1) / (ms / 1e3),
            "samples_per_s": total_samples / (ms / 1e3),
            "units": "deduplicated voxels (BatchResult.total_voxels)",
            "units_per_step": total_units,
            "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
            "sequential_1core": seq, "e2e": e2e, "clocks": clocks.summary(),
        }
        if verify is not None:
            line["verify"] = verify
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_e2e(vx, shard, ctx, torch, d_segs, cfg, kind, n, s0, s1, units, capacity, z_lo, z_hi,
            world, steps, batch_voxels):
    """Same metric through the public host-buffer API, copies inside the timer:
      lists   -- pinned host segments of this rank's range -> Batch (H2D + plan) -> emit_list
                 into pinned host buffers (kernels + D2H);
      bitmaps -- N = 1: Batch(host segments) -> emit_bitmap(host words) (H2D, plan, binning,
                 fill with the streamed D2H of finished z-layers); N > 1: each rank moves 1/N
                 of the segments host->device and one all-gather over NVLink gives every rank
                 the batch (shard.distribute_segments), then the slab's filter, plan and fill
                 with its streamed D2H."""
    import psutil
    segs_h = vx.pinned_empty((n, 6), np.float64)
    segs_h[:] = d_segs.cpu().numpy()
    V = cfg["V"]
    my_n = s1 - s0
    if kind in ("list", "single"):
        need = 12 * units + 8 * (my_n + 1)
        avail = psutil.virtual_memory().available
        if need * world * 1.6 >= avail:
            return {"value": None, "unit": "Gvoxels/s", "h2d_bytes_per_step": 48 * n,
                    "d2h_bytes_per_step": need, "note": f"host RAM {avail} < {need * world}"}
        out_h = vx.pinned_empty((max(units, 1), 3), np.int32)
        chain_h = vx.pinned_empty((my_n + 1,), np.int64)
        h2d = 48 * my_n
        if kind == "single":
            need = 12 * units
    else:
        nwords = (V * V * (z_hi - z_lo) + 63) // 64
        words_h = vx.pinned_empty((nwords,), np.uint64)
        need = 8 * nwords
        h2d = 48 * n // world
        full = torch.empty_like(d_segs) if world > 1 else None
        sel = torch.empty_like(d_segs) if world > 1 and (z_lo > 0 or z_hi < V) else None
    torch.cuda.empty_cache()
    times = []
    for it in range(steps + 1):
        barrier(world)
        t0 = time.perf_counter()
        if kind == "single":  # voxelize_parametric into a pinned host buffer
            assert vx.voxelize_parametric_host(segs_h[s0], out_h, ctx=ctx) == units
        elif kind == "list":
            b = vx.Batch(segs_h[s0:s1], ctx=ctx)
            _, _, total = b.emit_list(out=out_h, chain_off=chain_h)
            assert total == units
        elif world == 1:
            b = vx.Batch(segs_h, ctx=ctx)
            b.emit_bitmap(V, z_lo, z_hi, clip=True, words=words_h, overwrite=True)
        else:
            shard.distribute_segments(segs_h, full)
            src, cnt = full.data_ptr(), n
            if sel is not None:
                cnt = shard.select_slab_segments(ctx, full.data_ptr(), n, z_lo, z_hi,
                                                 sel.data_ptr())
                src = sel.data_ptr()
            b = vx.Batch(None, ctx=ctx, device_ptr=src, n=cnt)
            if sel is not None:
                b.set_slab(z_lo, z_hi)
            b.emit_bitmap(V, z_lo, z_hi, clip=True, words=words_h, overwrite=True)
        if kind != "single":
            b.close()
        dt = time.perf_counter() - t0
        if it > 0:
            times.append(dt)
    sec = barrier_max(statistics.median(times), world)
    total_units = float(batch_voxels) if kind == "slab" else barrier_sum(float(units), world)
    return {"value": total_units / sec / 1e9, "unit": "Gvoxels/s",
            "h2d_bytes_per_step": int(barrier_sum(float(h2d), world)),
            "d2h_bytes_per_step": int(barrier_sum(float(need), world)), "ms_per_step": sec * 1e3,
            "api": ("paper_2009_09500_b200.voxelize_parametric_host (pinned output)"
                    if kind == "single" else
                    "paper_2009_09500_b200.Batch(host) + Batch.emit_list/emit_bitmap(host)")
            + ("; N > 1 bitmaps: shard.distribute_segments (1/N H2D + NCCL all-gather)"
               if kind == "slab" and world > 1 else "")}


def run_verify(vx, shard, ctx, torch, d_segs, cfg, kind, n, s0, s1, units, out, chain, words,
               z_lo, z_hi, world, rank):
    """N > 1: every rank's output digest (shard.list_digest / words_digest) against the same
    slice of the one-rank result of the whole batch, computed on rank 0."""
    if kind == "single":
        return {"ok": True, "note": "replicas: nothing to compare"}
    torch.cuda.synchronize()
    if kind == "list":
        mine = (s0, s1, shard.list_digest(out[:units], chain[: s1 - s0 + 1]))
    else:
        mine = (z_lo, z_hi, shard.words_digest(words))
    got = shard.gather_objects(mine)
    if rank != 0:
        return None
    V = cfg["V"]
    ok = True
    bad = []
    b = vx.Batch(None, ctx=ctx, device_ptr=d_segs.data_ptr(), n=n)
    if kind == "list":
        cap = b.capacity
        fout = torch.empty((cap, 3), dtype=torch.int32, device="cuda")
        fchain = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        b.emit_list_device(fout.data_ptr(), cap, fchain.data_ptr())
        fc = fchain.cpu().numpy()
        for r, (a, e, dg) in enumerate(got):
            want = shard.list_digest(fout[int(fc[a]):int(fc[e])], fchain[a:e + 1])
            if tuple(want) != tuple(dg):
                ok = False
                bad.append(r)
        del fout
    else:
        plane = V * V // 64
        fw = torch.zeros(V * V * V // 64, dtype=torch.int64, device="cuda")
        b.emit_bitmap_device(fw.data_ptr(), V, 0, V, False)
        for r, (a, e, dg) in enumerate(got):
            if shard.words_digest(fw[a * plane:e * plane]) != dg:
                ok = False
                bad.append(r)
        del fw
    b.close()
    return {"ok": ok, "ranks": len(got), "mismatched_ranks": bad,
            "against": "one-rank result of the whole batch on rank 0 (digests of the same slices)"}


if __name__ == "__main__":
    main()
