"""Time every rank's step of config 5 on one GPU -- what bench.py --gpus N runs on rank r: filter
the 64M broadcast segments to the rank's z-slab (sample-balanced; --equal for equal depths),
plan them, bin and fill the slab -- device-resident, CUDA events. The max over ranks estimates
the N-GPU step time (the slabs are independent: no collective on the data path). Then, as
bench.py does before timing, the slabs are rebalanced once from those times and timed again.
Usage: python tools/slab_probe.py N [--equal] [--no-rebalance]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2009_09500_b200 as vx  # noqa: E402
from paper_2009_09500_b200.shard import (sample_balanced_slabs, select_slab_segments,  # noqa: E402
                                         slab_bounds, time_balanced_slabs)

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
equal = "--equal" in sys.argv
V, n = 4096, 64 * 1024 * 1024
ctx = vx.default_context()
ctx.use_torch_stream()
d = torch.empty((n, 6), dtype=torch.float64, device="cuda")
ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, 0, 2048, V, 0x5EED0105, d.data_ptr(), 1))
bb = vx.Batch(None, ctx=ctx, device_ptr=d.data_ptr(), n=n)
slabs = [slab_bounds(V, N, r) for r in range(N)] if equal else sample_balanced_slabs(bb.slab_samples, V, N)
local = torch.empty_like(d)


def rank_step(z0, z1, reps=3):
    """bench.py's per-rank step on slab [z0, z1): best device ms of reps - 1 (after one warm-up)."""
    words = torch.zeros(max(V * V * (z1 - z0) // 64, 1), dtype=torch.int64, device="cuda")
    times = []
    cnt = n
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        src, cnt = d, n
        if N > 1:
            cnt = select_slab_segments(ctx, d.data_ptr(), n, z0, z1, local.data_ptr())
            src = local
        b = vx.Batch(None, ctx=ctx, device_ptr=src.data_ptr(), n=cnt)
        if N > 1:
            b.set_slab(z0, z1)  # (as bench.py: filtered above)
        b.emit_bitmap_device(words.data_ptr(), V, z0, z1, True, overwrite=True)  # (as bench.py)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        b.close()
    del words
    return min(times[1:]), cnt


def run(slabs, label):
    ts = []
    for r, (z0, z1) in enumerate(slabs):
        t, cnt = rank_step(z0, z1)
        ts.append(t)
        print(f"N={N} {label} rank {r}: slab [{z0}, {z1}) {t:.2f} ms (segments {cnt})")
    print(f"N={N} {label}: max over ranks {max(ts):.2f} ms")
    return ts


ts = run(slabs, "equal" if equal else "balanced")
if N > 1 and not equal and "--no-rebalance" not in sys.argv:
    # bench.py's partition: the sample-balanced slabs refined once from the ranks' measured steps
    slabs2 = time_balanced_slabs(bb.slab_samples, V, slabs, ts)
    run(slabs2, "rebalanced")
bb.close()
