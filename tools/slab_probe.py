"""Time every rank's share of config 5 on one GPU: the z-slab bench.py --gpus N would give rank r
(sample-balanced by default, --equal for equal depths) over the full 64M segments,
device-resident, CUDA events. The max over ranks is the N-GPU step time (the ranks' slabs are
independent: no collective on the data path). Usage: python tools/slab_probe.py N [--equal]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2009_09500_b200 as vx  # noqa: E402
from paper_2009_09500_b200.shard import sample_balanced_slabs, slab_bounds  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
equal = "--equal" in sys.argv
V, n = 4096, 64 * 1024 * 1024
ctx = vx.default_context()
ctx.use_torch_stream()
d = torch.empty((n, 6), dtype=torch.float64, device="cuda")
ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, 0, 2048, V, 0x5EED0105, d.data_ptr(), 1))
bb = vx.Batch(None, ctx=ctx, device_ptr=d.data_ptr(), n=n)
slabs = [slab_bounds(V, N, r) for r in range(N)] if equal else sample_balanced_slabs(bb.slab_samples, V, N)
bb.close()
worst = 0.0
for r, (z0, z1) in enumerate(slabs):
    words = torch.zeros(max(V * V * (z1 - z0) // 64, 1), dtype=torch.int64, device="cuda")
    times = []
    for _ in range(3):
        b = vx.Batch(None, ctx=ctx, device_ptr=d.data_ptr(), n=n)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.emit_bitmap_device(words.data_ptr(), V, z0, z1, True)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        b.close()
    t = min(times[1:])
    worst = max(worst, t)
    print(f"N={N} rank {r}: slab [{z0}, {z1}) {t:.2f} ms")
    del words
print(f"N={N} {'equal' if equal else 'balanced'}: max over ranks {worst:.2f} ms")
