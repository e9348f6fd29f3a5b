"""Time one rank's share of config 5 on one GPU: the z-slab [r*V/N, (r+1)*V/N) of the full 64M
segments, as bench.py --gpus N would give rank r (device-resident, CUDA events). Used to choose
the walk-order sort for thin slabs. Usage: python tools/slab_probe.py N [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2009_09500_b200 as vx  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
V, n = 4096, 64 * 1024 * 1024
ctx = vx.default_context()
ctx.use_torch_stream()
d = torch.empty((n, 6), dtype=torch.float64, device="cuda")
ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, 0, 2048, V, 0x5EED0105, d.data_ptr(), 1))
h = V // N
words = torch.zeros(V * V * h // 64, dtype=torch.int64, device="cuda")
for r in (0, N // 2):
    times = []
    for _ in range(reps + 1):
        b = vx.Batch(None, ctx=ctx, device_ptr=d.data_ptr(), n=n)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.emit_bitmap_device(words.data_ptr(), V, r * h, (r + 1) * h, True)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        b.close()
    print(f"N={N} rank {r}: slab [{r * h}, {(r + 1) * h}) {min(times[1:]):.2f} ms")
