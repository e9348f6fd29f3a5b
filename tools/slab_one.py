"""One rank's share of config 5 (rank R of N, sample-balanced slab) through bench.py's N > 1
pipeline (device slab filter -> Batch -> clipped emit_bitmap), run twice -- for ncu launch lists.
Usage: python tools/slab_one.py N R"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2009_09500_b200 as vx  # noqa: E402
from paper_2009_09500_b200.shard import sample_balanced_slabs, select_slab_segments  # noqa: E402

N, R = int(sys.argv[1]), int(sys.argv[2])
V, n = 4096, 64 * 1024 * 1024
ctx = vx.default_context()
ctx.use_torch_stream()
d = torch.empty((n, 6), dtype=torch.float64, device="cuda")
ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, 0, 2048, V, 0x5EED0105, d.data_ptr(), 1))
bb = vx.Batch(None, ctx=ctx, device_ptr=d.data_ptr(), n=n)
z0, z1 = sample_balanced_slabs(bb.slab_samples, V, N)[R]
bb.close()
words = torch.zeros(V * V * (z1 - z0) // 64, dtype=torch.int64, device="cuda")
local = torch.empty_like(d)
for _ in range(2):
    cnt = select_slab_segments(ctx, d.data_ptr(), n, z0, z1, local.data_ptr()) if N > 1 else n
    b = vx.Batch(None, ctx=ctx, device_ptr=(local if N > 1 else d).data_ptr(), n=cnt)
    if N > 1:
        b.set_slab(z0, z1)  # (as bench.py: filtered above)
    b.emit_bitmap_device(words.data_ptr(), V, z0, z1, True, overwrite=True)  # (as bench.py)
    b.close()
torch.cuda.synchronize()
print(f"slab [{z0}, {z1})")
