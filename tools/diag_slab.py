"""GPU debug aid: config-5 geometry, full (unclipped) bitmap vs the 8 clipped z-slabs vs the
oracle; prints the first differing voxels and the segments that produce them."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_09500_b200 as vx  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402

o = Oracle()
V = 4096
ctx = vx.default_context()
nwords = V * V * V // 64
for n in [int(a) for a in (sys.argv[1:] or ["65536", "1048576"])]:
    d = torch.empty((n, 6), dtype=torch.float64, device="cuda")
    ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, 0, 2048, V, 0x5EED0005, d.data_ptr(), 1))
    b = vx.Batch(None, device_ptr=d.data_ptr(), n=n)
    full = torch.zeros(nwords, dtype=torch.int64, device="cuda")
    b.emit_bitmap_device(full.data_ptr(), V, 0, V, False)
    slabs = torch.zeros(nwords, dtype=torch.int64, device="cuda")
    h, per = V // 8, nwords // 8
    for g in range(8):
        b.emit_bitmap_device(slabs.data_ptr() + 8 * g * per, V, g * h, (g + 1) * h, True)
    cfull = torch.zeros(nwords, dtype=torch.int64, device="cuda")
    b.emit_bitmap_device(cfull.data_ptr(), V, 0, V, True)
    segs = d.cpu().numpy()
    ow, _ = o.bitmap(segs, V)
    ow = torch.from_numpy(ow.view(np.int64)).cuda()
    for name, x in [("full", full), ("slabs", slabs), ("clip-full", cfull)]:
        diff = torch.nonzero(x != ow).flatten()
        print(f"n={n} {name}: {diff.numel()} words differ from the oracle", flush=True)
        for w in diff[:4].tolist():
            a, r = int(x[w]), int(ow[w])
            dx = (a ^ r) & ((1 << 64) - 1)
            bit = (dx & -dx).bit_length() - 1
            bb = w * 64 + bit
            vox = (bb % V, (bb // V) % V, bb // (V * V))
            who = "gpu" if (a >> bit) & 1 else "oracle"
            lo = np.minimum(segs[:, :3], segs[:, 3:]) - 1
            hi = np.maximum(segs[:, :3], segs[:, 3:]) + 1
            cand = np.nonzero(np.all((lo <= vox) & (vox <= hi), axis=1))[0]
            hits = []
            for i in cand:
                ch = o.voxelize_parametric(segs[i])
                if np.any(np.all(ch == np.asarray(vox), axis=1)):
                    hits.append(i)
            print(f"   voxel {vox} only in {who}; oracle segments through it: "
                  f"{[(int(i), segs[i].tolist()) for i in hits[:3]]}", flush=True)
    del full, slabs, cfull, ow, d
    torch.cuda.empty_cache()

# write-only HBM roofline: zero / fill an 8 GiB buffer
buf = torch.empty(1 << 30, dtype=torch.int64, device="cuda")
for name, fn in [("zero_", lambda: buf.zero_()), ("fill_", lambda: buf.fill_(7))]:
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"write-only {name}: {8 * 2**30 / ms / 1e6:.1f} GB/s ({ms:.3f} ms per 8 GiB)")
