"""GPU debug aid: where does the device bitmap differ from the oracle's? (run on a GPU box)"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_09500_b200 as vx  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402

o = Oracle()
for n, L, V in [(20000, 64, 256), (200, 64, 256), (1, 64, 256), (64, 64, 256)]:
    segs = vx.gen_segments(n, L, 0, V, 77)
    words, outside = vx.voxelize_bitmap(segs, V, clip=False)
    ow, oo = o.bitmap(segs, V)
    diff = words ^ ow
    bad = np.nonzero(diff)[0]
    missing = int(np.unpackbits((ow & ~words).view(np.uint8)).sum())
    extra = int(np.unpackbits((words & ~ow).view(np.uint8)).sum())
    print(f"n={n}: words differ {len(bad)}, missing bits {missing}, extra bits {extra}, "
          f"set gpu {int(np.unpackbits(words.view(np.uint8)).sum())} oracle "
          f"{int(np.unpackbits(ow.view(np.uint8)).sum())}")
    if len(bad):
        w = bad[0]
        bits = np.nonzero(np.unpackbits(np.array([diff[w]]).view(np.uint8), bitorder="little"))[0]
        b = w * 64 + bits[0]
        print("  first differing voxel", b % V, (b // V) % V, b // (V * V),
              "gpu has" if (words[w] >> np.uint64(bits[0])) & np.uint64(1) else "oracle has")

# which sample is missing for a single segment?
V = 256
segs = vx.gen_segments(1, 64, 0, V, 77)
words, _ = vx.voxelize_bitmap(segs, V, clip=False)
s = segs[0]
n, w = o.make_plan(s)
for k in range(n + 1):
    g = s[3:] if k >= n else s[:3] + np.array(w) * k
    vox = [int(np.floor(c + 0.5)) for c in g]
    b = vox[0] + V * (vox[1] + V * vox[2])
    has = (int(words[b >> 6]) >> (b & 63)) & 1
    if not has:
        print("missing k", k, "of N", n, "voxel", vox)
words, _ = vx.voxelize_bitmap(segs, V, clip=True)
ow, _ = o.bitmap(segs, V)
print("clip=True equal:", np.array_equal(words, ow))
