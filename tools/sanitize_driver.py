"""Mid-size run of the look-back / shared-memory kernels for compute-sanitizer (tools/
gpu_sanitize.sh): plan_kernel (look-back offset scan), list_fused_kernel (count/emit task queues +
look-back), list_small_kernel (per-warp tiles + look-back), tiles_scan_lb_kernel, tiles_fill_kernel
(shared-memory tile, fixed-point samples with the FP64 redo of near-boundary lanes, streamed
readback), tiles_count / tiles_scatter (shared-memory walk state), perm_scatter (records copied
into walk order), long_chain_kernel (look-back over CTAs, shared-memory staging + bulk copy),
each output checked against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["VXG_LIST_MODE"] = "fused"  # the fused kernel even for a mid-size batch

import paper_2009_09500_b200 as vx  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402

orc = Oracle()
segs = vx.gen_segments(40000, 0, 600, 1024, 0x5A11)
vox, off, total = vx.run_batch_flat(segs)                      # plan_kernel + list_fused_kernel
ovox, ooff, ototal = orc.run_batch(segs)
assert total == ototal and np.array_equal(off, ooff) and np.array_equal(vox, ovox), "list"

rng = np.random.default_rng(0x5A15)  # tie lines: samples on half-integers (the fills' FP64 redo)
base = rng.integers(2, 200, size=(3000, 3)).astype(np.float64) + 0.5
ties = np.concatenate([base, base + rng.integers(1, 250, size=(3000, 1)) * np.array([1.0, 0.5, 0.25])],
                      axis=1)
bsegs = np.concatenate([vx.gen_segments(70000, 0, 300, 512, 0x5A12), ties])
b = vx.Batch(bsegs)
w, out = b.emit_bitmap(512, 0, 512)                             # count/scan_lb/scatter/fill
ow, oo = orc.bitmap(bsegs, 512)
assert out == oo and np.array_equal(w, ow), "bitmap"
w2, _ = b.emit_bitmap(512, 100, 300, clip=True)                 # slab select + clipped fill
ow2, _ = orc.bitmap(bsegs, 512, 100, 300)
assert np.array_equal(w2, ow2), "slab bitmap"
assert b.count_voxels() == orc.run_batch(bsegs)[2], "count"
junk = np.full(512 ** 3 // 64, np.uint64(0xF0F0F0F0F0F0F0F0), np.uint64)  # overwrite: store-only fill
w3, _ = b.emit_bitmap(512, 0, 512, words=junk, overwrite=True)
assert np.array_equal(w3, ow), "overwrite bitmap"
b.close()

import torch  # noqa: E402  (device buffers for the one-launch path)
vx.default_context().use_torch_stream()
ssegs = np.ascontiguousarray(vx.gen_segments(20000, 128, 0, 512, 0x5A13))
so, sc, st = orc.run_batch(ssegs)
d = torch.from_numpy(ssegs).cuda()
o = torch.empty((st, 3), dtype=torch.int32, device="cuda")
c = torch.empty(ssegs.shape[0] + 1, dtype=torch.int64, device="cuda")
t = vx.run_batch_device(d.data_ptr(), ssegs.shape[0], o.data_ptr(), st, c.data_ptr())
assert t == st and np.array_equal(o.cpu().numpy(), so) and np.array_equal(c.cpu().numpy(), sc)
for seg in (orc.gen_segment_of_length(200_000, 0x5A14),
            np.array([-7000.5, 300.5, 2.5, 60000.5, -4000.25, 900.0])):  # long chains, ties
    want = orc.voxelize_parametric(seg)
    lo = torch.zeros((len(want) + 3, 3), dtype=torch.int32, device="cuda")
    n = vx.voxelize_parametric_device(seg, lo.data_ptr(), lo.shape[0])
    assert n == len(want) and np.array_equal(lo[:n].cpu().numpy(), want), "long chain"
print("sanitize driver ok")
